# Round-2 ncu evidence (run on the GPU box through gpurun; summaries only come back: the raw reports
# exceed the 64 MiB limit of gpurun_out/).
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2
mkdir -p $O
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_bench_n125M.csv python bench.py --steps 2 --warmup 3 --skip-extras > $O/bench_under_ncu.log 2>&1
cap() {  # label, kernel filter, count, command...
  label=$1; filter=$2; count=$3; shift 3
  ncu --set full --clock-control none $filter -c $count -o /tmp/$label "$@" > /dev/null 2>&1
  python tools/ncu_summary.py $label=/tmp/$label.ncu-rep > $O/ncu_full_$label.csv
  rm -f /tmp/$label.ncu-rep
}
cap laplacian "-k regex:laplacian_kernel" 6 python bench.py --steps 1 --warmup 1 --skip-extras
cap gather_rows_ordered "" 40 python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1
cap gather_rows_hardware "" 10 python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1 hardware
cap gather_indirect_ordered "" 40 python tools/run_corpus_once.py gather_indirect compiled 134217728 1
cap gather_indirect_hardware "" 10 python tools/run_corpus_once.py gather_indirect compiled 134217728 1 hardware
cap mean_shift "" 10 python tools/run_corpus_once.py mean_shift compiled 134217728 1
ls -la $O
