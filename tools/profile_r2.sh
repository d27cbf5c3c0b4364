# Round-2 evidence (run on the GPU box through gpurun; only summaries come back: raw ncu reports
# exceed the 64 MiB limit of gpurun_out/).   bash tools/profile_r2.sh
set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2
mkdir -p $O
M=lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -c 40 --csv --log-file $O/two_d_counters_ordered.csv python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1 > /dev/null 2>&1
ncu --metrics $M --clock-control none -c 10 --csv --log-file $O/two_d_counters_hardware.csv python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1 hardware > /dev/null 2>&1
python tools/two_d_counters.py $O > $O/two_d_views_counters.json
cp $O/two_d_views_counters.json profiles/r2_two_d_views_counters.json  # bench.py attaches it to two_d_views
python bench.py > $O/bench_n1.json 2> $O/bench_n1.err
python bench.py --impl reference --steps 20 --warmup 3 > $O/bench_reference_arm.json 2>> $O/bench_n1.err
KRN_BENCH_BACKEND=gloo python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581 bench.py --gpus 2 --steps 20 --warmup 3 --rows 30000000 --skip-extras 2> /dev/null | tail -1 > $O/bench_2rank_one_gpu_rehearsal.json
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
cap ordered_16M "-k regex:ord_|scan_" 16 python tools/ordered_bench.py --only 16777216:uniform --reps 2
cap stencil_smooth "" 4 python tools/run_corpus_once.py stencil_smooth compiled 134217728 1
cap sum_squares_check_finite "-k regex:^g[0-9]" 4 python tools/run_corpus_once.py sum_squares compiled 33554432 1 check
python tools/ordered_bench.py --json $O/ordered_bench.json > $O/ordered_bench.txt 2>&1
python tools/atomic_policies.py --json $O/atomic_policies.json > $O/atomic_policies.txt 2>&1
python tools/sweep_mid.py --rows 10000 100000 300000 1000000 3000000 10000000 30000000 125000000 > $O/sweep_mid.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:laplacian -c 200 --csv --log-file $O/sweep_mid_ncu.csv python tools/sweep_mid.py --reps 4 > /dev/null 2>&1
python tools/corpus_bench.py --n 134217728 --md $O/corpus_generic_policies_134M.md > $O/corpus_134M.txt 2>&1
for p in inplace_axpy laplacian sum_squares; do python tools/check_finite_cost.py $p; done > $O/check_finite_cost.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
ls -la $O
