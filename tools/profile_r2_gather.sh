set -x
cd $GRAFT_REPO_ROOT
O=gpurun_out/r2
mkdir -p $O
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
cap() { label=$1; filter=$2; count=$3; shift 3
  ncu --set full --clock-control none $filter -c $count -o /tmp/$label "$@" > /dev/null 2>&1
  python tools/ncu_summary.py $label=/tmp/$label.ncu-rep > $O/ncu_full_$label.csv; rm -f /tmp/$label.ncu-rep; }
cap gather_rows_ordered "" 40 python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1
cap gather_rows_hardware "" 10 python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1 hardware
cap gather_indirect_ordered "" 40 python tools/run_corpus_once.py gather_indirect compiled 134217728 1
cap gather_indirect_hardware "" 10 python tools/run_corpus_once.py gather_indirect compiled 134217728 1 hardware
M=lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
ncu --metrics $M --clock-control none -c 40 --csv --log-file $O/two_d_counters_ordered.csv python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1 > /dev/null 2>&1
ncu --metrics $M --clock-control none -c 10 --csv --log-file $O/two_d_counters_hardware.csv python tools/run_corpus_once.py gather_rows_rank2 compiled 16777216 1 hardware > /dev/null 2>&1
cat $O/smoke.txt
