"""Selected columns of ncu --set full captures as one CSV: python tools/ncu_summary.py label=file.ncu-rep ... > profiles/x.csv"""
import csv, subprocess, sys
KEYS = ["Kernel Name","gpu__time_duration.sum","dram__bytes_read.sum","dram__bytes_write.sum","gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed","launch__registers_per_thread","launch__grid_size","launch__block_size","launch__shared_mem_per_block_static","launch__occupancy_limit_registers","launch__occupancy_limit_shared_mem","sm__warps_active.avg.pct_of_peak_sustained_active","smsp__inst_executed.sum","smsp__issue_active.avg.pct_of_peak_sustained_active","sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active","l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum","smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio","smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio","smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio","smsp__average_warps_issue_stalled_wait_per_issue_active.ratio","smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio","lts__t_sectors_op_red.sum","lts__t_sectors_op_atom.sum"]
out = csv.writer(sys.stdout)
first = True
for label, rep in [a.split("=") for a in sys.argv[1:]]:
    raw = subprocess.run(["ncu","-i",rep,"--page","raw","--csv"],capture_output=True,text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = [hdr.index(k) for k in KEYS if k in hdr]
    if first:
        out.writerow(["capture"] + [hdr[i] for i in idx]); first = False
    out.writerow([label + " [units]"] + [units[i] for i in idx])
    for r in data:
        out.writerow([label] + [r[i] for i in idx])
