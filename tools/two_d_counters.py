"""ncu counter CSVs of the gather_rows_rank2 gradient (tools/profile_r2.sh: two_d_counters_{ordered,hardware}.csv)
-> profiles/r2_two_d_views_counters.json, the object bench.py attaches to two_d_views.

    python tools/two_d_counters.py gpurun_out/r2 > profiles/r2_two_d_views_counters.json
"""
import csv
import json
import os
import re
import sys

ROWS, COLS = 16777216, 3


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    head = next(i for i, r in enumerate(rows) if r[0] == "ID")
    col = {name: k for k, name in enumerate(rows[head])}
    out: dict = {}
    for r in rows[head + 1:]:
        k = out.setdefault(int(r[col["ID"]]), {"kernel": r[col["Kernel Name"]]})
        value = float(r[col["Metric Value"]].replace(",", ""))
        unit = r[col["Metric Unit"]]
        scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "ns": 1e-3, "us": 1.0, "ms": 1e3}.get(unit, 1.0)
        k[r[col["Metric Name"]]] = value * scale
    return [out[i] for i in sorted(out)]


def short(name):
    name = re.sub(r"^void ", "", name)
    name = re.sub(r"\(anonymous namespace\)::|<unnamed>::", "", name)
    return name.split("(")[0]


def summary(path):
    ls = launches(path)
    first = next(i for i, k in enumerate(ls) if short(k["kernel"]) == "g1")  # the forward kernel of the primal run
    ls = ls[first + 1:]
    # the gradient call: its own forward-and-reverse kernel and whatever applies the queue
    grad = [k for k in ls if short(k["kernel"]) != "g1"]
    tot = lambda m: int(sum(k.get(m, 0.0) for k in grad))
    return {
        "kernels": len(grad),
        "time_us_sum": round(sum(k["gpu__time_duration.sum"] for k in grad), 1),
        "dram_bytes_read": tot("dram__bytes_read.sum"),
        "dram_bytes_write": tot("dram__bytes_write.sum"),
        "lts__t_sectors_op_red": tot("lts__t_sectors_op_red.sum"),
        "lts__t_sectors_op_atom": tot("lts__t_sectors_op_atom.sum"),
        "lts__t_sectors_op_read": tot("lts__t_sectors_op_read.sum"),
        "lts__t_sectors_op_write": tot("lts__t_sectors_op_write.sum"),
        "per_kernel": [{"kernel": short(k["kernel"]), "us": round(k["gpu__time_duration.sum"], 2),
                        "dram_bytes": int(k.get("dram__bytes_read.sum", 0) + k.get("dram__bytes_write.sum", 0)),
                        "lts_red_sectors": int(k.get("lts__t_sectors_op_red.sum", 0))} for k in grad],
    }


def main():
    d = sys.argv[1]
    out = {
        "rows": ROWS, "columns": COLS, "contributions": ROWS * COLS,
        "source": "ncu --metrics lts__t_sectors_op_red.sum,... --clock-control none, tools/run_corpus_once.py "
                  "gather_rows_rank2 compiled 16777216 1 [hardware] (tools/profile_r2.sh); gradient launch "
                  "sequence only (kernels after the forward kernel g1); tools/two_d_counters.py",
        "ordered": summary(os.path.join(d, "two_d_counters_ordered.csv")),
        "hardware_atomics": summary(os.path.join(d, "two_d_counters_hardware.csv")),
        # q rows x 3 read, idx and w read, _d_w written, _d_q rows x 3 read-modify-write (zero provenance: written)
        "compulsory_bytes": ROWS * 8 * (3 + 1 + 1 + 1 + 3 + 3),
        "note": "hardware policy: two 32 B reduction sectors per 8 B contribution at L2; ordered policy: no "
                "reductions, the queue moves through HBM in streaming passes (per-launch times are ncu's cold-cache, "
                "serialised figures)",
    }
    json.dump(out, sys.stdout, indent=1)
    print()


if __name__ == "__main__":
    main()
