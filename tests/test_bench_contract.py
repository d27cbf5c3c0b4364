"""CPU tier: the JSON lines committed under profiles/ (produced by bench.py on a B200) carry every
key of the measurement contract, and bench.py's reference arm / argument handling work without a
GPU as far as they can."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    with open(os.path.join(ROOT, "profiles", name)) as f:
        return json.loads(f.read().strip().splitlines()[-1])


def test_committed_bench_line_has_the_contract_keys():
    d = _load("r2_bench_n1.json")
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e",
              "gpu_launches", "clocks"):
        assert k in d, k
    assert d["dtype"] == "f64" and d["scaling"] == "weak" and d["vs_baseline"] is None and d["data"] == "synthetic"
    assert "workload" in d["config"] and "model" not in d["config"]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert r["traffic"] is None or r["traffic"] > 0
    c = d["cpu_baseline"]
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1 and c["value"] > 0 and c["sample"]
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and e["unit"] == d["unit"]
    assert e["value"] < d["value"]  # host buffers and PCIe inside the timed region: never the device-only figure
    assert d["gpu_launches"] == d["steps"]  # one fused kernel per step
    assert d["steps"] >= 1 and d["warmup"] >= 3
    assert set(d["clocks"]) >= {"sm_mhz", "sm_max_mhz", "reasons"}
    # BASELINE.json configs: [1] headline, [2] sweep, [3] 2-D Views
    ratio = d["ratio_grad_primal"]  # one object: the paper's size (latency bound) and the bandwidth-bound pair
    assert ratio["at_10k_entries_fused_one_launch_per_side"] <= 2.17 and ratio["at_10k_entries_statement_granular"] <= 2.17
    assert ratio["large_n_zero_shadows_40_over_24_bytes"] <= 2.17 < ratio["compulsory_bytes_ratio_accumulate"]
    assert "headline" in d and len(d["sweep"]) == 4 and "two_d_views" in d
    acc = d["two_d_views"]["gather_rows_rank2"]["accumulation"]  # configs[3]: both accumulation policies
    assert acc["ordered"]["bit_identical_to_reference"] and not acc["hardware_atomics"]["bit_identical_to_reference"]
    runs = c["interpreter"]["runs"]
    assert {(r["rows"], r["threads"] == 1) for r in runs} == {(10_000, True), (10_000, False), (100_000, True), (100_000, False)}
    assert d["generated_kernels"]["ld256"] is True


def test_committed_reference_arm_line():
    d = _load("r2_bench_reference_arm.json")
    mine = _load("r2_bench_n1.json")
    assert d["impl"] == "reference" and d["metric"] == mine["metric"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["e2e"]["value"] == d["value"] and d["cpu_baseline"]["value"] == d["value"]
    # the arm times the size its config names (round 1 labelled 125 M rows and timed 25 M)
    assert d["config"]["rows_per_gpu"] == mine["config"]["rows_per_gpu"] and d["config"]["rate_normalised"] is False
    assert d["config"]["workload"] == mine["config"]["workload"]


def test_reference_arm_runs_here():
    """the CPU arm needs no GPU: a short run must print one JSON line"""
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--rows", "200000"], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "port"
