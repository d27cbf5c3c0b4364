"""GPU parity of the ordered accumulation policy (csrc/krn_ordered.cu): deferred atomic_add
records applied per location as a left fold in (iteration, program order) - the reference's
apply loop, /root/reference/pkg/src/krn/runtime.py:430-447, 615-620 - through a stable radix
sort by target and an in-order segmented fold.  Bar: BIT-IDENTICAL to the CPU oracle and to the
vectors the reference produced, and identical from run to run (acceptance C5,
pkg/tests/test_acceptance.py:179-198)."""

import ctypes as C

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage, _cabi, parse
from paper_2507_13204_b200.runtime import Device
from conftest import assert_bits

pytestmark = pytest.mark.gpu


def _accumulate(target, keys, vals, width):
    """raw C ABI: krn_ordered_accumulate on device copies; returns the updated target"""
    dev = Device.get()
    lib = dev.lib
    t = np.ascontiguousarray(target, dtype=np.float64).copy()
    k = np.ascontiguousarray(keys, dtype=np.uint32)
    # the oracle takes record-major values (r * width + w), the library takes planes (w * records + r)
    v = np.ascontiguousarray(np.asarray(vals, dtype=np.float64).reshape(-1, width).T).reshape(-1)
    bufs = []
    for a in (t, k, v):
        p = dev.alloc(max(a.nbytes, 8))
        if a.nbytes:
            dev.upload(p, a)
        bufs.append(p)
    _cabi.check(lib.krn_ordered_accumulate(dev.h, C.c_void_p(bufs[0]), t.size, C.c_void_p(bufs[1]),
                                           C.c_void_p(bufs[2]), k.size, width))
    if t.size:
        dev.download(t, bufs[0])
    for p in bufs:
        dev.free(p)
    return t


def _key_maps(records, size, rng):
    maps = {
        "uniform": rng.integers(0, size, size=records),
        "all_zero": np.zeros(records, dtype=np.int64),
        "last": np.full(records, size - 1, dtype=np.int64),
        "hot_spot": np.where(rng.random(records) < 0.9, 3 % size, rng.integers(0, size, size=records)),
        "clustered": (np.arange(records) // 8) % size,
        "descending": (size - 1 - np.arange(records) % size),
    }
    # sites that did not execute: the all-ones mark
    holes = rng.integers(0, size, size=records).astype(np.uint32)
    holes[rng.random(records) < 0.3] = 0xFFFFFFFF
    maps["with_holes"] = holes
    # queues that are already in bucket order take the path on which no record moves (the in_order word of
    # csrc/krn_ordered.cu): sorted maps, affine maps with collisions, sorted with unexecuted sites at the end;
    # one unexecuted site or one early record in the middle puts the queue back on the partition path
    srt = np.sort(rng.integers(0, size, size=records)).astype(np.uint32)
    maps["sorted"] = srt
    maps["affine_collisions"] = np.minimum((np.arange(records) // 3) * 2 + (np.arange(records) % 3), size - 1)
    tail = srt.copy()
    tail[records - records // 4:] = 0xFFFFFFFF
    maps["sorted_holes_at_the_end"] = tail
    mid = srt.copy()
    if records > 2:
        mid[records // 2] = 0xFFFFFFFF
    maps["sorted_but_one_hole"] = mid
    late = srt.copy()
    if records > 2:
        late[records - 1] = srt[0]
    maps["sorted_but_the_last"] = late
    return maps


@pytest.mark.parametrize("size", [1, 2, 255, 256, 257, 5000, 65536, 1 << 20])
@pytest.mark.parametrize("records", [0, 1, 31, 4095, 4096, 4097, 70_001])
def test_queue_applied_like_the_reference(size, records):
    from oracle import cport

    rng = np.random.default_rng(size * 131 + records)
    for width in (1, 2, 3, 4):
        for label, keys in _key_maps(records, size, rng).items():
            keys = np.asarray(keys).astype(np.uint32)
            # magnitudes spread over 30 binades: any reordering of a location's fold shows in the bits
            vals = rng.normal(size=records * width) * np.exp2(rng.integers(-15, 15, size=records * width))
            target = rng.normal(size=size)
            want = target.copy()
            cport.apply_queue(want, keys, vals, width)
            got = _accumulate(target, keys, vals, width)
            assert_bits(got, want, f"size={size} records={records} width={width} {label}")


def test_queues_that_are_not_16_byte_aligned():
    """the second target of a launch starts wherever the first one's records end (key_off * n): the
    kernels' 128-bit key loads must not assume more than the element's own alignment"""
    from oracle import cport

    dev = Device.get()
    rng = np.random.default_rng(11)
    records, size = 70_001, 5000
    for label, keys in (("uniform", rng.integers(0, size, size=records)), ("sorted", np.sort(rng.integers(0, size, size=records)))):
        keys = keys.astype(np.uint32)
        vals = rng.normal(size=records)
        target = rng.normal(size=size)
        want = target.copy()
        cport.apply_queue(want, keys, vals, 1)
        for shift in (1, 2, 3):
            d_t, d_k, d_v = dev.alloc(8 * size), dev.alloc(4 * (records + 4)), dev.alloc(8 * (records + 4))
            dev.upload(d_t, target)
            dev.upload(d_k + 4 * shift, keys)
            dev.upload(d_v + 8 * shift, vals)
            _cabi.check(dev.lib.krn_ordered_accumulate(dev.h, C.c_void_p(d_t), size, C.c_void_p(d_k + 4 * shift),
                                                       C.c_void_p(d_v + 8 * shift), records, 1))
            got = np.empty(size)
            dev.download(got, d_t)
            for ptr in (d_t, d_k, d_v):
                dev.free(ptr)
            assert_bits(got, want, f"{label}, queue shifted by {shift} elements")


def test_long_runs_and_signed_zeros():
    """one location receiving a million records (the block-staged fold), -0.0 bookkeeping, NaN/Inf"""
    from oracle import cport

    rng = np.random.default_rng(3)
    records, size = 1_000_003, 1000
    keys = np.full(records, 7, dtype=np.uint32)
    keys[::1000] = rng.integers(0, size, size=keys[::1000].size)
    vals = rng.normal(size=2 * records)
    target = np.full(size, -0.0)
    want = target.copy()
    cport.apply_queue(want, keys, vals, 2)
    assert_bits(_accumulate(target, keys, vals, 2), want, "hot location")
    # -0.0 contributions leave -0.0; a location nobody names keeps its bits
    k = np.array([1, 1, 2], dtype=np.uint32)
    got = _accumulate(np.array([-0.0, -0.0, -0.0, 5.0]), k, np.array([-0.0, -0.0, 0.0]), 1)
    assert_bits(got, np.array([-0.0, -0.0, 0.0, 5.0]), "signed zeros")
    got = _accumulate(np.zeros(3), np.array([0, 0, 1, 1], dtype=np.uint32), np.array([np.inf, -np.inf, 1e308, 1e308]), 1)
    assert np.isnan(got[0]) and np.isinf(got[1]) and got[2] == 0.0


def test_sixteen_million_records_round_trip():
    """BASELINE-scale queue: sortedness-independent property - the fold of +v then -v over the same
    keys in the same order returns every location to target + (v - v) = target exactly when each
    location is hit once per sign... here: integer contributions, exact in any order, checked
    against bincount; and a second, identical call doubles them (run-to-run identical bits)."""
    rng = np.random.default_rng(9)
    records, size = 1 << 24, (1 << 22) + 17
    keys = rng.integers(0, size, size=records).astype(np.uint32)
    vals = rng.integers(1, 8, size=records).astype(np.float64)
    want = np.bincount(keys, weights=vals, minlength=size)
    got = _accumulate(np.zeros(size), keys, vals, 1)
    assert np.array_equal(got, want)


def _index_maps(n, rows, rng):
    return {
        "uniform": rng.integers(0, rows, size=n),
        "all_zero": np.zeros(n, dtype=np.int64),
        "hot_spot": np.where(rng.random(n) < 0.9, 3 % rows, rng.integers(0, rows, size=n)),
    }


@pytest.mark.parametrize("policy", ["fused", "compiled", "statements"])
def test_gather_indirect_gradient_bit_identical(policy):
    from oracle import interp

    prog = krn.load_program("gather_indirect")
    gp = krn.differentiate(prog, "gatherSquares", ("x",))
    rng = np.random.default_rng(21)
    for n, rows in ((1, 1), (257, 257), (5000, 64), (40_000, 40_000), (30_000, 7000)):
        x = rng.normal(size=rows) * np.exp2(rng.integers(-10, 10, size=rows))
        for label, idx in _index_maps(n, rows, rng).items():
            base = rng.normal(size=rows)
            want = {"x": x.copy(), "idx": idx.astype(np.float64), "_d_x": base.copy()}
            interp.run(gp, "gatherSquares_grad", want)
            runs = []
            for _ in range(2):
                got = {"x": ViewStorage.from_values("x", x), "idx": ViewStorage.from_values("idx", idx.astype(np.float64)),
                       "_d_x": ViewStorage.from_values("_d_x", base)}
                krn.execute(gp, "gatherSquares_grad", got, ExecutionConfig(policy=policy))
                runs.append(got["_d_x"].buffer.copy())
            assert_bits(runs[0], want["_d_x"], f"{policy} n={n} rows={rows} {label}")
            assert_bits(runs[1], runs[0], f"run to run {policy} n={n} rows={rows} {label}")


@pytest.mark.parametrize("policy", ["compiled", "statements"])
def test_one_million_rows_against_the_c_oracle(policy):
    """n = 10^6: the interpreter restatement is too slow here; the queue the
    gradient builds is r*x, x*r per iteration onto idx(i), which the C oracle applies in order"""
    from oracle import cport

    prog = krn.load_program("gather_indirect")
    gp = krn.differentiate(prog, "gatherSquares", ("x",))
    n = rows = 1_000_000
    rng = np.random.default_rng(4)
    x = rng.normal(size=rows)
    for label, idx in _index_maps(n, rows, rng).items():
        want = np.zeros(rows)
        r = 0.0 + 1.0  # _d_out(i) = 0 + seed
        vals = np.empty(2 * n)
        vals[0::2] = r * x[idx]
        vals[1::2] = x[idx] * r
        cport.apply_queue(want, idx.astype(np.uint32), vals, 2)
        got = {"x": ViewStorage.from_values("x", x), "idx": ViewStorage.from_values("idx", idx.astype(np.float64)),
               "_d_x": ViewStorage.zeros("_d_x", (rows,))}
        krn.execute(gp, "gatherSquares_grad", got, ExecutionConfig(policy=policy))
        first = got["_d_x"].buffer.copy()
        assert_bits(first, want, f"{policy} {label}")
        got = {"x": ViewStorage.from_values("x", x), "idx": ViewStorage.from_values("idx", idx.astype(np.float64)),
               "_d_x": ViewStorage.zeros("_d_x", (rows,))}
        krn.execute(gp, "gatherSquares_grad", got, ExecutionConfig(policy=policy, atomic_policy="ordered"))
        assert_bits(got["_d_x"].buffer, first, f"run to run {policy} {label}")


@pytest.mark.parametrize("policy", ["compiled", "statements"])
def test_guarded_sites_several_targets_and_reads_of_the_target(policy):
    """guarded sites (holes in the queue), two targets in one kernel, a rank-2 target, sites on one
    target that are NOT adjacent (separate records, program order), and a kernel that reads the View
    it scatters into (reads see pre-kernel values: the queue is applied at the kernel's end)"""
    from oracle import interp

    src = """fn f(idx: view<f64, 1>, v: view<f64, 1>, a: view<f64, 1>, m: view<f64, 2>, out: view<f64, 1>) {
        parallel_for i in 0..extent(idx, 0) {
            out(i) = a(idx(i)) + v(i);
            atomic_add(a(idx(i)), v(i));
            if (i != 0) { atomic_add(m(idx(i - 1), 1), v(i) * 3.0); }
            atomic_add(a(idx(i)), v(i) * v(i));
            atomic_add(a(0), 0.125);
            if (i < extent(idx, 0) - 2) { atomic_add(m(idx(i + 2), 2), v(i)); atomic_add(m(idx(i + 2), 2), -v(i + 1)); }
        } }"""
    p = parse(src)
    rng = np.random.default_rng(8)
    for n, rows in ((1, 1), (2, 3), (777, 50), (20_000, 20_000), (50_000, 9)):
        idx = rng.integers(0, rows, size=n).astype(np.float64)
        v = rng.normal(size=n) * np.exp2(rng.integers(-8, 8, size=n))
        a0, m0 = rng.normal(size=rows), rng.normal(size=(rows, 3))
        want = {"idx": idx.copy(), "v": v.copy(), "a": a0.copy(), "m": m0.copy(), "out": np.zeros(n)}
        interp.run(p, "f", want)
        got = {"idx": ViewStorage.from_values("idx", idx), "v": ViewStorage.from_values("v", v),
               "a": ViewStorage.from_values("a", a0), "m": ViewStorage.from_values("m", m0),
               "out": ViewStorage.zeros("out", (n,))}
        krn.execute(p, "f", got, ExecutionConfig(policy=policy))
        for k in ("a", "m", "out"):
            assert_bits(got[k].buffer, want[k], f"{policy} n={n} rows={rows} {k}")


def test_out_of_bounds_still_reported():
    p = parse("""fn f(idx: view<f64, 1>, a: view<f64, 1>) {
        parallel_for i in 0..extent(idx, 0) { atomic_add(a(idx(i)), 1.0); } }""")
    idx = np.array([0.0, 1.0, 5.0, 2.0])
    for policy in ("compiled", "statements"):
        with pytest.raises(krn.OutOfBounds, match=r"a\(5\) outside extent 3"):
            krn.execute(p, "f", {"idx": idx.copy(), "a": np.zeros(3)}, ExecutionConfig(policy=policy))


def test_hardware_policies_when_determinism_is_waived():
    """deterministic_reduction=False: 'auto' goes back to hardware reductions (rel 1e-12)"""
    from oracle import interp

    prog = krn.load_program("gather_indirect")
    gp = krn.differentiate(prog, "gatherSquares", ("x",))
    rng = np.random.default_rng(2)
    n = rows = 10_000
    x, idx = rng.normal(size=rows), rng.integers(0, rows, size=n).astype(np.float64)
    want = {"x": x.copy(), "idx": idx.copy(), "_d_x": np.zeros(rows)}
    interp.run(gp, "gatherSquares_grad", want)
    dev = Device.get()
    got = {"x": ViewStorage.from_values("x", x), "idx": ViewStorage.from_values("idx", idx),
           "_d_x": ViewStorage.zeros("_d_x", (rows,))}
    before = dev.launches()
    krn.execute(gp, "gatherSquares_grad", got, ExecutionConfig(deterministic_reduction=False))
    assert dev.launches() - before == 1  # one fused kernel, no sort
    assert np.all(np.abs(got["_d_x"].buffer - want["_d_x"]) <= 1e-12 * np.abs(want["_d_x"]))


@pytest.mark.parametrize("rows,ncols,cols", [(1, 3, (0, 1, 2)), (700, 3, (2, 0)), (5000, 3, (0, 1, 2)), (40_000, 5, (4, 1, 3, 0)),
                                             (3, 100, (99, 0, 50)), (300_000, 3, (1,))])
def test_row_records_with_column_planes(rows, ncols, cols):
    """krn_ordered_accumulate_rows: one record per ROW, value plane l goes to column cols[l] - the
    same as the flat queue in which every record is expanded into its per-element records"""
    from oracle import cport

    dev = Device.get()
    rng = np.random.default_rng(rows + ncols)
    for records in (1, 4097, 60_001):
        for label, keys in _key_maps(records, rows, rng).items():
            keys = np.asarray(keys).astype(np.uint32)
            planes = len(cols)
            vals = rng.normal(size=(records, planes)) * np.exp2(rng.integers(-12, 12, size=(records, planes)))
            target = rng.normal(size=(rows, ncols))
            # oracle: the flat queue, record r expanded in plane order (different columns never meet)
            flat_keys = np.where(keys[:, None] < rows, keys[:, None].astype(np.int64) * ncols + np.array(cols)[None, :],
                                 0xFFFFFFFF).astype(np.uint32).reshape(-1)
            want = target.copy()
            cport.apply_queue(want.reshape(-1), flat_keys, vals.reshape(-1), 1)
            t = target.copy()
            bufs = []
            for a in (t, keys, np.ascontiguousarray(vals.T)):
                p = dev.alloc(max(a.nbytes, 8))
                dev.upload(p, a)
                bufs.append(p)
            carr = (C.c_int * planes)(*cols)
            _cabi.check(dev.lib.krn_ordered_accumulate_rows(dev.h, C.c_void_p(bufs[0]), rows, ncols, carr, planes,
                                                            C.c_void_p(bufs[1]), C.c_void_p(bufs[2]), records))
            dev.download(t, bufs[0])
            for p in bufs:
                dev.free(p)
            assert_bits(t, want, f"rows={rows} ncols={ncols} cols={cols} records={records} {label}")


@pytest.mark.parametrize("policy", ["compiled", "statements"])
def test_lane_groups_mixed_with_other_sites_fall_back_to_element_records(policy):
    """a View whose lane groups do not all name the same columns (or that also has single-element
    sites) gives the row records up: still the reference's bits"""
    from oracle import interp

    src = """fn f(idx: view<f64, 1>, v: view<f64, 1>, m: view<f64, 2>) {
        parallel_for i in 0..extent(idx, 0) {
            atomic_add(m(idx(i), 0), v(i));
            atomic_add(m(idx(i), 2), 2.0 * v(i));
            atomic_add(m(0, 1), v(i));
            atomic_add(m(idx(i), 1), v(i) * v(i));
            atomic_add(m(idx(i), 2), -v(i));
        } }"""
    p = parse(src)
    rng = np.random.default_rng(1)
    for n, rows in ((1, 1), (500, 7), (30_000, 9000)):
        idx, v = rng.integers(0, rows, size=n).astype(np.float64), rng.normal(size=n)
        want = {"idx": idx.copy(), "v": v.copy(), "m": np.ones((rows, 3))}
        interp.run(p, "f", want)
        got = {"idx": ViewStorage.from_values("idx", idx), "v": ViewStorage.from_values("v", v),
               "m": ViewStorage.from_values("m", np.ones((rows, 3)))}
        krn.execute(p, "f", got, ExecutionConfig(policy=policy))
        assert_bits(got["m"].buffer, want["m"], f"{policy} n={n}")


# ---- errors of a gradient with indirect reads ---------------------------------------------------

def _gather_rows_case(n, rows, rng):
    return {"q": rng.normal(size=(rows, 3)), "idx": rng.integers(0, rows, size=n).astype(np.float64),
            "w": rng.normal(size=n), "_d_q": rng.normal(size=(rows, 3)), "_d_w": rng.normal(size=n)}


@pytest.mark.parametrize("fault", ["bad_row", "nan_row", "short_w", "short_w_and_shadow", "bad_row_and_short_shadow"])
def test_errors_of_a_gather_gradient_are_the_references(fault):
    """rowGather_grad: the statement the reference blames is the verbatim FORWARD sweep's (it runs
    first) even when the reverse sweep would fail as well; same exception class and message under the
    fused plan (forward and reverse sweep are one kernel there) and the statement path.
    (Measured and rejected in this round: NOT executing the dead forward sweep - every access of it is
    repeated by the reverse sweep - and replaying the statements when a status comes back: no gain,
    1.925 against 1.931 ms at 16.7 M rows; the sweep shares its loads with the reverse sweep.)"""
    from oracle import interp

    prog = krn.load_program("gather_rows_rank2")
    gp = krn.differentiate(prog, prog.functions[0].name, ("q", "w"))
    gfn = gp.functions[-1]
    rng = np.random.default_rng(5)
    data = _gather_rows_case(300, 40, rng)
    if fault in ("bad_row", "bad_row_and_short_shadow"):
        data["idx"][123] = 40.0
    if fault == "nan_row":
        data["idx"][7] = np.nan
    if fault in ("short_w", "short_w_and_shadow"):
        data["w"] = data["w"][:299]  # one failing iteration: which of several is reported first is a race
    if fault in ("short_w_and_shadow", "bad_row_and_short_shadow"):
        data["_d_w"] = data["_d_w"][:298]
    want = {k: v.copy() for k, v in data.items()}
    with pytest.raises(Exception) as ref:
        interp.run(gp, gfn.name, want)
    for policy in ("compiled", "statements"):
        got = {k: ViewStorage.from_values(k, v) for k, v in data.items()}
        with pytest.raises(Exception) as mine:
            krn.execute(gp, gfn.name, got, ExecutionConfig(policy=policy))
        assert type(mine.value).__name__ == type(ref.value).__name__, (policy, mine.value, ref.value)
        assert str(mine.value) == str(ref.value), (policy, str(mine.value), str(ref.value))
    # the context is usable afterwards
    good = _gather_rows_case(300, 40, np.random.default_rng(6))
    want = {k: v.copy() for k, v in good.items()}
    interp.run(gp, gfn.name, want)
    got = {k: ViewStorage.from_values(k, v) for k, v in good.items()}
    krn.execute(gp, gfn.name, got, ExecutionConfig(policy="compiled"))
    assert_bits(got["_d_q"].buffer, want["_d_q"], "_d_q after an error")
