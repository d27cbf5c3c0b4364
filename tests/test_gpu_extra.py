"""GPU parity of the additional programs (extra_programs/) against vectors produced by the
REFERENCE (tests/golden/extra.npz): BASELINE.json configs[3] - a 2-D View read through a
non-injective index map, whose gradient accumulates with atomics - and the shapes the
halo-recompute fusion must get right, under every execution policy."""

import numpy as np
import pytest

import paper_2507_13204_b200 as krn
from paper_2507_13204_b200 import ExecutionConfig, ViewStorage
from conftest import assert_bits
from test_extra_golden import EXTRA, SIZES, case, extra_golden  # noqa: F401

pytestmark = pytest.mark.gpu

POLICIES = {
    "fused": ExecutionConfig(policy="fused"),
    "compiled": ExecutionConfig(policy="compiled"),
    "pointwise": ExecutionConfig(policy="compiled", fuse_neighbours=False),
    "statements": ExecutionConfig(policy="statements"),
}
ATOMIC_TARGETS = {"gather_rows_rank2": {"_d_q"}}  # hardware atomics: order not deterministic


def _views(d):
    return {k: ViewStorage.from_values(k, v) if isinstance(v, np.ndarray) else v for k, v in d.items()}


@pytest.mark.parametrize("policy", sorted(POLICIES))
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("stem", EXTRA)
def test_primal_matches_reference(extra_golden, stem, n, policy):  # noqa: F811
    key, inputs, _ = case(extra_golden, stem, n)
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    call = _views(inputs)
    value = krn.execute(prog, fn.name, call, POLICIES[policy]).value
    want = extra_golden[f"{key}/primal/value"]
    if value is None:
        assert np.isnan(want)
    else:
        assert_bits(value, want, f"{key} {policy} value")
    for k, v in call.items():
        if isinstance(v, ViewStorage):
            assert_bits(v.buffer, extra_golden[f"{key}/primal/after/{k}"], f"{key} {policy} {k}")


def _gradient_cases():
    import os

    from conftest import GOLDEN

    g = np.load(os.path.join(GOLDEN, "extra.npz"))
    out = []
    for stem in EXTRA:
        if not bool(g[f"{stem}/has_grad"]):
            continue  # the reference's transform rejects the program (or it returns nothing)
        for apol in (["auto", "ordered", "red", "warp", "smem", "lead"] if stem in ATOMIC_TARGETS else ["auto"]):
            out.append((stem, apol))
    return out


@pytest.mark.parametrize("policy", sorted(POLICIES))
@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("stem,apol", _gradient_cases())
def test_gradient_matches_reference(extra_golden, stem, n, policy, apol):  # noqa: F811
    key, inputs, wrt = case(extra_golden, stem, n)
    prog = krn.load_program(stem)
    fn = prog.functions[0]
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    call = _views(inputs)
    for p in gfn.params[len(fn.params):]:
        call[p.name] = ViewStorage.from_values(p.name, extra_golden[f"{key}/grad/in/{p.name}"])  # accumulates
    cfg = POLICIES[policy]
    cfg = ExecutionConfig(policy=cfg.policy, fuse_neighbours=cfg.fuse_neighbours, atomic_policy=apol)
    assert krn.execute(gp, gfn.name, call, cfg).value is None
    for k, v in call.items():
        if not isinstance(v, ViewStorage):
            continue
        want = extra_golden[f"{key}/grad/after/{k}"]
        if k in ATOMIC_TARGETS.get(stem, ()) and apol not in ("auto", "ordered"):
            # BASELINE.json: relative 1e-12, stated because the order of atomics is not deterministic
            err = np.abs(v.buffer - want)
            assert np.all(err <= 1e-12 * np.maximum(np.abs(want), 1.0)), (key, policy, apol, k, err.max())
        else:
            assert_bits(v.buffer, want, f"{key} {policy} grad {k}")


def test_rank2_scatter_with_integer_contributions_is_exact():
    """sums of small integers are exact in any order: every accumulation policy must return the
    same bits for a rank-2 target hit through a non-injective map"""
    src = """fn f(idx: view<f64, 1>, acc: view<f64, 2>) {
        parallel_for i in 0..extent(idx, 0) {
            atomic_add(acc(idx(i), 0), 1.0);
            atomic_add(acc(idx(i), 2), 3.0);
            atomic_add(acc(0, 1), 2.0);
        } }"""
    p = krn.parse(src)
    rng = np.random.default_rng(5)
    n, rows = 150_000, 61
    idx = rng.integers(0, rows, size=n)
    counts = np.bincount(idx, minlength=rows).astype(np.float64)
    want = np.full((rows, 3), 0.25)
    want[:, 0] += counts
    want[:, 2] += 3.0 * counts
    want[0, 1] += 2.0 * n
    for policy in ("compiled", "statements"):
        for apol in ("red", "warp", "smem", "lead", "auto", "ordered"):
            acc = ViewStorage.from_values("acc", np.full((rows, 3), 0.25))
            krn.execute(p, "f", {"idx": ViewStorage.from_values("idx", idx.astype(np.float64)), "acc": acc},
                        ExecutionConfig(policy=policy, atomic_policy=apol))
            assert np.array_equal(acc.buffer, want), (policy, apol)


@pytest.mark.parametrize("policy", sorted(POLICIES))
@pytest.mark.parametrize("n", [1, 2, 7, 130, 1030, 300_001])
def test_taped_gradients_on_the_gpu(policy, n):
    """differentiate(tape=True) (lang/tape.py): the emitted gradient is an ordinary program; every
    policy must execute it like the oracle does, bit for bit (snapshots in registers or in HBM)"""
    from oracle import interp
    from test_tape import CASES, _inputs

    for name, (prog, fn_name, wrt) in sorted(CASES.items()):
        fn = prog.function(fn_name)
        gp = krn.differentiate(prog, fn_name, wrt, tape=True)
        gfn = gp.functions[-1]
        base = _inputs(fn, n, np.random.default_rng(n))
        shadows = [p.name for p in gfn.params[len(fn.params):]]
        got = _views(base)
        for s_, w in zip(shadows, wrt):
            got[s_] = ViewStorage.zeros(s_, base[w].shape)
        krn.execute(gp, gfn.name, got, POLICIES[policy])
        if n <= 2000:
            want = {k: v.copy() for k, v in base.items()}
            for s_, w in zip(shadows, wrt):
                want[s_] = np.zeros_like(base[w])
            interp.run(gp, gfn.name, want)
        else:
            ref = _views(base)
            for s_, w in zip(shadows, wrt):
                ref[s_] = ViewStorage.zeros(s_, base[w].shape)
            krn.execute(gp, gfn.name, ref, POLICIES["statements"])
            want = {k: v.buffer for k, v in ref.items()}
        for k in want:
            assert_bits(got[k].buffer, want[k], f"{name} {policy} n={n} {k}")


@pytest.mark.parametrize("policy", sorted(POLICIES))
@pytest.mark.parametrize("stem,wrt", [("stride2_scatter", ("fine", "w")), ("stride2_collide", ("fine", "w")),
                                      ("rank2_row_offset", ("m", "r"))])
def test_affine_maps_beyond_unit_stride_on_fresh_inputs(stem, wrt, policy):
    """general affine gather form: stride-2 maps with one writing iteration per location
    (direct read-modify-write), stride-2 maps where two iterations meet (ordered policy), row offsets
    onto a rank-2 target (gather form) - bit-identical to the CPU oracle at sizes the stored vectors
    do not cover, one launch for the gradients that need no sort"""
    from oracle import interp

    prog = krn.load_program(stem)
    fn = prog.functions[0]
    gp = krn.differentiate(prog, fn.name, wrt)
    gfn = gp.functions[-1]
    dev = krn.Device.get()
    for n in (3, 257, 4099, 40_001):
        rng = np.random.default_rng(n)
        data = {}
        for p in fn.params:
            data[p.name] = rng.normal(size=(2 * n + 1) if p.name == "fine" else ((n, 3) if p.type.rank == 2 else n))
        for sp, w in zip(gfn.params[len(fn.params):], wrt):
            data[sp.name] = rng.normal(size=np.shape(data[w]))
        want = {k: v.copy() for k, v in data.items()}
        interp.run(gp, gfn.name, want)
        got = _views(data)
        before = dev.launches()
        cfg = POLICIES[policy]
        krn.execute(gp, gfn.name, got, cfg)
        launches = dev.launches() - before
        for k, v in got.items():
            assert_bits(v.buffer, want[k], f"{stem} {policy} n={n} {k}")
        if policy in ("fused", "compiled") and stem != "stride2_collide":
            assert launches == 1, (stem, policy, n, launches)
