"""The reference's API on a B200, end to end: parse a kernel-language program, generate its
reverse-mode gradient, run both on the GPU, check the gradient, look at what the fusion pass built.

    python examples/quickstart.py [rows]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2507_13204_b200 as krn  # noqa: E402  (same names as the reference's `krn` package)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
rng = np.random.default_rng(0)

# 1. the headline objective of the paper: ||A(3x) - b||^2 with the 1-D Laplacian stencil
program = krn.load_program("laplacian")              # or krn.parse(open("my.krn").read())
fn = "normRes1DLaplacianSQ"
x, b = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)

xv = krn.ViewStorage.from_values("x", x)             # Views live in HBM; .buffer is the host mirror
f = krn.execute(program, fn, {"x": xv, "b": krn.ViewStorage.from_values("b", b)}).value
print(f"f(x, b)            = {f!r}   (x was scaled in place: x[0] = {xv.buffer[0]!r} = 3 * {x[0]!r})")

# 2. its Clad-style gradient: a new function of the same language, then one fused kernel on the GPU
gp = krn.differentiate(program, fn, ("x", "b"))
print("generated gradient :", sum(1 for _ in krn.emit(gp.functions[-1]).splitlines()), "lines of kernel language")
grads = krn.ad_gradient(program, fn, {"x": x, "b": b}, ("x", "b"), grad_program=gp)
print(f"df/dx[:3]          = {grads['x'][:3]}")

# 3. checked against the analytic gradient (the reference's oracle) at relative 1e-12
f_ref, gx_ref, gb_ref = krn.laplacian_oracle(x, b)
m = min(n, 2000)  # check_gradient builds a per-entry report: a sample is enough here
report = krn.check_gradient(np.concatenate([grads["x"][:m], grads["b"][:m]]), np.concatenate([gx_ref[:m], gb_ref[:m]]),
                            atol=0.0, rtol=1e-12)
print(f"against the analytic gradient: max relative error {report.max_rel_error:.2e}, passed = {report.passed}")

# 4. any other program goes through the fusion pass: CUDA generated from the tree
src = """fn energy(u: view<f64,1>) -> f64 {
    let s: view<f64,1> = view("s", extent(u, 0));
    parallel_for i in 0..extent(u, 0) {
        s(i) = u(i);
        if (i != 0) { s(i) += 0.25 * u(i - 1); }
        if (i != extent(u, 0) - 1) { s(i) += 0.25 * u(i + 1); }
    }
    parallel_for i in 0..extent(u, 0) { s(i) = s(i) * s(i); }
    e = parallel_sum(s);
    return e;
}"""
mine = krn.parse(src)
try:
    krn.differentiate(mine, "energy", ("u",))
except krn.NotFeasible as e:
    # like the reference: `s(i) = s(i) * s(i)` overwrites the value its own reversal needs ...
    print("reference behaviour:", e)
# ... tape=True snapshots it instead (not in the reference)
g = krn.differentiate(mine, "energy", ("u",), tape=True)
u = rng.normal(size=n)
dev = krn.Device.get()
before = dev.launches()
du = krn.ad_gradient(mine, "energy", {"u": u}, ("u",), grad_program=g)["u"]
print(f"energy gradient    : {dev.launches() - before} kernel launch(es) for "
      f"{sum(1 for s in g.functions[-1].body if type(s).__name__ in ('ParallelFor', 'ParallelSum', 'ParallelSumInto', 'DeepCopy'))}"
      f" statements; du[:3] = {du[:3]}")
# ... and against central finite differences on a few entries
probe = {"u": [0, 1, n // 2, n - 1]}
fd = krn.finite_difference_gradient(mine, "energy", {"u": u}, ("u",), entries=probe)["u"]
print(f"finite differences : {fd}  vs AD {du[probe['u']]}")

# 5. a NON-injective scatter (the adjoint of x(idx(i))): the reference applies its queue of atomic_adds in
#    (iteration, program order); so does the default policy here (stable partition by target + in-order
#    fold on the GPU), which makes the gradient bit-identical to the reference and to itself on every run.
#    deterministic_reduction=False trades that for hardware fp64 reductions (relative 1e-12).
gather = krn.load_program("gather_indirect")
m = min(n, 1 << 20)
xs, idx = rng.normal(size=m), rng.integers(0, m, size=m).astype(np.float64)
runs = [krn.ad_gradient(gather, "gatherSquares", {"x": xs, "idx": idx}, ("x",))["x"].copy() for _ in range(2)]
fast = krn.ad_gradient(gather, "gatherSquares", {"x": xs, "idx": idx}, ("x",),
                       cfg=krn.ExecutionConfig(deterministic_reduction=False))["x"]
print(f"indirect scatter   : two runs identical = {np.array_equal(runs[0], runs[1])}; hardware reductions differ by at most "
      f"{np.max(np.abs(fast - runs[0]) / np.maximum(np.abs(runs[0]), 1e-300)):.1e} (relative)")
print("done")
