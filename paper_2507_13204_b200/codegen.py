"""Program tree -> CUDA C++ for the statement-granular execution path.

One module per function: a grid-stride kernel per ``parallel_for``
(reference: _Compiler / _Interpreter.parallel_for,
/root/reference/pkg/src/krn/runtime.py:230-447, 567-624) and a one-thread kernel
per run of function-scope element statements (runtime.py:536-550).  The text
is compiled by NVRTC for sm_100a with ``--fmad=false``; it includes the
library's hand-written prelude (csrc/krn_prelude.cuh) for the accumulation
policies.

Semantics carried over from the interpreter, with the reference line:

* every access is bounds checked (runtime.py:299-321): the first failure is
  recorded in the context's status word and the iteration stops there
* a view value used as an index truncates toward zero (runtime.py:335)
* value expressions keep the tree's evaluation order; literals are emitted as
  hexadecimal floats so no decimal rounding can creep in
* ``atomic_add`` inside a kernel is deferred to the kernel boundary and applied
  in (iteration, program order) (runtime.py:430-447, 615-620).  Two policies,
  chosen per target view by ``plan_atomics``:

  - *gather* (targets of the form ``v(i + c [, const])``): the kernel stores
    each site's contribution into a staging column; a second generated kernel
    walks the *target locations* and adds the contributions that land there in
    exactly the reference's order.  Conflict-free, no atomics, bit-identical to
    the interpreter, and reads inside the kernel see pre-kernel values as the
    deferred semantics demand.
  - *atomic* (indirect or otherwise non-injective targets): hardware fp64
    reductions, warp-aggregated; the sum is exact up to reassociation (the
    1e-12 relative tolerance of the parity contract).  If the kernel also reads
    or plainly writes the target view the contributions are staged and applied
    by a second kernel so that the deferral is still honoured.
"""

from __future__ import annotations

import dataclasses as _dc

from .lang.dataflow import normalize_index
from .lang.nodes import kind, walk_expr, walk_statements

_ELEMENT = ("DeclScalar", "AssignScalar", "AssignView", "AtomicAdd", "If")


def c_double(v: float) -> str:
    v = float(v)
    if v != v or v in (float("inf"), float("-inf")):
        raise ValueError("non-finite literal")
    return "(" + v.hex() + ")"


# ---------------------------------------------------------------------------
# atomic scheduling


@_dc.dataclass
class Site:
    """One atomic_add statement of a kernel."""

    index: int  # program order among the kernel's sites
    stmt: object
    guards: tuple  # enclosing If conditions, outermost first
    view: str
    offset: object = None  # int c when the row index is `counter + c`
    column: object = None  # int or None (rank-1)
    mode: str = "atomic"  # "gather" | "direct" | "atomic" | "staged_atomic"
    merged: tuple = ()  # sites folded into this one (merge_adjacent_atomics)
    absorbed: bool = False  # this site's contribution travels with an earlier site
    ord: object = None  # (key offset, value offset, groups, width, group): record layout of the ordered policy
    lanes: bool = False  # head of a run of sites on the literal columns of ONE row of a rank-2 View (`merged`)


def _unit_affine(idx, counter):
    """``counter + c`` with literal c -> c, else None."""
    try:
        const, terms = normalize_index(idx)
    except (TypeError, ValueError):
        return None
    if terms == ((("counter", counter), 1),):
        return const
    return None


def _constant(idx):
    try:
        const, terms = normalize_index(idx)
    except (TypeError, ValueError):
        return None
    return const if not terms else None


def _affine(idx, counter):
    """``a * counter + c (+ counter-free symbolic terms)`` -> (a, c, symbolic terms), a != 0; else None."""
    try:
        const, terms = normalize_index(idx)
    except (TypeError, ValueError):
        return None
    a, rest = 0, []
    for atom, coef in terms:
        if atom == ("counter", counter):
            a = coef
        elif atom[0] in ("counter", "view"):
            return None
        else:
            rest.append((atom, coef))
    return (a, const, tuple(rest)) if a != 0 else None


def _injective(group, counter) -> bool:
    """True when no two DIFFERENT iterations of the kernel can name one location through the sites of
    `group` (all on one View): every row index is ``a*i + c_k`` with one common stride a and one common
    symbolic part, and two sites either name the same location in the same iteration (equal c, equal
    column) or can never meet (different literal columns, or c_k - c_l not a multiple of a).  This is
    the injectivity refinement of the reference's conservative race rule 2 (analysis.py:204-248,
    271-303: `normalize_index` is the information source)."""
    forms = []
    for st in group:
        idx = st.stmt.target.indices
        f = _affine(idx[0], counter)
        col = _constant(idx[1]) if len(idx) == 2 else 0
        if f is None or col is None:
            return False
        forms.append((f, col))
    (a, _, sym), _ = forms[0]
    for (fa, fc, fs), col in forms:
        if fa != a or fs != sym:
            return False
    for i, ((_, c1, _), col1) in enumerate(forms):
        for (_, c2, _), col2 in forms[i + 1:]:
            if col1 == col2 and c1 != c2 and (c1 - c2) % abs(a) == 0:
                return False
    return True


def plan_atomics(loop) -> list:
    """Sites of a kernel with their accumulation policy."""
    sites: list = []

    def collect(body, guards):
        for s in body:
            if kind(s) == "AtomicAdd":
                sites.append(Site(len(sites), s, guards, s.target.view))
            elif kind(s) == "If":
                collect(s.body, guards + (s.cond,))

    collect(loop.body, ())
    if not sites:
        return sites

    touched_plainly = set()  # views read or plainly written by the kernel
    for s in walk_statements(loop.body):
        k = kind(s)
        exprs = []
        if k == "AssignView":
            touched_plainly.add(s.target.view)
            exprs = list(s.target.indices) + [s.rhs]
        elif k == "AtomicAdd":
            exprs = list(s.target.indices) + [s.value]
        elif k == "DeclScalar":
            exprs = [s.init]
        elif k == "AssignScalar":
            exprs = [s.rhs]
        for e in exprs:
            for n in walk_expr(e):
                if kind(n) == "ViewAccess":
                    touched_plainly.add(n.view)

    by_view: dict = {}
    for st in sites:
        by_view.setdefault(st.view, []).append(st)
    for view, group in by_view.items():
        gather = True
        for st in group:
            idx = st.stmt.target.indices
            st.offset = _unit_affine(idx[0], loop.counter)
            st.column = _constant(idx[1]) if len(idx) == 2 else None
            if st.offset is None or (len(idx) == 2 and st.column is None):
                gather = False
        # every location has ONE writing iteration (strided / reversed / column-disjoint affine maps the
        # reference flags conservatively): that iteration adds its contributions itself, in program
        # order - plain read-modify-write, no staging, no atomics, bit-identical.  Not when the kernel
        # also reads the View (deferral: reads must see pre-kernel values).
        direct = not gather and view not in touched_plainly and _injective(group, loop.counter)
        for st in group:
            if gather:
                st.mode = "gather"
            elif direct:
                st.mode = "direct"
            else:
                st.mode = "staged_atomic" if view in touched_plainly else "atomic"
    merge_adjacent_atomics(loop.body, {id(st.stmt): st for st in sites})
    return sites


def merge_adjacent_atomics(body, by_id) -> None:
    """Hardware-atomic sites that follow each other directly and name the same location - the
    product rule's `atomic_add(_d_x(idx(i)), r * x(idx(i))); atomic_add(_d_x(idx(i)), x(idx(i)) * r);`
    - issue ONE reduction with the sum of their values.  Nothing can observe the location in
    between (an "atomic"-mode target is neither read nor plainly written by the kernel), and the
    policy is exact only up to reassociation anyway (d + (a + b) for (d + a) + b); gather-mode
    sites, which are bit-identical to the interpreter, are never merged.  Under the ordered policy
    the merged sites stay apart as the values of one record.

    Sites that follow each other directly and name DIFFERENT literal columns of one row of a rank-2
    View (`atomic_add(_d_q(idx(i), 0), .); atomic_add(_d_q(idx(i), 1), .); ...`) are grouped the
    same way (`lanes`): one record per row under the ordered policy instead of one per element."""
    head = None
    for s in body:
        k = kind(s)
        st = by_id.get(id(s)) if k == "AtomicAdd" else None
        if st is not None and st.mode == "atomic":
            idx = s.target.indices
            if head is not None and len(head.merged) + 1 < ORDERED_WIDTH:
                hidx = head.stmt.target.indices
                if not head.lanes and head.stmt.target == s.target:
                    head.merged += (st,)
                    st.absorbed = True
                    continue
                col, hcols = (_constant(idx[1]) if len(idx) == 2 else None), None
                if len(idx) == 2 and len(hidx) == 2 and head.stmt.target.view == s.target.view and hidx[0] == idx[0] \
                        and (head.lanes or not head.merged):
                    hcols = [_constant(hidx[1])] + [_constant(m.stmt.target.indices[1]) for m in head.merged]
                if hcols is not None and col is not None and None not in hcols and col not in hcols:
                    head.merged += (st,)
                    head.lanes = True
                    st.absorbed = True
                    continue
            head = st
            continue
        head = None
        if k == "If":
            merge_adjacent_atomics(s.body, by_id)


ORDERED_WIDTH = 4  # values one record of the ordered policy carries (krn_ordered_accumulate: width <= 4)


def assign_ordered(site_lists) -> list:
    """Record layout of the ordered accumulation policy (csrc/krn_ordered.cu) for the kernels
    that share one launch.  Per kernel and target View with hardware-atomic sites: the sites in
    program order form `groups` record slots per iteration (a head site and the sites merged
    into it share one record of `width` values), record number = iteration * groups + group -
    the reference's queue order (runtime.py:430-447: appended per iteration in program order,
    sorted by (iteration, sequence number)).  Offsets are in units of the trip count.

    `cols` (a tuple of literal columns) marks a queue of ROW records: every group of the View is a
    run of sites on the same literal columns of one row, the key is the row and value plane l goes
    to column cols[l].  A View with lane groups that do not all name the same columns gives the
    grouping up: each of those sites becomes a record of its own again."""
    entries, key_off, val_off = [], 0, 0
    for sites in site_lists:
        by_view: dict = {}
        for st in sites:
            if st.mode in ("atomic", "staged_atomic"):
                by_view.setdefault(st.view, []).append(st)
        for view, every in by_view.items():
            lane_heads = [st for st in every if st.lanes]
            cols = None
            if lane_heads:
                shapes = {tuple([_constant(st.stmt.target.indices[1])] + [_constant(m.stmt.target.indices[1]) for m in st.merged])
                          for st in lane_heads}
                heads_all = [st for st in every if not st.absorbed]
                if len(shapes) == 1 and len(lane_heads) == len(heads_all):
                    cols = next(iter(shapes))
                else:
                    for st in lane_heads:  # mixed shapes: back to one record per site
                        for m in st.merged:
                            m.absorbed = False
                        st.merged, st.lanes = (), False
            heads = [st for st in every if not st.absorbed]
            groups, width = len(heads), max(1 + len(st.merged) for st in heads)
            for g, st in enumerate(heads):
                st.ord = (key_off, val_off, groups, width, g)
            entries.append(dict(view=view, groups=groups, width=width, key_off=key_off, val_off=val_off, cols=cols,
                                guarded=any(st.guards for st in every)))
            key_off += groups
            val_off += groups * width
    return entries


def _never_same_location(t1, t2) -> bool:
    """Index tuples t1 (evaluated by iteration i1) and t2 (by a DIFFERENT iteration i2), both in
    normalize_index form: True when they provably never name one location."""
    for (c1, terms1), (c2, terms2) in zip(t1, t2):
        if terms1 != terms2 or any(atom[0] == "view" for atom, _ in terms1):
            continue  # nothing to conclude from this component
        coef = [c for atom, c in terms1 if atom[0] == "counter"]
        if not coef:
            if c1 != c2:
                return True  # two different constants (same extent terms)
        elif c1 == c2 or (c1 - c2) % coef[0] != 0:
            return True  # a*i1 + c1 == a*i2 + c2 would need i1 == i2 / a non-integer shift
    return False


def carries_across_iterations(loop) -> bool:
    """True when, as far as the index expressions tell, two different iterations of `loop` may
    touch one location with a plain write among the two accesses - the situation in which the
    result depends on the order of the iterations (the reference at threads=1 runs them 0..n-1,
    runtime.py:586-593; its own tests rely on it: tests/test_runtime.py:101-115).  Index
    expressions are affine in the counter or go through a View (then nothing is known)."""
    writes: dict = {}
    every: dict = {}

    def note(acc, plain_write=False):
        try:
            norm = tuple(normalize_index(i) for i in acc.indices)
        except (TypeError, ValueError):
            norm = None
        every.setdefault(acc.view, []).append(norm)
        if plain_write:
            writes.setdefault(acc.view, []).append(norm)
        for i in acc.indices:
            for node in walk_expr(i):
                if kind(node) == "ViewAccess":
                    note(node)

    for s in walk_statements(loop.body):
        k = kind(s)
        exprs = []
        if k == "AssignView":
            note(s.target, True)
            exprs = [s.rhs]
        elif k == "AtomicAdd":
            note(s.target)
            exprs = [s.value]
        elif k == "DeclScalar":
            exprs = [s.init]
        elif k == "AssignScalar":
            exprs = [s.rhs]
        elif k == "If":
            exprs = [s.cond.lhs, s.cond.rhs]
        for e in exprs:
            for node in walk_expr(e):
                if kind(node) == "ViewAccess":
                    note(node)
    for view, ws in writes.items():
        for w in ws:
            for other in every[view]:
                if w is None or other is None or not _never_same_location(w, other):
                    return True
    return False


def guard_interval(guards, counter, trip, sym):
    """(lo, up): the running index satisfies lo <= i <= n-1-up under `guards`, where n is the
    trip count (`trip` = its canonical form, `sym` = the canonicaliser)."""
    lo, up = 0, 0
    counter_terms = ((("counter", counter), 1),)
    for c in guards:
        try:
            (lc, lt), (rc, rt) = sym(c.lhs), sym(c.rhs)
        except (TypeError, ValueError):
            continue
        op = c.op
        if rt == counter_terms and lt != counter_terms:  # put the counter on the left
            (lc, lt), (rc, rt) = (rc, rt), (lc, lt)
            op = {"<": ">", "<=": ">=", ">": "<", ">=": "<=", "==": "==", "!=": "!="}[op]
        if lt != counter_terms:
            continue
        k_const = rc - lc  # condition reads: i  op  (rt-part) + k_const
        if not rt:  # compared with a constant
            if op == "!=" and k_const == lo:
                lo += 1
            elif op == ">":
                lo = max(lo, k_const + 1)
            elif op == ">=":
                lo = max(lo, k_const)
        elif (0, rt) == (0, trip[1]):  # compared with n + k  (same symbolic terms as the trip count)
            k_rel = k_const - trip[0]  # rhs = n + k_rel
            if op == "!=" and k_rel == -1 - up:
                up += 1
            elif op == "<":
                up = max(up, -k_rel)
            elif op == "<=":
                up = max(up, -k_rel - 1)
    return lo, up


# ---------------------------------------------------------------------------
# module generation

_PREAMBLE = r"""
#include "krn_prelude.cuh"
#define NV %(nv)d
#define NH %(nh)d
struct Env {
    double *v[NV > 0 ? NV : 1];
    krn_i64 e0[NV > 0 ? NV : 1];
    krn_i64 e1[NV > 0 ? NV : 1];
    double *S;          // function-scope scalars that live on the device (gather results, ...)
    krn_i64 *status;
    double H[NH > 0 ? NH : 1];  // function-scope scalars the host knows, passed by value
    krn_i64 priv_rows;  // accumulation policy of atomic_add targets (chosen by the host per launch):
    int apol;           //   0 plain RED.ADD.F64, 1 warp-aggregated, 2 shared-memory privatised, 3 leader-aggregated
    int priv_vid;       //   view whose rows are privatised when apol == 2
    unsigned *okeys;    // apol == 4 (ordered): the kernel only records (target offset, values) per site group,
    double *ovals;      //   krn_ordered_accumulate applies them afterwards in the reference's order
    krn_i64 on;         //   trip count of the kernel (records of one group: on)
    int *fin;           // check_finite inside fused kernels: fin[checkpoint * NV + view] = 1 when a value of the
};                      //   View is non-finite after that statement (compiled._CompiledRun.finite_replay)
__device__ __forceinline__ void krn_fin(const Env &E, int slot, double x)
{
    if ((__double2hiint(x) & 0x7ff00000) == 0x7ff00000) E.fin[slot] = 1;  // Inf or NaN: exponent all ones
}
// element k (-4 .. 7, relative to the lane's own four) of a read-only View held as P[4] plus halo registers
#define KRN_NBR(P, k) ((k) < 0 ? P##L[-(k) - 1] : (k) < 4 ? P[(k) < 0 ? 0 : (k) < 4 ? (k) : 0] : P##R[(k) - 4 < 0 ? 0 : (k) - 4])
// the same test as one bit of a per-thread mask (tilegen._defer_finite_flags): !(|x| < Inf) is true for Inf and NaN
#define KRN_FINB(k, x) (finbits_ |= (unsigned long long)(!(fabs(x) < __longlong_as_double(0x7ff0000000000000ll))) << (k))
extern __shared__ double krn_priv[];
__device__ __forceinline__ void krn_scatter(const Env &E, int v, krn_i64 o, double t)
{
    if (E.apol == 2 && v == E.priv_vid) atomicAdd(&krn_priv[o], t);
    else if (E.apol == 1) krn_red_add_aggregated(&E.v[v][o], t);
    else if (E.apol == 3) krn_red_add_leader(&E.v[v][o], t);
    else krn_red_add(&E.v[v][o], t);
}
// ordered policy: record r = i * G + g of the target's queue (layout: codegen.assign_ordered); values
// beyond the group's own sites are -0.0, the additive identity (x + -0.0 == x bit for bit, -0.0 included)
__device__ __forceinline__ void krn_ord_put(const Env &E, krn_i64 ko, krn_i64 vo, int G, int W, int g, krn_i64 i,
                                            krn_i64 o, double a, double b, double c, double d)
{
    const krn_i64 r = i * G + g, plane = E.on * G;  // values are planes of on * G doubles
    E.okeys[ko * E.on + r] = (unsigned)o;
    double *p = E.ovals + vo * E.on + r;
    p[0] = a;
    if (W > 1) p[plane] = b;
    if (W > 2) p[2 * plane] = c;
    if (W > 3) p[3 * plane] = d;
}
// -0.0 is the additive identity: a privatised row that still holds it received nothing
__device__ __forceinline__ void krn_priv_begin(const Env &E)
{
    if (E.apol == 2) {
        for (krn_i64 k = threadIdx.x; k < E.priv_rows; k += blockDim.x) krn_priv[k] = -0.0;
        __syncthreads();
    }
}
__device__ __forceinline__ void krn_priv_end(const Env &E)
{
    if (E.apol == 2) {
        __syncthreads();
        for (krn_i64 k = threadIdx.x; k < E.priv_rows; k += blockDim.x) {
            double s = krn_priv[k];
            if (__double_as_longlong(s) != __double_as_longlong(-0.0)) krn_red_add(&E.v[E.priv_vid][k], s);
        }
    }
}
// bounds-checked linear offsets; on failure record {code,line,view,i,j} and flag the iteration
__device__ __forceinline__ krn_i64 off1(const Env &E, int v, krn_i64 i, int line, bool &bad)
{
    if (i < 0 || i >= E.e0[v]) {
        if (!bad) krn_fail(E.status, 1, line, v, i, 0);
        bad = true;
        return 0;
    }
    return i;
}
__device__ __forceinline__ krn_i64 off2(const Env &E, int v, krn_i64 i, krn_i64 j, int line, bool &bad)
{
    if (i < 0 || i >= E.e0[v] || j < 0 || j >= E.e1[v]) {
        if (!bad) krn_fail(E.status, 1, line, v, i, j);
        bad = true;
        return 0;
    }
    return i * E.e1[v] + j;
}
__device__ __forceinline__ double rd(const Env &E, int v, krn_i64 off, bool bad)
{
    return bad ? 0.0 : E.v[v][off];
}
// int(value): truncation toward zero; NaN/Inf cannot be converted
__device__ __forceinline__ krn_i64 to_index(const Env &E, double x, int line, int v, bool &bad)
{
    if (bad) return 0;
    if (!(x == x) || x - x != 0.0) {
        krn_fail(E.status, 2, line, v, x == x ? 1 : 0, 0);
        bad = true;
        return 0;
    }
    if (x >= 4.0e18) return 4000000000000000000ll;
    if (x <= -4.0e18) return -4000000000000000000ll;
    return (krn_i64)x;
}
"""

# Conflict detector (reference: _Tracer, runtime.py:198-227; parallel_for under
# cfg.conflict_detect, runtime.py:574-585).  A traced kernel is a DRY replay of the body: every
# address is computed and checked as in the real kernel, loads are performed, stores and
# atomic_adds are not; each access tags its location instead.  One 64-bit word per element:
#   bits 0-2  kinds seen (1 read, 2 plain write, 4 atomic)
#   bit  3    touched by at least two distinct iterations
#   bits 4-   first iteration seen, plus one (0 = untouched)
# The word is order independent in everything the report uses (kinds, the two-iterations bit).
# phase 0 tags and counts the locations that become conflicts (two iterations, one plain write);
# phase 1 replays and emits (view | kinds << 32, offset, iteration) for every access to such a
# location, which the host sorts into the reference's records.
_TRACE = r"""
struct Trace {
    unsigned long long *tag[NV > 0 ? NV : 1];
    unsigned long long *count;   // [0] conflicting locations (phase 0), [1] triples produced (phase 1)
    krn_i64 *triples;
    krn_i64 cap;                 // triples the buffer holds; production beyond it is only counted
    int phase;
};
__device__ __forceinline__ void krn_touch(const Trace &T, int v, krn_i64 off, krn_i64 i, unsigned kind)
{
    unsigned long long *w = T.tag[v] + off;
    unsigned long long cur = *(volatile unsigned long long *)w;
    if (T.phase == 0) {
        const unsigned long long me = (unsigned long long)(i + 1);
        for (;;) {
            unsigned long long want;
            if (cur == 0) want = (me << 4) | kind;
            else if ((cur >> 4) == me) want = cur | kind;
            else want = cur | 8ull | kind;
            if (want == cur) return;
            const unsigned long long old = atomicCAS(w, cur, want);
            if (old == cur) {
                const bool was = (cur & 8ull) && (cur & 2ull), is = (want & 8ull) && (want & 2ull);
                if (is && !was) atomicAdd(&T.count[0], 1ull);
                return;
            }
            cur = old;
        }
    } else if ((cur & 8ull) && (cur & 2ull)) {
        const unsigned long long k = atomicAdd(&T.count[1], 1ull);
        if ((krn_i64)k < T.cap) {
            T.triples[3 * k] = (krn_i64)v | ((krn_i64)(cur & 7ull) << 32);
            T.triples[3 * k + 1] = off;
            T.triples[3 * k + 2] = i;
        }
    }
}
__device__ __forceinline__ double krn_trace_rd(const Env &E, const Trace &T, krn_i64 i, int v, krn_i64 off, bool bad)
{
    if (bad) return 0.0;
    krn_touch(T, v, off, i, 1u);
    return E.v[v][off];
}
"""


class ModuleBuilder:
    """Generates the CUDA source of one function and the launch recipes the
    executor needs (kernel names, staging requirements)."""

    def __init__(self, fn, host_scalars=()):
        self.fn = fn
        self.host_scalars = set(host_scalars)
        self.hslots: dict = {}  # host-known scalar -> slot in Env.H
        self.promoted: dict = {}  # view -> register array name, while a tile kernel is generated
        self.windows: dict = {}  # view -> warp-private shared-memory window (window kernels, tilegen.py)
        self.stage_windows: dict = {}  # atomic site index -> window name (contribution read by a neighbour row)
        self.in_tile = False  # a window kernel is being generated
        self.interior = None  # dict(counter, trip, sym, lo, up) while an interior warp step is generated
        self.counter = None  # AST counter of the statement being generated (window kernels)
        self.nbr = {}  # read-only Views read at i + c inside a tile kernel's interior steps: view -> register stem
        self.elide = None  # bounds-check elision context (tile kernels only)
        self.guards: list = []  # enclosing If conditions of the statement being generated
        self.tracing = False  # a dry, access-tagging replay of a kernel is being generated (kernel_trace)
        self.track = None  # check_finite plans: id(source statement) -> checkpoint number (compiled.CompiledPlan)
        self.init_tested: set = set()  # Views whose loaded values a tracked kernel tests (checkpoint 0)
        self.touched_before: set = set()  # Views earlier kernels of the plan touched: their loads are not "as they came in"
        self.has_trace = False
        self.views: list = []  # view table: name -> index
        self.rank: dict = {}
        self.slots: dict = {}  # function-scope scalar -> slot in S
        self.parts: list = []
        self.kernels: dict = {}  # id(stmt) -> recipe
        for p in fn.params:
            if p.is_view:
                self._add_view(p.name, p.type.rank)
            else:
                self.slot(p.name)
        for s in walk_statements(fn.body):
            if kind(s) == "DeclView":
                self._add_view(s.name, s.descriptor.rank)

    def _add_view(self, name, rank):
        if name not in self.rank:
            self.views.append(name)
            self.rank[name] = rank

    def vid(self, name) -> int:
        return self.views.index(name)

    def slot(self, name) -> int:
        if name not in self.slots:
            self.slots[name] = len(self.slots)
        return self.slots[name]

    def hslot(self, name) -> int:
        if name not in self.hslots:
            self.hslots[name] = len(self.hslots)
        return self.hslots[name]

    def _reg(self, acc):
        """Register holding acc's element when its view is promoted in the tile kernel
        being generated (pointwise access by construction)."""
        r = self.promoted.get(acc.view)
        if r is not None:
            if len(acc.indices) == 2:  # rank-2 row at the running index: one register column per literal column
                return f"{r}c{_constant(acc.indices[1])}[e]"
            return f"{r}[e]"
        nb = self.nbr.get(acc.view)
        if nb is not None:
            # neighbour registers (tilegen.tile_kernel): element e + c of the lane's four, or the halo
            # values fetched from the adjacent lanes; only for accesses proven in range on interior steps
            const = _unit_affine(acc.indices[0], self.counter) if len(acc.indices) == 1 else None
            el = self.interior
            if const is not None and el is not None and -const <= el["lo"] and const <= el["up"]:
                if self.elide is not None:
                    self.elide["views"].add(acc.view)  # the host verifies extent >= n before it launches
                return f"KRN_NBR({nb}, e + ({const}))"
            return None
        w = self.windows.get(acc.view)
        if w is not None:
            # every access to a window View is `counter + c`, proven in range when the group was formed
            const = _unit_affine(acc.indices[0], self.counter)
            if const is None or len(acc.indices) != 1:
                raise TypeError(f"window view {acc.view} accessed with a non-affine index")
            if self.elide is not None:
                self.elide["views"].add(acc.view)
            return f"{w}[wq + ({const})]"
        return None

    # ---- expressions -----------------------------------------------------------

    def index(self, e, local) -> str:
        k = kind(e)
        if k == "IntLiteral":
            return f"((krn_i64){e.value}ll)" if e.value >= 0 else f"((krn_i64)({e.value}ll))"
        if k == "Counter":
            return "i"
        if k == "Extent":
            return f"E.e{e.dim}[{self.vid(e.view)}]"
        if k == "ViewAccess":
            line = getattr(e.span, "line", 0)
            return f"to_index(E, {self.load(e, local)}, {line}, {self.vid(e.view)}, bad)"
        if k == "IdxBinary":
            return f"({self.index(e.lhs, local)} {e.op} {self.index(e.rhs, local)})"
        raise TypeError(f"cannot generate index {k}")

    # ---- static bounds-check elision (tile kernels) -------------------------------------
    # `self.elide` = dict(counter, trip, sym, views) while a fused group is generated.  The
    # running index i satisfies L <= i <= n-1-U, refined by the enclosing guards
    # (`i != 0`, `i != extent(x,0) - 1`, `i >= c`, `i < n + k`, ...).  An access v(i + c) is
    # in range for every i if L + c >= 0 and c - U <= 0 PROVIDED extent(v, 0) >= n, which the
    # host verifies before launching (otherwise the call runs on the statement path, with
    # every check in place).
    def _range(self):
        el = self.elide
        return guard_interval(self.guards, el["counter"], el["trip"], el["sym"])

    def _provably_in_range(self, acc) -> bool:
        el = self.elide
        if el is None or len(acc.indices) != 1 or self.rank.get(acc.view) != 1:
            return False
        try:
            const, terms = normalize_index(acc.indices[0])
        except (TypeError, ValueError):
            return False
        if terms != ((("counter", el["counter"]), 1),):
            return False
        lo, up = self._range()
        if lo + const >= 0 and const - up <= 0:
            el["views"].add(acc.view)
            return True
        return False

    def offset(self, acc, local) -> str:
        v = self.vid(acc.view)
        line = getattr(acc.span, "line", 0)
        idx = [self.index(i, local) for i in acc.indices]
        if self._provably_in_range(acc):
            return f"({idx[0]})"
        if len(idx) == 1:
            return f"off1(E, {v}, {idx[0]}, {line}, bad)"
        return f"off2(E, {v}, {idx[0]}, {idx[1]}, {line}, bad)"

    def load(self, acc, local) -> str:
        reg = self._reg(acc)
        if reg is not None:
            return reg
        if self.tracing:
            return f"krn_trace_rd(E, T, i, {self.vid(acc.view)}, {self.offset(acc, local)}, bad)"
        # the offset expression may set `bad`; rd() then yields 0.0 without touching memory
        return f"krn_seq_rd(E, {self.vid(acc.view)}, {self.offset(acc, local)}, bad)"

    def value(self, e, local) -> str:
        k = kind(e)
        if k == "Literal":
            return c_double(e.value)
        if k == "ScalarVar":
            if e.name in local:
                return f"L_{e.name}"
            if e.name in self.host_scalars:
                return f"E.H[{self.hslot(e.name)}]"
            return f"E.S[{self.slot(e.name)}]"
        if k == "IndexVar":
            return "((double)i)"
        if k == "ViewAccess":
            return self.load(e, local)
        if k == "Extent":
            return f"((double)E.e{e.dim}[{self.vid(e.view)}])"
        if k == "Neg":
            return f"(-{self.value(e.operand, local)})"
        if k == "Binary":
            # C++ leaves operand evaluation order unspecified; only `bad` bookkeeping is
            # order-sensitive and it is idempotent, the arithmetic itself is a tree
            return f"({self.value(e.lhs, local)} {e.op} {self.value(e.rhs, local)})"
        raise TypeError(f"cannot generate value {k}")

    def compare(self, c, local) -> str:
        if self.interior is not None:
            # interior warp step (window kernels): every iteration the warp touches lies at least
            # `lo` rows from the start and `up` rows from the end of the range, so guards of the
            # forms the interval analysis understands are known to hold
            el = self.interior
            lo, up = guard_interval([c], el["counter"], el["trip"], el["sym"])
            if (lo or up) and lo <= el["lo"] and up <= el["up"]:
                return "(true)"
        return f"({self.index(c.lhs, local)} {c.op} {self.index(c.rhs, local)})"

    # ---- statements ----------------------------------------------------------------

    def element(self, s, local: set, out: list, pad: str, sites: dict, in_kernel: bool):
        """One element statement; `local` = names living in C++ locals."""
        k = kind(s)
        stop = "continue;" if in_kernel else "return;"
        if k == "DeclScalar":
            if in_kernel:
                local.add(s.name)
                out.append(f"{pad}double L_{s.name} = {self.value(s.init, local)};")
            else:
                out.append(f"{pad}{{ double t_ = {self.value(s.init, local)}; if (bad) {stop} "
                           f"E.S[{self.slot(s.name)}] = t_; }}")
                return
            out.append(f"{pad}if (bad) {stop}")
        elif k == "AssignScalar":
            tgt = f"L_{s.name}" if s.name in local else f"E.S[{self.slot(s.name)}]"
            rhs = self.value(s.rhs, local)
            expr = {"=": "t_", "+=": f"{tgt} + t_", "-=": f"{tgt} - t_"}[s.op]
            out.append(f"{pad}{{ double t_ = {rhs}; if (bad) {stop} {tgt} = {expr}; }}")
        elif k == "AssignView" and self._reg(s.target) is not None:
            reg = self._reg(s.target)
            expr = {"=": "t_", "+=": f"{reg} + t_", "-=": f"{reg} - t_"}[s.op]
            out.append(f"{pad}{{ double t_ = {self.value(s.rhs, local)}; if (bad) {stop} {reg} = {expr}; }}")
        elif k in ("AssignView", "AtomicAdd") and self.tracing:
            # dry replay: same evaluation order as the interpreter (offset, then value, then the
            # record: runtime.py:414-419, 435-440); nothing is stored
            v = self.vid(s.target.view)
            rhs = s.rhs if k == "AssignView" else s.value
            out.append(
                f"{pad}{{ krn_i64 o_ = {self.offset(s.target, local)}; if (bad) {stop} "
                f"double t_ = {self.value(rhs, local)}; (void)t_; if (bad) {stop} "
                f"krn_touch(T, {v}, o_, i, {2 if k == 'AssignView' else 4}u); }}"
            )
        elif k == "AssignView":
            v = self.vid(s.target.view)
            expr = {"=": "t_", "+=": f"E.v[{v}][o_] + t_", "-=": f"E.v[{v}][o_] - t_"}[s.op]
            out.append(
                f"{pad}{{ krn_i64 o_ = {self.offset(s.target, local)}; if (bad) {stop} "
                f"double t_ = {self.value(s.rhs, local)}; if (bad) {stop} E.v[{v}][o_] = {expr}; }}"
            )
        elif k == "AtomicAdd":
            v = self.vid(s.target.view)
            head = (f"{pad}{{ krn_i64 o_ = {self.offset(s.target, local)}; if (bad) {stop} "
                    f"double t_ = {self.value(s.value, local)}; if (bad) {stop} ")
            site = sites.get(id(s)) if sites else None
            if site is not None and site.absorbed:
                return  # its value travels with the preceding site's (merge_adjacent_atomics)
            extra, lane_offsets = [], []
            if site is not None and site.merged:
                for j, m in enumerate(site.merged):
                    if site.lanes:  # another literal column of the same row: its own bounds check
                        head += f"krn_i64 o{j}_ = {self.offset(m.stmt.target, local)}; if (bad) {stop} "
                        lane_offsets.append(f"o{j}_")
                    head += f"double u{j}_ = {self.value(m.stmt.value, local)}; if (bad) {stop} "
                    extra.append(f"u{j}_")
            ordered = None
            if site is not None and site.ord is not None:
                ko, vo, G, W, g = site.ord
                vals = (["t_"] + extra + ["-0.0"] * ORDERED_WIDTH)[:ORDERED_WIDTH]
                key = f"o_ / E.e1[{v}]" if site.lanes else "o_"  # row records: the key is the row
                ordered = f"krn_ord_put(E, {ko}, {vo}, {G}, {W}, {g}, i, {key}, {', '.join(vals)});"
            if site is None:  # function scope: applies immediately (runtime.py:441-442)
                out.append(head + f"E.v[{v}][o_] = E.v[{v}][o_] + t_; }}")
            elif site.mode == "gather" and site.index in self.stage_windows:
                out.append(head + f"{self.stage_windows[site.index]}[wq] = t_; }}")
            elif site.mode == "gather" and (self.promoted or self.in_tile):
                out.append(head + f"T{site.index}[e] = t_; }}")  # tile kernel: staging column in registers
            elif site.mode == "gather":
                out.append(head + f"stage[{site.index} * n + i] = t_; }}")
            elif site.mode == "direct":
                # window kernels re-run statements on halo iterations (slot e == 4): those belong to a
                # neighbouring warp, which performs the update itself
                own = "if (e < 4) " if self.in_tile else ""
                out.append(head + f"{own}E.v[{v}][o_] = E.v[{v}][o_] + t_; }}")
            elif site.mode == "staged_atomic":
                out.append(head + (f"if (E.apol == 4) {{ {ordered} }} else " if ordered else "") +
                           f"{{ stage[{site.index} * n + i] = t_; ostage[{site.index} * n + i] = o_; }} }}")
            else:
                # hardware reductions are exact only up to reassociation, so adjacent sites on one
                # location issue one reduction with the sum of their values; the ordered policy
                # keeps them apart (d + a) + b
                if site.lanes:
                    total = "".join(f" krn_scatter(E, {v}, {o}, {u});" for o, u in zip(lane_offsets, extra))
                    out.append(head + (f"if (E.apol == 4) {{ {ordered} }} else " if ordered else "") +
                               f"{{ krn_scatter(E, {v}, o_, t_);{total} }} }}")
                else:
                    total = "".join(f" t_ = t_ + {u};" for u in extra)
                    out.append(head + (f"if (E.apol == 4) {{ {ordered} }} else " if ordered else "") +
                               f"{{{total} krn_scatter(E, {v}, o_, t_); }} }}")
        elif k == "If":
            out.append(f"{pad}if {self.compare(s.cond, local)} {{")
            self.guards.append(s.cond)
            try:
                for inner in s.body:
                    self.element(inner, local, out, pad + "    ", sites, in_kernel)
            finally:
                self.guards.pop()
            out.append(f"{pad}}}")
        else:
            raise TypeError(f"statement not allowed here: {k}")

    def kernel(self, loop, name: str) -> dict:
        sites = plan_atomics(loop)
        ordered = assign_ordered([sites])
        by_id = {id(st.stmt): st for st in sites}
        staged = [st for st in sites if st.mode in ("gather", "staged_atomic")]
        needs_offsets = any(st.mode == "staged_atomic" for st in sites)
        body: list = []
        local = {loop.counter}
        for s in loop.body:
            self.element(s, local, body, "        ", by_id, True)
        src = [
            f'extern "C" __global__ void __launch_bounds__(256) {name}(Env E, krn_i64 n, double *stage, '
            "krn_i64 *ostage)",
            "{",
            "    krn_priv_begin(E);" if any(st.mode == "atomic" for st in sites) else "",
            "    for (krn_i64 i = blockIdx.x * (krn_i64)blockDim.x + threadIdx.x; i < n; "
            "i += (krn_i64)gridDim.x * blockDim.x) {",
            "        bool bad = false;",
        ]
        if staged:
            # a site that does not execute (guard false) must not contribute: mark with the
            # offsets column when present, else re-evaluate guards in the apply kernel
            for st in staged:
                if st.mode == "staged_atomic":
                    src.append(f"        if (E.apol != 4) ostage[{st.index} * n + i] = -1;")
        src += body + ["    }", "    krn_priv_end(E);" if any(st.mode == "atomic" for st in sites) else "", "}"]
        self.parts.append("\n".join(src))
        recipe = dict(name=name, sites=sites, n_staged=len(sites) if staged else 0,
                      needs_offsets=needs_offsets, apply=[], ordered=ordered,
                      atomic_views=sorted({st.view for st in sites if st.mode == "atomic"}))
        # apply kernels
        gather_views: dict = {}
        for st in sites:
            if st.mode == "gather":
                gather_views.setdefault(st.view, []).append(st)
        for view, group in gather_views.items():
            recipe["apply"].append(self._gather_apply(loop, view, group, f"{name}_g{self.vid(view)}"))
        if needs_offsets:
            recipe["apply"].append(self._staged_apply(sites, f"{name}_a"))
        return recipe

    def kernel_trace(self, loop, name: str) -> dict:
        """Dry, access-tagging replay of `loop` for the conflict detector (see _TRACE)."""
        body: list = []
        local = {loop.counter}
        self.tracing, self.has_trace = True, True
        try:
            for s in loop.body:
                self.element(s, local, body, "        ", None, True)
        finally:
            self.tracing = False
        src = [
            f'extern "C" __global__ void __launch_bounds__(256) {name}(Env E, krn_i64 n, Trace T)',
            "{",
            "    for (krn_i64 i = blockIdx.x * (krn_i64)blockDim.x + threadIdx.x; i < n; "
            "i += (krn_i64)gridDim.x * blockDim.x) {",
            "        bool bad = false;",
        ] + body + ["    }", "}"]
        self.parts.append("\n".join(src))
        touched = set()
        for s in walk_statements(loop.body):
            k = kind(s)
            exprs = []
            if k in ("AssignView", "AtomicAdd"):
                touched.add(s.target.view)
                exprs = list(s.target.indices) + [s.rhs if k == "AssignView" else s.value]
            elif k == "DeclScalar":
                exprs = [s.init]
            elif k == "AssignScalar":
                exprs = [s.rhs]
            elif k == "If":
                exprs = [s.cond.lhs, s.cond.rhs]
            for e in exprs:
                for node in walk_expr(e):
                    if kind(node) == "ViewAccess":
                        touched.add(node.view)
        return dict(name=name, views=sorted(touched))

    def _gather_apply(self, loop, view, group, name) -> dict:
        """Kernel over the rows k of `view`: adds, in (iteration, program order),
        the staged contributions whose target is row k."""
        v = self.vid(view)
        rank2 = self.rank[view] == 2
        # iteration of site s for row k is k - c_s: ascending iteration = descending c_s
        order = sorted(group, key=lambda st: (-st.offset, st.index))
        lines = [
            f'extern "C" __global__ void __launch_bounds__(256) {name}(Env E, krn_i64 n, '
            "const double *stage, const krn_i64 *ostage)",
            "{",
            f"    const krn_i64 rows = E.e0[{v}];",
            "    for (krn_i64 k = blockIdx.x * (krn_i64)blockDim.x + threadIdx.x; k < rows; "
            "k += (krn_i64)gridDim.x * blockDim.x) {",
        ]
        columns = sorted({st.column for st in group}) if rank2 else [None]
        for col in columns:
            if rank2:
                lines.append(f"        if ({col} >= 0 && {col} < E.e1[{v}]) {{")
                lines.append(f"            double acc = E.v[{v}][k * E.e1[{v}] + {col}];")
            else:
                lines.append("        {")
                lines.append(f"            double acc = E.v[{v}][k];")
            for st in order:
                if rank2 and st.column != col:
                    continue
                guard = " && ".join(
                    ["i >= 0", "i < n"] + [self.compare(g, {loop.counter}) for g in st.guards]
                )
                lines.append(f"            {{ const krn_i64 i = k - ({st.offset}); bool bad = false; (void)bad; "
                             f"if ({guard}) acc = acc + stage[{st.index} * n + i]; }}")
            if rank2:
                lines.append(f"            E.v[{v}][k * E.e1[{v}] + {col}] = acc;")
            else:
                lines.append(f"            E.v[{v}][k] = acc;")
            lines.append("        }")
        lines += ["    }", "}"]
        self.parts.append("\n".join(lines))
        return dict(name=name, over="rows", view=view)

    def _staged_apply(self, sites, name) -> dict:
        lines = [
            f'extern "C" __global__ void __launch_bounds__(256) {name}(Env E, krn_i64 n, '
            "const double *stage, const krn_i64 *ostage)",
            "{",
            "    for (krn_i64 i = blockIdx.x * (krn_i64)blockDim.x + threadIdx.x; i < n; "
            "i += (krn_i64)gridDim.x * blockDim.x) {",
        ]
        for st in sites:
            if st.mode == "staged_atomic":
                v = self.vid(st.view)
                lines.append(f"        {{ krn_i64 o = ostage[{st.index} * n + i]; "
                             f"if (o >= 0) krn_red_add(&E.v[{v}][o], stage[{st.index} * n + i]); }}")
        lines += ["    }", "}"]
        self.parts.append("\n".join(lines))
        return dict(name=name, over="iterations", view=None)

    def scalar_block(self, stmts, name: str) -> dict:
        """One-thread kernel for a run of function-scope element statements."""
        body: list = []
        for s in stmts:
            self.element(s, set(), body, "    ", None, False)
        src = [f'extern "C" __global__ void {name}(Env E)', "{", "    bool bad = false;"] + body + ["}"]
        self.parts.append("\n".join(src))
        return dict(name=name)

    def return_block(self, expr, name: str) -> dict:
        slot = self.slot("__return__")
        src = [
            f'extern "C" __global__ void {name}(Env E)',
            "{",
            "    bool bad = false;",
            f"    double t_ = {self.value(expr, set())};",
            f"    if (!bad) E.S[{slot}] = t_;",
            "}",
        ]
        self.parts.append("\n".join(src))
        return dict(name=name, slot=slot)

    def source(self) -> str:
        head = _PREAMBLE % dict(nv=len(self.views), nh=len(self.hslots))
        if self.has_trace:
            head += _TRACE
        head += (
            "__device__ __forceinline__ double krn_seq_rd(const Env &E, int v, krn_i64 off, bool &bad)\n"
            "{ return rd(E, v, off, bad); }\n"
        )
        return head + "\n\n" + "\n\n".join(self.parts) + "\n"
