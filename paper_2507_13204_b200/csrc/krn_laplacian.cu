// Fused kernels for the headline objective normRes1DLaplacianSQ and its
// generated gradient: one launch each, every compulsory byte moved once.
//
//   primal   reads x, b (16 B/row), writes 3x (8 B/row)                = 24 B/row
//   gradient reads x, b [, _d_x, _d_b], writes 3x, _d_x, _d_b   = 40 or 56 B/row
//
// What is computed is the execution of the reference's statement sequence
// (forward: programs/laplacian.krn:4-21; reverse: the emitted text frozen in
// reference tests/test_adjoint.py:43-94) with the same IEEE operations in the
// same order per output element:
//
//   xs_j  = 3.0 * x_j
//   y_j   = ((2.0*xs_j - b_j) - [j!=0] xs_{j-1}) - [j!=n-1] xs_{j+1}
//   f     = tree_j(y_j * y_j)                      (reference pairwise tree)
//   r4    = 0.0 + (0.0 + seed)                     (_d_sum, then _d_y2 broadcast)
//   dy_j  = (0.0 + r4*y_j) + y_j*r4
//   [j!=n-1]  r3 = dy; dy = (dy - r3) + r3         -> -r3 to _d_x(j+1)
//   [j!=0]    r2 = dy; dy = (dy - r2) + r2         -> -r2 to _d_x(j-1)
//   r1 = dy                                        -> 2.0*r1 to _d_x(j), -r1 to _d_b(j)
//
// The reference queues the three _d_x contributions as atomic adds and applies
// them after the kernel sorted by (iteration, program order)
// (runtime.py:615-620).  Location k therefore receives, in this order,
// -r3_{k-1}, 2.0*r1_k, -r2_{k+1}.  Here every thread *gathers* those three
// terms for its own k in exactly that order: no atomics, no conflicts, and the
// result is bit-identical to the interpreter.  The reverse of the scale kernel
// is folded in: r0 = acc; _d_x_k = (acc - r0) + 3.0*r0.
//
// Work decomposition: a block owns an aligned chunk of 1024*R rows, warp w the
// aligned sub-chunk of 128*R rows, processed as R steps of 128 rows (4 per lane,
// one LDG.E.256 per operand); R = 1 for the gradient, 1 or 4 for the primal (steps_for).  Neighbour values travel by warp shuffle; the two
// edge lanes fetch the ghost rows of the neighbouring warp themselves (L2 hits).
// Interior steps need no guard at all; the (at most three) steps per shard that
// touch row 0, row n-1, a shard boundary or the ragged tail take a scalar,
// fully guarded path.
#include "krn_common.cuh"
#include "krn_prelude.cuh"

#include <cstdlib>

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kStep = 128;  // rows per warp step

struct Shard {
    const double *x;     // original x, local rows
    const double *b;
    const double *halo;  // x[-2], x[-1], b[-1], x[n], x[n+1], b[n] (local indexing) or null
    // neighbour shards addressed directly (their own buffers, mapped into this process: peer memory
    // over NVLink, or the same device): xp[-1] / bp[-1] is the previous shard's last row, xn[0] / bn[0]
    // the next shard's first row.  Null: the halo array is used instead.
    const double *xp, *bp, *xn, *bn;
    krn_i64 n_local;
    krn_i64 offset;
    krn_i64 n_global;
};

// original x / b at local row i in [-2, n_local + 2); caller guarantees the global row exists
__device__ __forceinline__ double x_at(const Shard &s, krn_i64 i)
{
    if (i < 0) return s.xp ? s.xp[i] : s.halo[2 + i];
    if (i >= s.n_local) return s.xn ? s.xn[i - s.n_local] : s.halo[3 + (i - s.n_local)];
    return krn_ld1(s.x + i);
}
__device__ __forceinline__ double b_at(const Shard &s, krn_i64 i)
{
    if (i < 0) return s.bp ? s.bp[i] : s.halo[2];
    if (i >= s.n_local) return s.bn ? s.bn[i - s.n_local] : s.halo[5];
    return krn_ld1(s.b + i);
}

struct Chain {
    double r3, r2, r1;
};

// reverse of the stencil kernel for one row, statement by statement
__device__ __forceinline__ Chain adjoint_chain(double y, double r4, bool has_up, bool has_down)
{
    Chain c;
    double dy = 0.0 + r4 * y;   // _d_y(j) += _r_d4 * y(j)   (shadow starts at +0.0)
    dy = dy + y * r4;           // _d_y(j) += y(j) * _r_d4
    c.r3 = 0.0;
    c.r2 = 0.0;
    if (has_up) {               // if (j != extent - 1)
        c.r3 = dy;
        dy = dy - c.r3;
        dy = dy + c.r3;
    }
    if (has_down) {             // if (j != 0)
        c.r2 = dy;
        dy = dy - c.r2;
        dy = dy + c.r2;
    }
    c.r1 = dy;
    return c;
}

__device__ __forceinline__ double stencil_row(double xm, double xc, double xp, double b, bool has_down,
                                              bool has_up)
{
    double y = 2.0 * xc - b;
    if (has_down) y = y - xm;
    if (has_up) y = y - xp;
    return y;
}

// _d_x(k): gather of the queued contributions in the reference's order, then the
// reverse of the scale kernel
__device__ __forceinline__ double finish_dx(double dx_in, double r3_left, double r1, double r2_right,
                                            bool has_left, bool has_right)
{
    double acc = dx_in;
    if (has_left) acc = acc + (-r3_left);
    acc = acc + 2.0 * r1;
    if (has_right) acc = acc + (-r2_right);
    double r0 = acc;
    acc = acc - r0;
    acc = acc + 3.0 * r0;
    return acc;
}

// ---- guarded scalar path: any step, any boundary --------------------------------
template <bool GRAD>
__device__ __forceinline__ double edge_step(const Shard &s, krn_i64 base, int lane, double *x_out,
                                            double *dx, double *db, bool dx_zero, bool db_zero,
                                            double r4)
{
    double node[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
        krn_i64 i = base + 4 * lane + e;
        krn_i64 g = s.offset + i;
        if (i >= s.n_local) {
            // beyond the shard: tree padding if also beyond the problem, identity otherwise
            node[e] = (g >= s.n_global) ? krn_tree_pad((krn_u64)g, (krn_u64)s.n_global) : -0.0;
            continue;
        }
        const krn_i64 last = s.n_global - 1;
        // scaled rows g-2 .. g+2 where they exist
        double xs[5];
#pragma unroll
        for (int d = -2; d <= 2; ++d) {
            krn_i64 gg = g + d;
            bool need = GRAD || (d >= -1 && d <= 1);
            xs[d + 2] = (need && gg >= 0 && gg <= last) ? 3.0 * x_at(s, i + d) : 0.0;
        }
        double y = stencil_row(xs[1], xs[2], xs[3], b_at(s, i), g != 0, g != last);
        x_out[i] = xs[2];
        if (!GRAD) {
            node[e] = y * y;
            continue;
        }
        node[e] = -0.0;
        Chain own = adjoint_chain(y, r4, g != last, g != 0);
        double r3_left = 0.0, r2_right = 0.0;
        if (g != 0) {  // row g-1 exists: its "j+1" contribution lands here
            double yl = stencil_row(xs[0], xs[1], xs[2], b_at(s, i - 1), g - 1 != 0, true);
            r3_left = adjoint_chain(yl, r4, true, g - 1 != 0).r3;
        }
        if (g != last) {  // row g+1 exists: its "j-1" contribution lands here
            double yr = stencil_row(xs[2], xs[3], xs[4], b_at(s, i + 1), true, g + 1 != last);
            r2_right = adjoint_chain(yr, r4, g + 1 != last, true).r2;
        }
        if (dx != nullptr) {
            double in = dx_zero ? 0.0 : dx[i];
            dx[i] = finish_dx(in, r3_left, own.r1, r2_right, g != 0, g != last);
        }
        if (db != nullptr) {
            double in = db_zero ? 0.0 : db[i];
            db[i] = in + (-own.r1);
        }
    }
    return (node[0] + node[1]) + (node[2] + node[3]);
}

// ---- interior path: 128 full rows, ghosts inside the shard, no guards -----------------
// Split into a load half and a compute half so the kernel can issue the loads of
// step t+1 before it computes step t (two steps of every operand in flight per warp).
struct StepData {
    krn_d4 x, b, dx, db;
    double g_near, g_far, g_b;  // ghost rows of the neighbouring warp step (edge lanes only)
};

template <bool GRAD, bool HAS_DX, bool HAS_DB, bool DX_ZERO, bool DB_ZERO>
__device__ __forceinline__ StepData load_interior(const double *__restrict__ x, const double *__restrict__ b,
                                                  const double *dx, const double *db, krn_i64 base, int lane)
{
    StepData d;
    const krn_i64 i0 = base + 4 * lane;
    d.x = krn_ld4_stream(x + i0);
    d.b = krn_ld4_stream(b + i0);
    d.dx = {0.0, 0.0, 0.0, 0.0};
    d.db = {0.0, 0.0, 0.0, 0.0};
    if (GRAD && HAS_DX && !DX_ZERO) d.dx = krn_ld4_rmw(dx + i0);
    if (GRAD && HAS_DB && !DB_ZERO) d.db = krn_ld4_rmw(db + i0);
    d.g_near = d.g_far = d.g_b = 0.0;
    if (lane == 0) {
        d.g_near = krn_ld1(x + i0 - 1);
        if (GRAD && HAS_DX) {
            d.g_far = krn_ld1(x + i0 - 2);
            d.g_b = krn_ld1(b + i0 - 1);
        }
    } else if (lane == 31) {
        d.g_near = krn_ld1(x + i0 + 4);
        if (GRAD && HAS_DX) {
            d.g_far = krn_ld1(x + i0 + 5);
            d.g_b = krn_ld1(b + i0 + 4);
        }
    }
    return d;
}

template <bool GRAD, bool HAS_DX, bool HAS_DB>
__device__ __forceinline__ double compute_interior(const StepData &d, krn_i64 base, int lane,
                                                   double *__restrict__ x_out, double *dx, double *db,
                                                   double r4)
{
    const krn_i64 i0 = base + 4 * lane;
    const bool left_edge = lane == 0, right_edge = lane == 31;
    krn_d4 xs = {3.0 * d.x.a, 3.0 * d.x.b, 3.0 * d.x.c, 3.0 * d.x.d};
    krn_st4(x_out + i0, xs);

    double xl = __shfl_up_sync(KRN_FULL_MASK, xs.d, 1);
    double xr = __shfl_down_sync(KRN_FULL_MASK, xs.a, 1);
    const double g_near_s = 3.0 * d.g_near;
    if (left_edge) xl = g_near_s;
    if (right_edge) xr = g_near_s;

    double y0 = stencil_row(xl, xs.a, xs.b, d.b.a, true, true);
    double y1 = stencil_row(xs.a, xs.b, xs.c, d.b.b, true, true);
    double y2 = stencil_row(xs.b, xs.c, xs.d, d.b.c, true, true);
    double y3 = stencil_row(xs.c, xs.d, xr, d.b.d, true, true);

    if (!GRAD) return (y0 * y0 + y1 * y1) + (y2 * y2 + y3 * y3);

    Chain c0 = adjoint_chain(y0, r4, true, true);
    Chain c1 = adjoint_chain(y1, r4, true, true);
    Chain c2 = adjoint_chain(y2, r4, true, true);
    Chain c3 = adjoint_chain(y3, r4, true, true);

    if (HAS_DX) {
        // r3 of the row left of this lane, r2 of the row right of it
        double r3_left = __shfl_up_sync(KRN_FULL_MASK, c3.r3, 1);
        double r2_right = __shfl_down_sync(KRN_FULL_MASK, c0.r2, 1);
        if (left_edge || right_edge) {
            const double g_far_s = 3.0 * d.g_far;
            double ym = left_edge ? g_far_s : xs.d;
            double yp = left_edge ? xs.a : g_far_s;
            Chain g = adjoint_chain(stencil_row(ym, g_near_s, yp, d.g_b, true, true), r4, true, true);
            if (left_edge) r3_left = g.r3;
            if (right_edge) r2_right = g.r2;
        }
        krn_d4 o;
        o.a = finish_dx(d.dx.a, r3_left, c0.r1, c1.r2, true, true);
        o.b = finish_dx(d.dx.b, c0.r3, c1.r1, c2.r2, true, true);
        o.c = finish_dx(d.dx.c, c1.r3, c2.r1, c3.r2, true, true);
        o.d = finish_dx(d.dx.d, c2.r3, c3.r1, r2_right, true, true);
        krn_st4(dx + i0, o);
    }
    if (HAS_DB) {
        krn_d4 o = {d.db.a + (-c0.r1), d.db.b + (-c1.r1), d.db.c + (-c2.r1), d.db.d + (-c3.r1)};
        krn_st4(db + i0, o);
    }
    return -0.0;
}

// complete in-order tree over STEPS (power of two) nodes
template <int STEPS>
__device__ __forceinline__ double static_tree(double (&v)[STEPS])
{
#pragma unroll
    for (int w = 1; w < STEPS; w <<= 1) {
#pragma unroll
        for (int i = 0; i < STEPS; i += 2 * w) v[i] = v[i] + v[i + w];
    }
    return v[0];
}

template <bool GRAD, bool HAS_DX, bool HAS_DB, bool DX_ZERO, bool DB_ZERO, int STEPS>
__global__ void __launch_bounds__(kThreads, 4)  // <= 64 registers: 4 blocks (32 warps) per SM
laplacian_kernel(Shard s, double *__restrict__ x_out, double *dx, double *db, double seed, bool vector_ok,
                 double *partials, double *scratch, unsigned int *ticket, double *f_out, int accumulate)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr krn_i64 chunk = (krn_i64)kThreads * 4 * STEPS;
    const krn_i64 warp_base = (krn_i64)blockIdx.x * chunk + (krn_i64)warp * kStep * STEPS;
    const double d_sum = 0.0 + seed;   // let _d_sum = 0.0;  _d_sum += seed;
    const double r4 = 0.0 + d_sum;     // parallel_sum(_d_y2, _d_sum) on a zero shadow

    auto interior = [&](krn_i64 base) { return vector_ok && base >= 2 && base + kStep + 2 <= s.n_local; };

    // one step of the warp's sub-chunk that is not a plain interior step
    auto other_step = [&](krn_i64 base) -> double {
        if (base >= s.n_local) {
            // nothing of this step lies in the shard; it still owns a node of the tree
            double node = -0.0;
            if (!GRAD) {
                double v[4];
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    krn_i64 g = s.offset + base + 4 * lane + e;
                    v[e] = g >= s.n_global ? krn_tree_pad((krn_u64)g, (krn_u64)s.n_global) : -0.0;
                }
                node = (v[0] + v[1]) + (v[2] + v[3]);
            }
            return node;
        }
        return edge_step<GRAD>(s, base, lane, x_out, HAS_DX ? dx : nullptr, HAS_DB ? db : nullptr, DX_ZERO,
                               DB_ZERO, r4);
    };

    double nodes[STEPS];
    if constexpr (GRAD) {
        // four operand streams per step already keep 4 KB per warp in flight at 4 blocks/SM;
        // a deeper software pipeline only costs occupancy here (measured: -1.5%)
#pragma unroll 1
        for (int t = 0; t < STEPS; ++t) {
            const krn_i64 base = warp_base + (krn_i64)t * kStep;
            if (interior(base)) {
                StepData d = load_interior<GRAD, HAS_DX, HAS_DB, DX_ZERO, DB_ZERO>(s.x, s.b, dx, db, base, lane);
                compute_interior<GRAD, HAS_DX, HAS_DB>(d, base, lane, x_out, dx, db, r4);
            } else {
                other_step(base);
            }
        }
        return;
    } else {
        // primal: two operand streams only, so the loads of step t+1 are issued before step t
        // is computed (measured: +7% bandwidth)
        StepData cur;
        bool cur_ok = interior(warp_base);
        if (cur_ok)
            cur = load_interior<GRAD, HAS_DX, HAS_DB, DX_ZERO, DB_ZERO>(s.x, s.b, dx, db, warp_base, lane);
#pragma unroll
        for (int t = 0; t < STEPS; ++t) {
            const krn_i64 base = warp_base + (krn_i64)t * kStep;
            StepData nxt;
            bool nxt_ok = false;
            if (t + 1 < STEPS) {
                nxt_ok = interior(base + kStep);
                if (nxt_ok)
                    nxt = load_interior<GRAD, HAS_DX, HAS_DB, DX_ZERO, DB_ZERO>(s.x, s.b, dx, db, base + kStep,
                                                                                lane);
            }
            double node = cur_ok ? compute_interior<GRAD, HAS_DX, HAS_DB>(cur, base, lane, x_out, dx, db, r4)
                                 : other_step(base);
            nodes[t] = krn_warp_tree(node);
            if (t + 1 < STEPS) {
                cur = nxt;
                cur_ok = nxt_ok;
            }
        }
    }

    __shared__ double s_warp[kWarps];
    const double warp_total = static_tree<STEPS>(nodes);
    if (lane == 0) s_warp[warp] = warp_total;
    __syncthreads();
    if (warp == 0) {
        double v = krn_smem_tree(s_warp, kWarps, lane);
        if (lane == 0) partials[blockIdx.x] = v;
    }
    if (krn_last_block(ticket, gridDim.x)) {
        double root = krn_final_tree(partials, scratch, gridDim.x);
        if (threadIdx.x == 0) *f_out = (accumulate ? *f_out : 0.0) + root;
    }
}

int steps_for(size_t n_global, bool grad)
{
    // Measured on B200 (tools/microbench.py, 125 M rows, device time):
    //   steps per warp      1        2        4        8       16
    //   gradient (56 B)  1.010    1.034    1.061    1.107    1.101 ms
    //   primal           0.609    0.482    0.460    0.484    0.512 ms
    // The gradient has no block epilogue, so the finest decomposition wins (most blocks in flight,
    // the whole device sweeps memory front to back): 6.93 TB/s.  The primal pays a block-level tree,
    // a ticket and a partial per block: 4 steps balance that against the sweep (6.52 TB/s); small
    // problems are latency bound and spread over as many blocks as possible.
    if (grad) return 1;
    if (const char *e = getenv("KRN_LAP_STEPS")) return atoi(e);  // experiments (tools/sweep_mid.py)
    // mid sizes, measured (tools/sweep_mid.py, device time incl. ~6 us of launch + event cost, L2 flushed):
    //   rows      0.5 M   0.7 M    1 M     2 M     3 M     10 M
    //   1 step    11.4    12.5    14.3    19.5    26.6    61.5 us
    //   2 steps   12.3    12.4    13.2    18.4    23.5    52.2
    //   4 steps   12.3    13.2    14.3    16.4    22.6    49.3
    if (n_global < 768 * 1024) return 1;
    if (n_global < 1536 * 1024) return 2;
    return 4;
}

template <bool GRAD, int STEPS>
void dispatch(krn_ctx *ctx, dim3 grid, const Shard &s, double *x_out, double *dx, double *db, int dx_zero,
              int db_zero, double seed, bool vec, double *f, int accumulate)
{
    double *partials = ctx->d_partials, *scratch = ctx->d_partials + ctx->partial_capacity;
    dim3 block(kThreads);
#define KRN_LAP(G, HX, HB, ZX, ZB)                                                       \
    laplacian_kernel<G, HX, HB, ZX, ZB, STEPS><<<grid, block, 0, ctx->stream>>>(         \
        s, x_out, dx, db, seed, vec, partials, scratch, ctx->d_ticket, f, accumulate)
    if (!GRAD) {
        KRN_LAP(false, false, false, false, false);
    } else {
        const bool hx = dx != nullptr, hb = db != nullptr, zx = hx && dx_zero, zb = hb && db_zero;
        if (hx && hb) {
            if (zx && zb) KRN_LAP(true, true, true, true, true);
            else if (zx) KRN_LAP(true, true, true, true, false);
            else if (zb) KRN_LAP(true, true, true, false, true);
            else KRN_LAP(true, true, true, false, false);
        } else if (hx) {
            if (zx) KRN_LAP(true, true, false, true, false);
            else KRN_LAP(true, true, false, false, false);
        } else if (hb) {
            if (zb) KRN_LAP(true, false, true, false, true);
            else KRN_LAP(true, false, true, false, false);
        } else {
            KRN_LAP(true, false, false, false, false);
        }
    }
#undef KRN_LAP
}

template <bool GRAD>
int launch(krn_ctx *ctx, const double *x_in, double *x_out, const double *b, double *dx, double *db,
           int dx_zero, int db_zero, size_t n_local, size_t offset, size_t n_global, const double *halo,
           double seed, double *f, int accumulate, const double *xp = nullptr, const double *bp = nullptr,
           const double *xn = nullptr, const double *bn = nullptr)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    KRN_REQUIRE(x_in && x_out && b, "null view pointer");
    KRN_REQUIRE(x_in != x_out, "x_out must not alias x_in");
    KRN_REQUIRE(offset + n_local <= n_global, "shard exceeds the problem");
    KRN_REQUIRE(halo != nullptr || ((offset == 0 || (xp && bp)) && (offset + n_local == n_global || (xn && bn))),
                "a shard that is not the whole problem needs halo rows or its neighbours' buffers");
    KRN_REQUIRE(n_global < (size_t(1) << 62), "problem too large");
    if (!GRAD) KRN_REQUIRE(f != nullptr, "null result pointer");
    if (n_local == 0) {
        if (!GRAD && !accumulate) KRN_CUDA(cudaMemsetAsync(f, 0, sizeof(double), ctx->stream));
        return KRN_OK;
    }
    const int steps = steps_for(n_global, GRAD);
    const size_t chunk = size_t(kThreads) * 4 * steps;
    const size_t blocks = (n_local + chunk - 1) / chunk;
    KRN_REQUIRE(blocks <= 0x7fffffffu, "too many blocks");
    if (!GRAD) {
        int rc = krn_reserve_partials(ctx, blocks);
        if (rc) return rc;
    }
    Shard s{x_in, b, halo, xp, bp, xn, bn, (krn_i64)n_local, (krn_i64)offset, (krn_i64)n_global};
    bool vec = krn_aligned32(x_in) && krn_aligned32(x_out) && krn_aligned32(b) &&
               (dx == nullptr || krn_aligned32(dx)) && (db == nullptr || krn_aligned32(db));
    dim3 grid((unsigned)blocks);
    if (steps == 1)
        dispatch<GRAD, 1>(ctx, grid, s, x_out, dx, db, dx_zero, db_zero, seed, vec, f, accumulate);
    else if (steps == 2)
        dispatch<GRAD, 2>(ctx, grid, s, x_out, dx, db, dx_zero, db_zero, seed, vec, f, accumulate);
    else if (steps == 8)
        dispatch<GRAD, 8>(ctx, grid, s, x_out, dx, db, dx_zero, db_zero, seed, vec, f, accumulate);
    else
        dispatch<GRAD, 4>(ctx, grid, s, x_out, dx, db, dx_zero, db_zero, seed, vec, f, accumulate);
    KRN_LAUNCH_CHECK(ctx);
    return KRN_OK;
}

}  // namespace

extern "C" size_t krn_laplacian_partial_span(size_t n_global)
{
    return size_t(kThreads) * 4 * steps_for(n_global, false);
}

extern "C" int krn_laplacian_primal(krn_ctx *ctx, const double *d_x_in, double *d_x_out,
                                    const double *d_b, size_t n_local, size_t offset, size_t n_global,
                                    const double *d_halo, double *d_f, int accumulate)
{
    return launch<false>(ctx, d_x_in, d_x_out, d_b, nullptr, nullptr, 0, 0, n_local, offset, n_global,
                         d_halo, 1.0, d_f, accumulate);
}

extern "C" int krn_laplacian_grad(krn_ctx *ctx, const double *d_x_in, double *d_x_out, const double *d_b,
                                  double *d_dx, double *d_db, int dx_zero, int db_zero, size_t n_local,
                                  size_t offset, size_t n_global, const double *d_halo, double seed)
{
    return launch<true>(ctx, d_x_in, d_x_out, d_b, d_dx, d_db, dx_zero, db_zero, n_local, offset,
                        n_global, d_halo, seed, nullptr, 0);
}

extern "C" int krn_laplacian_primal_peers(krn_ctx *ctx, const double *d_x_in, double *d_x_out, const double *d_b,
                                          size_t n_local, size_t offset, size_t n_global,
                                          const double *d_x_prev_end, const double *d_b_prev_end,
                                          const double *d_x_next, const double *d_b_next, double *d_f,
                                          int accumulate)
{
    return launch<false>(ctx, d_x_in, d_x_out, d_b, nullptr, nullptr, 0, 0, n_local, offset, n_global, nullptr,
                         1.0, d_f, accumulate, d_x_prev_end, d_b_prev_end, d_x_next, d_b_next);
}

extern "C" int krn_laplacian_grad_peers(krn_ctx *ctx, const double *d_x_in, double *d_x_out, const double *d_b,
                                        double *d_dx, double *d_db, int dx_zero, int db_zero, size_t n_local,
                                        size_t offset, size_t n_global, const double *d_x_prev_end,
                                        const double *d_b_prev_end, const double *d_x_next,
                                        const double *d_b_next, double seed)
{
    return launch<true>(ctx, d_x_in, d_x_out, d_b, d_dx, d_db, dx_zero, db_zero, n_local, offset, n_global,
                        nullptr, seed, nullptr, 0, d_x_prev_end, d_b_prev_end, d_x_next, d_b_next);
}

extern "C" int krn_laplacian_partials(krn_ctx *ctx, double *d_out, size_t count)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    KRN_REQUIRE(count <= ctx->partial_capacity, "more partials requested than the last launch produced");
    if (count == 0) return KRN_OK;
    KRN_REQUIRE(d_out != nullptr, "null output pointer");
    KRN_CUDA(cudaMemcpyAsync(d_out, ctx->d_partials, count * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    return KRN_OK;
}
