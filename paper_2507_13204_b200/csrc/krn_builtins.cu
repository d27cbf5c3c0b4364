// Bulk builtins: fill, copy, view += scalar, view += view, the reference's
// pairwise-tree gather, and the finiteness probe.  All HBM-bound streaming
// kernels: 256-bit accesses, grids sized as a multiple of the SM count.
#include "krn_common.cuh"
#include "krn_prelude.cuh"

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kStep = 128;

inline unsigned stream_grid(const krn_ctx *ctx, size_t n)
{
    size_t want = (n / 4 + kThreads - 1) / kThreads;
    size_t cap = size_t(ctx->sms) * 16;  // 16 resident blocks of 256 threads would overfill an SM: 8 do; two waves
    if (want == 0) want = 1;
    return unsigned(want < cap ? want : cap);
}

enum class Op { Fill, AddScalar, AddView };

template <Op OP, bool VEC>
__global__ void __launch_bounds__(kThreads)
stream_kernel(double *__restrict__ dst, const double *__restrict__ src, size_t n, double s,
              const double *__restrict__ s_dev)
{
    if (s_dev != nullptr) s = *s_dev;
    const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthreads = size_t(gridDim.x) * blockDim.x;
    const size_t nvec = VEC ? n / 4 : 0;
    for (size_t q = tid; VEC && q < nvec; q += nthreads) {
        double *p = dst + 4 * q;
        krn_d4 o;
        if (OP == Op::Fill) {
            o = {s, s, s, s};
        } else if (OP == Op::AddScalar) {
            krn_d4 v = krn_ld4_rmw(p);
            o = {v.a + s, v.b + s, v.c + s, v.d + s};
        } else {
            krn_d4 v = krn_ld4_rmw(p);
            krn_d4 w = krn_ld4_stream(src + 4 * q);
            o = {v.a + w.a, v.b + w.b, v.c + w.c, v.d + w.d};
        }
        krn_st4(p, o);
    }
    for (size_t i = 4 * nvec + tid; i < n; i += nthreads) {
        if (OP == Op::Fill) dst[i] = s;
        else if (OP == Op::AddScalar) dst[i] = dst[i] + s;
        else dst[i] = dst[i] + src[i];
    }
}

template <Op OP>
int launch_stream(krn_ctx *ctx, double *dst, const double *src, size_t n, double s, const double *s_dev)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (n == 0) return KRN_OK;
    KRN_REQUIRE(dst != nullptr, "null view pointer");
    bool vec = krn_aligned32(dst) && (src == nullptr || krn_aligned32(src));
    unsigned grid = stream_grid(ctx, n);
    if (vec) stream_kernel<OP, true><<<grid, kThreads, 0, ctx->stream>>>(dst, src, n, s, s_dev);
    else stream_kernel<OP, false><<<grid, kThreads, 0, ctx->stream>>>(dst, src, n, s, s_dev);
    KRN_LAUNCH_CHECK(ctx);
    return KRN_OK;
}

// ---- pairwise-tree gather --------------------------------------------------------
// Same decomposition as the fused objective kernel: block = aligned chunk of
// 1024*steps leaves, warp = aligned sub-chunk, lane = 4 consecutive leaves.
template <bool VEC, int STEPS>
__global__ void __launch_bounds__(kThreads)
tree_kernel(const double *__restrict__ v, krn_u64 n, double *partials, double *scratch,
            unsigned int *ticket, double *out, int accumulate)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr krn_u64 chunk = krn_u64(kThreads) * 4 * STEPS;
    const krn_u64 warp_base = krn_u64(blockIdx.x) * chunk + krn_u64(warp) * kStep * STEPS;
    // all loads of the warp's sub-chunk are issued before the first add
    krn_d4 q[STEPS];
#pragma unroll
    for (int t = 0; t < STEPS; ++t) {
        const krn_u64 j0 = warp_base + krn_u64(t) * kStep + 4 * lane;
        if (VEC && j0 + 4 <= n) {
            q[t] = krn_ld4_stream(v + j0);
        } else {
            q[t].a = j0 + 0 < n ? krn_ld1(v + j0 + 0) : krn_tree_pad(j0 + 0, n);
            q[t].b = j0 + 1 < n ? krn_ld1(v + j0 + 1) : krn_tree_pad(j0 + 1, n);
            q[t].c = j0 + 2 < n ? krn_ld1(v + j0 + 2) : krn_tree_pad(j0 + 2, n);
            q[t].d = j0 + 3 < n ? krn_ld1(v + j0 + 3) : krn_tree_pad(j0 + 3, n);
        }
    }
    double nodes[STEPS];
#pragma unroll
    for (int t = 0; t < STEPS; ++t) nodes[t] = krn_warp_tree((q[t].a + q[t].b) + (q[t].c + q[t].d));
#pragma unroll
    for (int w = 1; w < STEPS; w <<= 1) {
#pragma unroll
        for (int i = 0; i < STEPS; i += 2 * w) nodes[i] = nodes[i] + nodes[i + w];
    }
    __shared__ double s_warp[kWarps];
    if (lane == 0) s_warp[warp] = nodes[0];
    __syncthreads();
    if (warp == 0) {
        double r = krn_smem_tree(s_warp, kWarps, lane);
        if (lane == 0) partials[blockIdx.x] = r;
    }
    if (krn_last_block(ticket, gridDim.x)) {
        double root = krn_final_tree(partials, scratch, gridDim.x);
        if (threadIdx.x == 0) *out = (accumulate ? *out : 0.0) + root;
    }
}

__global__ void scalar_accumulate_zero(double *out, int accumulate)
{
    // gather over an empty view: total = 0.0
    *out = (accumulate ? *out : 0.0) + 0.0;
}

__global__ void __launch_bounds__(kThreads) finite_kernel(const double *__restrict__ v, size_t n, int *flag)
{
    const size_t tid = size_t(blockIdx.x) * blockDim.x + threadIdx.x;
    const size_t nthreads = size_t(gridDim.x) * blockDim.x;
    bool bad = false;
    for (size_t i = tid; i < n; i += nthreads) bad |= !isfinite(v[i]);
    if (__any_sync(KRN_FULL_MASK, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

}  // namespace

extern "C" int krn_fill(krn_ctx *ctx, double *d_v, size_t n, double value, const double *d_value)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (n == 0) return KRN_OK;
    KRN_REQUIRE(d_v != nullptr, "null view pointer");
    // +0.0 is all-zero bytes: the copy engine's memset is the fastest fill there is
    if (d_value == nullptr && value == 0.0 && !signbit(value)) {
        KRN_CUDA(cudaMemsetAsync(d_v, 0, n * sizeof(double), ctx->stream));
        return KRN_OK;
    }
    return launch_stream<Op::Fill>(ctx, d_v, nullptr, n, value, d_value);
}

extern "C" int krn_copy(krn_ctx *ctx, double *d_dst, const double *d_src, size_t n)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (n == 0) return KRN_OK;
    KRN_REQUIRE(d_dst && d_src, "null view pointer");
    KRN_CUDA(cudaMemcpyAsync(d_dst, d_src, n * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    return KRN_OK;
}

extern "C" int krn_add_scalar(krn_ctx *ctx, double *d_v, size_t n, double s, const double *d_s)
{
    return launch_stream<Op::AddScalar>(ctx, d_v, nullptr, n, s, d_s);
}

extern "C" int krn_add_view(krn_ctx *ctx, double *d_dst, const double *d_src, size_t n)
{
    KRN_REQUIRE(n == 0 || d_src != nullptr, "null source view");
    return launch_stream<Op::AddView>(ctx, d_dst, d_src, n, 0.0, nullptr);
}

extern "C" int krn_reduce_pairwise(krn_ctx *ctx, const double *d_v, size_t n, double *d_out, int accumulate)
{
    KRN_REQUIRE(ctx && d_out, "null argument");
    if (n == 0) {
        scalar_accumulate_zero<<<1, 1, 0, ctx->stream>>>(d_out, accumulate);
        KRN_LAUNCH_CHECK(ctx);
        return KRN_OK;
    }
    KRN_REQUIRE(d_v != nullptr, "null view pointer");
    const int steps = n <= (size_t(1) << 20) ? 1 : 8;
    const size_t chunk = size_t(kThreads) * 4 * steps;
    const size_t blocks = (n + chunk - 1) / chunk;
    KRN_REQUIRE(blocks <= 0x7fffffffu, "view too large");
    int rc = krn_reserve_partials(ctx, blocks);
    if (rc) return rc;
    double *partials = ctx->d_partials, *scratch = ctx->d_partials + ctx->partial_capacity;
    const bool vec = krn_aligned32(d_v);
#define KRN_TREE(V, S)                                                              \
    tree_kernel<V, S><<<unsigned(blocks), kThreads, 0, ctx->stream>>>(d_v, n, partials, scratch, \
                                                                      ctx->d_ticket, d_out, accumulate)
    if (steps == 1) {
        if (vec) KRN_TREE(true, 1);
        else KRN_TREE(false, 1);
    } else {
        if (vec) KRN_TREE(true, 8);
        else KRN_TREE(false, 8);
    }
#undef KRN_TREE
    KRN_LAUNCH_CHECK(ctx);
    return KRN_OK;
}

extern "C" int krn_check_finite(krn_ctx *ctx, const double *d_v, size_t n, int *d_flag)
{
    KRN_REQUIRE(ctx && d_flag, "null argument");
    if (n == 0) return KRN_OK;
    KRN_REQUIRE(d_v != nullptr, "null view pointer");
    size_t want = (n + kThreads - 1) / kThreads;
    size_t cap = size_t(ctx->sms) * 16;
    finite_kernel<<<unsigned(want < cap ? want : cap), kThreads, 0, ctx->stream>>>(d_v, n, d_flag);
    KRN_LAUNCH_CHECK(ctx);
    return KRN_OK;
}
