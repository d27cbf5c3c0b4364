// Device-side building blocks shared by the ahead-of-time kernels and by the
// kernels generated at run time from program trees (this file is also embedded
// in the library as a string and handed to NVRTC, so it must stay
// self-contained: no #include, builtin types only).
//
// sm_100a only.  fp64 IEEE, compiled with --fmad=false.
#pragma once

typedef unsigned long long krn_u64;
typedef long long krn_i64;

#define KRN_WARP 32
#define KRN_FULL_MASK 0xffffffffu

struct krn_d4 {
    double a, b, c, d;
};

// ---- 256-bit global accesses (LDG.E.256 / STG.E.256, new on sm_100) --------
// "stream": read-once data, bypasses L1 allocation.
// The 256-bit forms need PTX ISA 8.8 (CUDA 12.9).  When this header is compiled at run
// time by an older NVRTC the loader defines KRN_NO_LD256 and each access becomes two
// 128-bit ones (same bytes, same coalescing, twice the instructions).
#ifndef KRN_NO_LD256
__device__ __forceinline__ krn_d4 krn_ld4_stream(const double *p)
{
    krn_d4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d)
        : "l"(p));
    return v;
}
// same, for buffers the kernel also writes (read-modify-write shadows): no .nc
__device__ __forceinline__ krn_d4 krn_ld4_rmw(const double *p)
{
    krn_d4 v;
    asm("ld.global.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
        : "=d"(v.a), "=d"(v.b), "=d"(v.c), "=d"(v.d)
        : "l"(p));
    return v;
}
__device__ __forceinline__ void krn_st4(double *p, const krn_d4 &v)
{
    asm volatile("st.global.L1::no_allocate.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.a), "d"(v.b),
                 "d"(v.c), "d"(v.d)
                 : "memory");
}
#else
__device__ __forceinline__ krn_d4 krn_ld4_stream(const double *p)
{
    krn_d4 v;
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.a), "=d"(v.b) : "l"(p));
    asm("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.c), "=d"(v.d) : "l"(p + 2));
    return v;
}
__device__ __forceinline__ krn_d4 krn_ld4_rmw(const double *p)
{
    krn_d4 v;
    asm("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.a), "=d"(v.b) : "l"(p));
    asm("ld.global.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(v.c), "=d"(v.d) : "l"(p + 2));
    return v;
}
__device__ __forceinline__ void krn_st4(double *p, const krn_d4 &v)
{
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" ::"l"(p), "d"(v.a), "d"(v.b) : "memory");
    asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1,%2};" ::"l"(p + 2), "d"(v.c), "d"(v.d) : "memory");
}
#endif
__device__ __forceinline__ double krn_ld1(const double *p) { return __ldg(p); }

// ---- the reference's reduction tree ----------------------------------------
// pairwise_sum (reference runtime.py:166-177) folds adjacent pairs level by
// level and pads a level of odd length with one +0.0.  Seen from the leaves
// that is a complete binary tree over indices 0..2^L-1 in which a missing leaf
// j >= n behaves as
//     +0.0  if j is the first missing node of a level whose real length is odd
//           and greater than one  (j = roundup(n, 2^l), l = ctz(j), j != 2^l)
//     -0.0  otherwise (the additive identity, also for -0.0 partners)
// With these leaf values a plain padded tree reproduces the reference bit for
// bit, signed zeros included (proof sketch in DESIGN.md, test in
// tests/test_tree_padding.py).
__device__ __forceinline__ double krn_tree_pad(krn_u64 j, krn_u64 n)
{
    krn_u64 low = j & (~j + 1ull);  // 2^ctz(j)
    return (j - low < n && j != low) ? 0.0 : -0.0;
}

// lanes hold 32 consecutive nodes; every lane returns their tree sum
__device__ __forceinline__ double krn_warp_tree(double v)
{
#pragma unroll
    for (int o = 1; o < KRN_WARP; o <<= 1) v = v + __shfl_xor_sync(KRN_FULL_MASK, v, o);
    return v;
}

// Four 32-leaf subtrees at once: r_e of lane L is leaf 32*e + L of a 128-leaf tree (the lane-strided
// mapping of the generated kernels).  Instead of four butterflies (20 shuffles) the lanes split the
// work: after the xor-1 level even lanes carry subtrees 0,1 and odd lanes 2,3, after the xor-2 level
// every lane carries ONE subtree, three more levels finish it, two more fold the four roots:
// 8 shuffles.  Every addition pairs the same two nodes as the reference's tree (operands possibly
// swapped, and IEEE addition is commutative), so the result is bit-identical.  Valid in all lanes.
__device__ __forceinline__ double krn_warp_tree4(double r0, double r1, double r2, double r3)
{
    const int lane = threadIdx.x & 31;
    const bool b0 = lane & 1, b1 = lane & 2;
    double k0 = b0 ? r2 : r0, k1 = b0 ? r3 : r1;  // kept
    double s0 = b0 ? r0 : r2, s1 = b0 ? r1 : r3;  // sent to the partner, which keeps them
    k0 = k0 + __shfl_xor_sync(KRN_FULL_MASK, s0, 1);
    k1 = k1 + __shfl_xor_sync(KRN_FULL_MASK, s1, 1);
    double k = b1 ? k1 : k0, s = b1 ? k0 : k1;
    k = k + __shfl_xor_sync(KRN_FULL_MASK, s, 2);
#pragma unroll
    for (int o = 4; o < KRN_WARP; o <<= 1) k = k + __shfl_xor_sync(KRN_FULL_MASK, k, o);
    // lane bits (b0, b1) now select the subtree: 00 -> 0, 01(b1) -> 1, 10(b0) -> 2, 11 -> 3
    k = k + __shfl_xor_sync(KRN_FULL_MASK, k, 2);  // (0 + 1) in lanes with b0 = 0, (2 + 3) in the others
    return k + __shfl_xor_sync(KRN_FULL_MASK, k, 1);
}

// Tree over `count` (power of two, <= 1024) consecutive nodes held in shared
// memory, by the first warp; result valid in every lane of warp 0.
__device__ __forceinline__ double krn_smem_tree(const double *s, int count, int lane)
{
    // each lane folds a contiguous aligned run of count/32 nodes, then a warp tree
    int per = count >> 5;
    if (per == 0) {  // fewer than 32 nodes: upper lanes hold the identity
        double v = lane < count ? s[lane] : -0.0;
        // identity lanes sit above the real ones and count is a power of two, so
        // the levels beyond log2(count) only add -0.0
        return krn_warp_tree(v);
    }
    // binary-counter evaluation of an in-order tree over `per` leaves
    double stack[6];
    int depth = 0;
    for (int i = 0; i < per; ++i) {
        double v = s[lane * per + i];
        int m = i;
        while (m & 1) {
            v = stack[--depth] + v;
            m >>= 1;
        }
        stack[depth++] = v;
    }
    return krn_warp_tree(stack[0]);
}

// Final stage, run by the last block to arrive: tree over `m` block partials
// (each already the exact tree node of an aligned power-of-two span) using two
// ping-pong arrays.  Explicit per-level rule: odd length and more than one node
// -> last node + (+0.0).  Returns the root in thread 0.
__device__ __forceinline__ double krn_final_tree_levels(double *ping, double *pong, krn_u64 m)
{
    double *src = ping, *dst = pong;
    while (m > 1) {
        krn_u64 half = m >> 1;
        for (krn_u64 i = threadIdx.x; i < half; i += blockDim.x) dst[i] = __ldcg(src + 2 * i) + __ldcg(src + 2 * i + 1);
        if ((m & 1) && threadIdx.x == 0) dst[half] = __ldcg(src + m - 1) + 0.0;
        __syncthreads();
        m = (m + 1) >> 1;
        double *t = src;
        src = dst;
        dst = t;
    }
    return __ldcg(src);
}

// Same result in ONE pass (one round trip to L2 instead of one per level): the m
// partials are themselves the leaves of a reference tree, so the padding rule
// applies again in partial-index space.  Thread t folds the aligned run
// [t*per, (t+1)*per) in order (binary counter), then warp shuffles, then shared
// memory across the block's warps (blockDim.x must be a power of two <= 1024).
__device__ __forceinline__ double krn_final_tree(const double *partials, double * /*scratch*/, krn_u64 m)
{
    __shared__ double s_final[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    krn_u64 per = 1;
    while (per * blockDim.x < m) per <<= 1;
    const krn_u64 first = (krn_u64)threadIdx.x * per;
    double stack[34];
    int depth = 0;
    for (krn_u64 base = 0; base < per; base += 8) {
        // up to 8 independent loads in flight, then folded in order
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            krn_u64 i = first + base + u;
            v[u] = (base + u < per) ? (i < m ? __ldcg(partials + i) : krn_tree_pad(i, m)) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            if (base + u < per) {
                double x = v[u];
                krn_u64 c = base + u;
                while (c & 1) {
                    x = stack[--depth] + x;
                    c >>= 1;
                }
                stack[depth++] = x;
            }
        }
    }
    double r = krn_warp_tree(stack[0]);
    if (lane == 0) s_final[warp] = r;
    __syncthreads();
    double root = 0.0;
    if (warp == 0) root = krn_smem_tree(s_final, nwarps, lane);
    return root;  // valid in thread 0
}

// arrival ticket: returns true in every thread of the block that arrives last.
// Contract: thread 0 is the thread that stored this block's partial, so only it
// needs the release fence (an all-thread fence stalls every warp on MEMBAR).
__device__ __forceinline__ bool krn_last_block(unsigned int *ticket, unsigned int total)
{
    __shared__ unsigned int s_last;
    if (threadIdx.x == 0) {
        __threadfence();
        unsigned int t = atomicAdd(ticket, 1u);
        s_last = (t == total - 1u);
        if (s_last) *ticket = 0u;  // re-arm for the next launch on this stream
    }
    __syncthreads();
    if (s_last) __threadfence();
    return s_last != 0u;
}

// ---- status word -------------------------------------------------------------
__device__ __forceinline__ void krn_fail(krn_i64 *status, krn_i64 code, krn_i64 line, krn_i64 view,
                                         krn_i64 index, krn_i64 index2)
{
    if (atomicCAS((krn_u64 *)status, 0ull, (krn_u64)code) == 0ull) {
        status[1] = line;
        status[2] = view;
        status[3] = index;
        status[4] = index2;
    }
}

// ---- accumulation policies for atomic_add (reference runtime.py:430-447) -----
// hardware fp64 atomic, fire-and-forget (RED.E.ADD.F64)
__device__ __forceinline__ void krn_red_add(double *p, double v) { atomicAdd(p, v); }

// leader-aggregated: only the lanes that hit the SAME address as the first live lane are
// folded (one shuffle + one ballot to find them); everybody else issues its own RED.  Costs
// almost nothing when targets are spread out and removes the same-address serialisation at
// L2 when one row is hot (measured: 0.7 -> 18 Gcontrib/s with 90% of the lanes on one row).
__device__ __forceinline__ void krn_red_add_leader(double *p, double v)
{
    const int lane = threadIdx.x & 31;
    bool done = false;
    // two rounds: the first live lane names an address, the lanes sharing it fold and leave;
    // the second round catches a hot row that the first leader happened not to hit
#pragma unroll
    for (int round = 0; round < 2; ++round) {
        unsigned int live = __ballot_sync(__activemask(), !done);
        if (done) break;
        int leader = __ffs(live) - 1;
        krn_u64 lp = __shfl_sync(live, (krn_u64)p, leader);
        bool mine = (krn_u64)p == lp;
        unsigned int same = __ballot_sync(live, mine);
        if (mine) {
            if (same == (1u << leader)) {
                atomicAdd(p, v);
            } else {
                double acc = 0.0;
                bool first = true;
                unsigned int rest = same;
                while (rest) {  // lowest lane first; every lane of `same` runs the same trip count
                    int src = __ffs(rest) - 1;
                    double pv = __shfl_sync(same, v, src);
                    acc = first ? pv : acc + pv;
                    first = false;
                    rest &= rest - 1;
                }
                if (lane == leader) atomicAdd(p, acc);
            }
            done = true;
        }
    }
    if (!done) atomicAdd(p, v);
}

// warp-aggregated: lanes hitting the same address are folded first (in lane
// order) so one RED leaves the warp per distinct address
__device__ __forceinline__ void krn_red_add_aggregated(double *p, double v)
{
    unsigned int live = __activemask();  // the lanes that reached this site together
    unsigned int peers = __match_any_sync(live, (krn_u64)p);
    int lane = threadIdx.x & 31;
    int leader = __ffs(peers) - 1;
    if (peers == (1u << lane)) {  // sole owner of this address
        atomicAdd(p, v);
        return;
    }
    // fold peer values into the leader, lowest lane first
    double acc = 0.0;
    bool first = true;
    unsigned int rest = peers;
    while (rest) {
        int src = __ffs(rest) - 1;
        double pv = __shfl_sync(peers, v, src);
        acc = first ? pv : acc + pv;
        first = false;
        rest &= rest - 1;
    }
    if (lane == leader) atomicAdd(p, acc);
}
