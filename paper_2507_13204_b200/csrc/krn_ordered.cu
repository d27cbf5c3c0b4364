// Ordered accumulation of deferred atomic_add contributions onto arbitrary
// (non-injective) targets: the reference queues every atomic_add of a kernel as
// (iteration, program order, offset, value), sorts the queue by (iteration,
// program order) and applies `flat[offset] += value` one after the other
// (runtime.py:430-447, 615-620).  Each location therefore receives its
// contributions as a LEFT FOLD in (iteration, program order) - a fixed order,
// which is what makes the reference bit-reproducible for any thread count
// (acceptance C5).
//
// Here: the generated kernel writes one record per executed site group,
//     key[r]               = flat offset of the target element (uint32)
//     val[w * records + r] = the values of the group's sites, program order
// at r = iteration * groups + group, so record order IS the reference's queue
// order.  krn_ordered_accumulate then brings every location's records together
// WITHOUT changing their relative order and folds them in that order:
//
//   A. bucket partition in HBM.  The targets are cut into buckets of 2^LB
//      consecutive elements (LB <= 12: a bucket's targets fit in 32 KB of shared
//      memory).  One or two STABLE least-significant-digit passes over the bits
//      [LB, LB + high) of the key - up to 10 bits each - move (key, values) so
//      that the records of a bucket are contiguous and still in queue order.
//      Per pass: per-tile digit histogram -> exclusive scan of the [digit][tile]
//      table -> scatter that ranks equal digits in tile order (ballots, no
//      atomics) and leaves the tile through shared memory as coalesced runs.
//   B. one block per bucket: the bucket's targets are loaded into shared
//      memory, its records are streamed in chunks; every chunk is sorted
//      stably by the low key bits INSIDE shared memory (one or two 6-7 bit
//      ranking passes over packed (key, slot) words) and each run of equal keys
//      is folded in order onto the target element; the targets are written
//      back with plain coalesced stores.
//
// No atomics on the target, nothing depends on the schedule: the result is
// bit-identical to the reference and identical from run to run.  A location
// that receives very many records is a long chain of dependent fp64 additions
// by definition of the result; it bounds the time of its bucket's block.
//
// All kernels are integer/byte streaming work (no tensor-core shape).  HBM
// traffic per record of width W: pass = 4 B (histogram) + 2 x (4 + 8 W) B;
// final = (4 + 8 W) B read + 16 B per touched target.
#include "krn_common.cuh"
#include "krn_prelude.cuh"

namespace {

typedef unsigned int u32;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                 // records per thread and tile (8: scatter -6%, histogram +35%: no gain)
constexpr int kTile = kThreads * kItems;   // 4096 records per tile of a partition pass
constexpr int kWarpSpan = 32 * kItems;     // consecutive records ranked by one warp
constexpr int kScanChunk = kThreads * 8;
constexpr int kMaxWidth = 4;
constexpr int kMaxPassBits = 10;           // digits of a partition pass
constexpr int kMaxLocalBits = 12;          // low key bits resolved inside shared memory
// a bucket's block stages 256 * PER records per round (PER = 8 for one value per record, 4 for wider
// records: the staged values must leave room for 3 blocks per SM); packed word = (low key << slot bits) | slot
constexpr u32 kNone = 0xffffffffu;

__device__ __forceinline__ u32 lanemask_lt()
{
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Lanes of the warp holding the same digit as the caller (valid lanes only): one ballot per
// bit.  (match.any does the same in one instruction but its cost grows with the number of distinct
// values in the warp - measured: 166 us per 16.7 M-record pass against 110 us with ballots; shared
// memory atomics cost 2 cycles per lane and bounded the histogram at 115 us per pass.)
template <int BITS>
__device__ __forceinline__ u32 same_digit_lanes(u32 d, bool valid)
{
    u32 peers = __ballot_sync(KRN_FULL_MASK, valid);
#pragma unroll
    for (int b = 0; b < BITS; ++b) {
        const bool bit = (d >> b) & 1u;
        const u32 with = __ballot_sync(KRN_FULL_MASK, bit);
        peers &= bit ? with : ~with;
    }
    return peers;
}
// Exclusive scan over `radix` per-digit totals held in shared memory (radix <= 1024, a power of two
// or less than kThreads): thread t owns the digits [t*per, (t+1)*per).  out[d] = sum of tot[< d].
__device__ __forceinline__ void digit_scan(const u32 *tot, u32 *out, int radix, u32 *s_wsum)
{
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int per = (radix + kThreads - 1) / kThreads;
    u32 mine[4];
    u32 sum = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int d = threadIdx.x * per + u;
        mine[u] = (u < per && d < radix) ? tot[d] : 0u;
        sum += mine[u];
    }
    u32 inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(KRN_FULL_MASK, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    u32 run = inc - sum;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
        if (w < warp) run += s_wsum[w];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int d = threadIdx.x * per + u;
        if (u < per && d < radix) out[d] = run;
        run += mine[u];
    }
    __syncthreads();
}

// ---- pass step 1: digit histogram of every tile ---------------------------------------
// table[digit * tiles + tile]: scanned in this order it yields, for every (digit, tile), the
// number of records with a smaller digit anywhere plus those with the same digit in earlier
// tiles - the stable destination of the tile's first record with that digit.
// The first pass also finds out whether the queue is ALREADY in bucket order (bucket id = (key >> lb) &
// hmask never decreases from one record to the next): affine non-injective maps (restriction stencils),
// sorted or block-clustered index maps.  Then no record has to move: *in_order stays kNone, every later
// kernel of the partition returns at once, and boundaries + fold read the queue where it is.
// (record p - 1 is the neighbouring lane's record of the same round: only lane 0 has to load it; the all-ones
// mark of a site that did not execute is the largest bucket id with or without hmask)
__device__ __forceinline__ bool out_of_order(const u32 *__restrict__ keys, size_t p, size_t m, u32 key, int lb)
{
    const u32 bucket = key >> lb;
    u32 before = __shfl_up_sync(KRN_FULL_MASK, bucket, 1);
    if ((threadIdx.x & 31) == 0) before = (p > 0 && p < m) ? keys[p - 1] >> lb : 0u;
    return p < m && before > bucket;
}
// one store per BLOCK at most (a random queue has a violation at every other record: per-thread stores to
// the one word were measured at +0.25 ms per 16.7 M records)
__device__ __forceinline__ void publish_order(bool bad, u32 *in_order)
{
    if (__syncthreads_or(bad) && threadIdx.x == 0 && *in_order != 0u) *in_order = 0u;
}

template <int BITS>
__global__ void __launch_bounds__(kThreads)
ord_hist(const u32 *__restrict__ keys, size_t m, int shift, u32 tiles, u32 *__restrict__ table, int lb, u32 hmask,
         u32 *in_order, int check)
{
    if (!check && *in_order == kNone) return;
    // digits of 9 and 10 bits: per-warp counters, bumped by the lowest lane of every group of equal
    // digits (ballots) with a plain read-modify-write
    constexpr u32 mask = (1u << BITS) - 1u;
    constexpr int kRadix = 1 << BITS;
    __shared__ u32 s_cnt[kWarps][kRadix];
    for (int k = threadIdx.x; k < kWarps * kRadix; k += kThreads) (&s_cnt[0][0])[k] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = size_t(blockIdx.x) * kTile + size_t(warp) * kWarpSpan;
    u32 key[kItems];
    bool bad = false;
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const size_t p = base + size_t(r) * 32 + lane;
        key[r] = p < m ? keys[p] : 0u;
    }
    if (check) {  // (behind ALL the loads: a test right behind its load would wait for it before the next is issued)
#pragma unroll
        for (int r = 0; r < kItems; ++r) bad |= out_of_order(keys, base + size_t(r) * 32 + lane, m, key[r], lb);
        publish_order(bad, in_order);
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const bool valid = base + size_t(r) * 32 + lane < m;
        const u32 d = (key[r] >> shift) & mask;
        const u32 peers = same_digit_lanes<BITS>(d, valid);
        if (valid && lane == __ffs(peers) - 1) s_cnt[warp][d] += (u32)__popc(peers);
        __syncwarp();
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kThreads) {
        u32 total = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) total += s_cnt[w][d];
        table[size_t(d) * tiles + blockIdx.x] = total;
    }
}

// Digits of up to 8 bits: every THREAD counts its 16 records in byte counters of its own (a thread
// sees at most 16 records: a byte holds the count), so counting is a byte load, an add and a byte
// store per record - no ballots, no atomics: 0.5 instead of 2.1 warp instructions per record.
// Row d of the counter matrix holds the 256 threads' counts of digit d; thread t uses byte t/64 of word
// t%64, so the lanes of a warp always hit 32 different banks.  The per-digit totals are then summed
// one word (four counts) per dp4a.
template <int BITS>
__global__ void __launch_bounds__(kThreads)
ord_hist_bytes(const u32 *__restrict__ keys, size_t m, int shift, u32 tiles, u32 *__restrict__ table, int lb,
               u32 hmask, u32 *in_order, int check)
{
    if (!check && *in_order == kNone) return;
    constexpr u32 mask = (1u << BITS) - 1u;
    constexpr int kRadix = 1 << BITS;
    extern __shared__ __align__(16) unsigned char ord_smem[];
    u32 *words = reinterpret_cast<u32 *>(ord_smem);  // [kRadix][64]
    for (int k = threadIdx.x; k < kRadix * 16; k += kThreads) reinterpret_cast<uint4 *>(words)[k] = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const size_t base = size_t(blockIdx.x) * kTile;
    unsigned char *mine = ord_smem + 4 * (threadIdx.x & 63) + (threadIdx.x >> 6);
    // which records a thread counts is immaterial for a histogram: four CONSECUTIVE records per 128-bit load
    // (the tile starts at a multiple of 4096 records; a caller's queue need not be 16-byte aligned), four
    // loads per thread
    const bool vec = (reinterpret_cast<size_t>(keys) & 15u) == 0;
    u32 key[kItems];
#pragma unroll
    for (int g = 0; g < kItems / 4; ++g) {
        const size_t p = base + (size_t(g) * kThreads + threadIdx.x) * 4;
        if (vec && p + 4 <= m) {
            const uint4 q = *reinterpret_cast<const uint4 *>(keys + p);
            key[4 * g] = q.x, key[4 * g + 1] = q.y, key[4 * g + 2] = q.z, key[4 * g + 3] = q.w;
        } else {
#pragma unroll
            for (int u = 0; u < 4; ++u) key[4 * g + u] = p + u < m ? keys[p + u] : 0u;
        }
    }
    if (check) {
        // in bucket order?  Three comparisons inside the thread's four records, one with the record before
        // them: the neighbouring lane's last one (lane 0 loads it).  Behind ALL the loads: a test right behind
        // its load would wait for it before the next load is issued.
        bool bad = false;
#pragma unroll
        for (int g = 0; g < kItems / 4; ++g) {
            const size_t p = base + (size_t(g) * kThreads + threadIdx.x) * 4;
            const u32 b0 = key[4 * g] >> lb, b1 = key[4 * g + 1] >> lb, b2 = key[4 * g + 2] >> lb, b3 = key[4 * g + 3] >> lb;
            u32 before = __shfl_up_sync(KRN_FULL_MASK, b3, 1);
            if ((threadIdx.x & 31) == 0) before = (p > 0 && p < m) ? keys[p - 1] >> lb : 0u;
            bad |= (p < m && before > b0) | (p + 1 < m && b0 > b1) | (p + 2 < m && b1 > b2) | (p + 3 < m && b2 > b3);
        }
        publish_order(bad, in_order);
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        if (base + (size_t(r / 4) * kThreads + threadIdx.x) * 4 + (r & 3) < m) {
            unsigned char *c = mine + (((key[r] >> shift) & mask) << 8);
            *c = (unsigned char)(*c + 1);
        }
    }
    __syncthreads();
    for (int d = threadIdx.x; d < kRadix; d += kThreads) {
        const uint4 *row = reinterpret_cast<const uint4 *>(words + d * 64);
        u32 total = 0;
#pragma unroll
        for (int g = 0; g < 16; ++g) {
            const uint4 q = row[(g + threadIdx.x) & 15];  // rotated: the lanes read different banks
            total = __dp4a(q.x, 0x01010101u, total);
            total = __dp4a(q.y, 0x01010101u, total);
            total = __dp4a(q.z, 0x01010101u, total);
            total = __dp4a(q.w, 0x01010101u, total);
        }
        table[size_t(d) * tiles + blockIdx.x] = total;
    }
}

// ---- pass step 2: exclusive scan of the table -------------------------------------------
// Block-wide exclusive scan of kScanChunk consecutive entries held 8 per thread; returns the
// chunk total in every thread.
__device__ __forceinline__ u32 block_scan8(u32 (&x)[8], u32 carry)
{
    __shared__ u32 s_w[kWarps];
    __shared__ u32 s_total;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    u32 sum = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) sum += x[u];
    u32 inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(KRN_FULL_MASK, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_w[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        u32 w = lane < kWarps ? s_w[lane] : 0, winc = w;
#pragma unroll
        for (int o = 1; o < kWarps; o <<= 1) {
            const u32 t = __shfl_up_sync(KRN_FULL_MASK, winc, o);
            if (lane >= o) winc += t;
        }
        if (lane < kWarps) s_w[lane] = winc - w;
        if (lane == kWarps - 1) s_total = winc;
    }
    __syncthreads();
    u32 run = carry + s_w[warp] + (inc - sum);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const u32 t = x[u];
        x[u] = run;
        run += t;
    }
    const u32 total = s_total;
    __syncthreads();  // s_w / s_total are reused by the caller's next round
    return total;
}

__device__ __forceinline__ void load8(const u32 *data, size_t first, size_t count, u32 (&x)[8])
{
#pragma unroll
    for (int u = 0; u < 8; ++u) x[u] = first + u < count ? data[first + u] : 0u;
}
__device__ __forceinline__ void store8(u32 *data, size_t first, size_t count, const u32 (&x)[8])
{
#pragma unroll
    for (int u = 0; u < 8; ++u)
        if (first + u < count) data[first + u] = x[u];
}

// one block walks the whole array, chunk after chunk (small tables, and the block sums of big ones)
__global__ void __launch_bounds__(kThreads) scan_single(u32 *data, size_t count, const u32 *in_order)
{
    if (*in_order == kNone) return;
    u32 carry = 0;
    for (size_t base = 0; base < count; base += kScanChunk) {
        u32 x[8];
        const size_t first = base + size_t(threadIdx.x) * 8;
        load8(data, first, count, x);
        carry += block_scan8(x, carry);
        store8(data, first, count, x);
    }
}

__global__ void __launch_bounds__(kThreads) scan_sums(const u32 *__restrict__ data, size_t count, u32 *__restrict__ sums,
                                                       const u32 *in_order)
{
    if (*in_order == kNone) return;
    __shared__ u32 s_w[kWarps];
    const size_t first = size_t(blockIdx.x) * kScanChunk + size_t(threadIdx.x) * 8;
    u32 x[8], sum = 0;
    load8(data, first, count, x);
#pragma unroll
    for (int u = 0; u < 8; ++u) sum += x[u];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(KRN_FULL_MASK, sum, o);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = sum;
    __syncthreads();
    if (threadIdx.x == 0) {
        u32 t = 0;
        for (int w = 0; w < kWarps; ++w) t += s_w[w];
        sums[blockIdx.x] = t;
    }
}

__global__ void __launch_bounds__(kThreads) scan_apply(u32 *data, size_t count, const u32 *__restrict__ sums,
                                                        const u32 *in_order)
{
    if (*in_order == kNone) return;
    const size_t first = size_t(blockIdx.x) * kScanChunk + size_t(threadIdx.x) * 8;
    u32 x[8];
    load8(data, first, count, x);
    block_scan8(x, sums[blockIdx.x]);
    store8(data, first, count, x);
}

// ---- pass step 3: stable scatter ------------------------------------------------------------
// Warp w of the tile ranks records [w*512, (w+1)*512) of the tile, 32 consecutive records per
// round: the lanes holding the same digit find each other with ballots; their rank within the
// round is the number of lower lanes among them, and the warp's running count of the digit
// (shared memory, bumped by the lowest lane) orders the rounds.  Tile order = (warp, round, lane),
// so equal digits keep their input order.  Keys, then every value plane in turn, are placed in
// shared memory in digit order and leave the tile as runs of consecutive destinations.
// Values are planes: vals[w * m + record].
template <int BITS>
__global__ void __launch_bounds__(kThreads)
ord_scatter(const u32 *__restrict__ keys_in, const double *__restrict__ vals_in, u32 *__restrict__ keys_out,
            double *__restrict__ vals_out, const u32 *__restrict__ table, size_t m, int shift, u32 tiles, int width,
            const u32 *in_order)
{
    if (*in_order == kNone) return;
    constexpr u32 mask = (1u << BITS) - 1u;
    constexpr int kRadix = 1 << BITS;
    extern __shared__ __align__(16) unsigned char ord_smem[];
    double *s_val = reinterpret_cast<double *>(ord_smem);   // [kTile]
    u32 *s_key = reinterpret_cast<u32 *>(s_val + kTile);     // [kTile]
    u32 *s_g = s_key + kTile;                                // [kTile] global destination of every sorted slot
    u32 *s_cnt = s_g + kTile;      // [kWarps][kRadix] per-warp digit counts, then the warp's first slot of the digit
    u32 *s_tot = s_cnt + kWarps * kRadix;  // [kRadix] records of the digit in the tile
    u32 *s_first = s_tot + kRadix;          // [kRadix] first slot of the digit in the sorted tile
    u32 *s_dest = s_first + kRadix;         // [kRadix] global destination of that slot
    __shared__ u32 s_wsum[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = size_t(blockIdx.x) * kTile;
    const u32 live = u32(m - base < size_t(kTile) ? m - base : size_t(kTile));  // records of this tile
    for (int k = threadIdx.x; k < kWarps * kRadix; k += kThreads) s_cnt[k] = 0;
    // the tile's values are not needed before the keys are ranked: start them towards L2 now (one 128-byte
    // line per thread and plane), so that their loads below do not pay the DRAM latency a second time
    // (measured: 0.704 -> 0.690 ms per 16.7 M records together with the prefetch in the fold)
    for (int w = 0; w < width; ++w) {
        const u32 first = u32(threadIdx.x) * 16u;
        if (first < live) asm volatile("prefetch.global.L2 [%0];" ::"l"(vals_in + size_t(w) * m + base + first));
    }
    __syncthreads();

    u32 key[kItems];
    unsigned short slot[kItems];
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const u32 t = u32(warp) * kWarpSpan + u32(r) * 32 + lane;  // position in the tile
        key[r] = t < live ? keys_in[base + t] : 0u;
    }
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const u32 t = u32(warp) * kWarpSpan + u32(r) * 32 + lane;
        const bool valid = t < live;
        const u32 d = (key[r] >> shift) & mask;
        const u32 peers = same_digit_lanes<BITS>(d, valid);
        const int leader = valid ? __ffs(peers) - 1 : lane;
        u32 before = 0;
        if (valid && lane == leader) {
            before = s_cnt[warp * kRadix + d];
            s_cnt[warp * kRadix + d] = before + (u32)__popc(peers);
        }
        before = __shfl_sync(KRN_FULL_MASK, before, leader);
        slot[r] = (unsigned short)(before + (u32)__popc(peers & lt));
        __syncwarp();  // the next round's leader of this digit may be another lane
    }
    __syncthreads();

    // per digit: exclusive prefix over the warps and the tile total; then an exclusive scan over the digits
    for (int d = threadIdx.x; d < kRadix; d += kThreads) {
        u32 total = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const u32 c = s_cnt[w * kRadix + d];
            s_cnt[w * kRadix + d] = total;
            total += c;
        }
        s_tot[d] = total;
        s_dest[d] = table[size_t(d) * tiles + blockIdx.x];
    }
    __syncthreads();
    digit_scan(s_tot, s_first, kRadix, s_wsum);

#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const u32 t = u32(warp) * kWarpSpan + u32(r) * 32 + lane;
        if (t < live) {
            const u32 d = (key[r] >> shift) & mask;
            const u32 s = s_first[d] + s_cnt[warp * kRadix + d] + slot[r];
            slot[r] = (unsigned short)s;
            s_key[s] = key[r];
        }
    }
    __syncthreads();
    // sorted slot s leaves the tile to s_g[s] (computed once, reused by every value plane)
    for (u32 s = threadIdx.x; s < live; s += kThreads) {
        const u32 k = s_key[s];
        const u32 d = (k >> shift) & mask;
        const u32 g = s_dest[d] + (s - s_first[d]);
        s_g[s] = g;
        keys_out[g] = k;
    }
    for (int w = 0; w < width; ++w) {
        const double *__restrict__ src = vals_in + size_t(w) * m + base;
        double *__restrict__ dst = vals_out + size_t(w) * m;
#pragma unroll
        for (int r = 0; r < kItems; ++r) {
            const u32 t = u32(warp) * kWarpSpan + u32(r) * 32 + lane;
            // (the values of a site that did not execute travel along unread: the producer of the queue
            // clears them when it has guarded sites, OrderedStage in runtime.py)
            if (t < live) s_val[slot[r]] = src[t];
        }
        __syncthreads();
        for (u32 s = threadIdx.x; s < live; s += kThreads) dst[s_g[s]] = s_val[s];
        __syncthreads();
    }
}

// ---- bucket boundaries -----------------------------------------------------------------------
// records are sorted by bucket id = (key >> lb) & hmask: first / one-past-last position per bucket
__global__ void __launch_bounds__(kThreads)
ord_mark(const u32 *__restrict__ keys_moved, const u32 *__restrict__ keys_queue, const u32 *in_order, size_t m, int lb,
         u32 hmask, u32 *__restrict__ start, u32 *__restrict__ end)
{
    const u32 *__restrict__ keys = *in_order == kNone ? keys_queue : keys_moved;
    // 4 consecutive records per thread (one 128-bit load when the buffer is 16-byte aligned: the moved
    // queue always is, a caller's queue need not be)
    const size_t p = (size_t(blockIdx.x) * kThreads + threadIdx.x) * 4;
    if (p >= m) return;
    u32 k[6];  // k[0] = predecessor of record p, k[5] = successor of record p + 3
    if ((reinterpret_cast<size_t>(keys) & 15u) == 0 && p + 4 <= m) {
        const uint4 q = *reinterpret_cast<const uint4 *>(keys + p);
        k[1] = q.x, k[2] = q.y, k[3] = q.z, k[4] = q.w;
    } else {
        for (int u = 0; u < 4; ++u) k[1 + u] = p + u < m ? keys[p + u] : 0u;
    }
    k[0] = p > 0 ? keys[p - 1] : 0u;
    k[5] = p + 4 < m ? keys[p + 4] : 0u;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        if (p + u >= m) break;
        const u32 b = (k[1 + u] >> lb) & hmask;
        if (p + u == 0 || ((k[u] >> lb) & hmask) != b) start[b] = u32(p + u);
        if (p + u + 1 == m || ((k[2 + u] >> lb) & hmask) != b) end[b] = u32(p + u + 1);
    }
}

// ---- phase B: one block per bucket ---------------------------------------------------------
// Stable ranking pass over the packed words in[0, cnt) by the 4 bits at `shift`, inside shared
// memory.  Thread t owns the PER CONSECUTIVE words [PER*t, PER*t + PER) and counts their digits
// in 16 counters of its own (plain loads and stores: no ballots, no atomics); an exclusive scan of
// the counter matrix in (digit, thread) order - thread-major within a digit, i.e. input order - turns
// every counter into the first output slot of that thread's words with that digit.  0.8 instead of
// 3.3 warp instructions per record and pass compared with ballot ranking (which pays per digit BIT
// and per 32 records; it stays the choice of the partition passes, whose digits are 7-10 bits wide).
constexpr int kLocalBits = 4;

template <int kPerThread>
__device__ __forceinline__ void local_pass4(const u32 *in, u32 *out, int cnt, int shift, unsigned short *c16,
                                            u32 *s_wsum)
{
    const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
#pragma unroll
    for (int d = 0; d < 16; ++d) c16[d * kThreads + t] = 0;
    u32 w[kPerThread];
    unsigned char r[kPerThread];
#pragma unroll
    for (int g = 0; g < kPerThread / 4; ++g) {
        const uint4 a = reinterpret_cast<const uint4 *>(in)[(kPerThread / 4) * t + g];
        w[4 * g] = a.x, w[4 * g + 1] = a.y, w[4 * g + 2] = a.z, w[4 * g + 3] = a.w;
    }
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
        if (kPerThread * t + j < cnt) {
            unsigned short *c = c16 + ((w[j] >> shift) & 15u) * kThreads + t;
            const unsigned short before = *c;
            r[j] = (unsigned char)before;
            *c = (unsigned short)(before + 1);
        }
    }
    __syncthreads();
    // exclusive scan of the 16 x 256 counters in row-major order: thread t takes entries [16t, 16t + 16)
    {
        uint4 *mine = reinterpret_cast<uint4 *>(c16) + 2 * t;
        uint4 q[2] = {mine[0], mine[1]};
        u32 *h = reinterpret_cast<u32 *>(q);  // 8 words, two counts each
        u32 v[16], sum = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            v[2 * k] = h[k] & 0xffffu;
            v[2 * k + 1] = h[k] >> 16;
        }
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            const u32 c = v[k];
            v[k] = sum;
            sum += c;
        }
        u32 inc = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const u32 up = __shfl_up_sync(KRN_FULL_MASK, inc, o);
            if (lane >= o) inc += up;
        }
        if (lane == 31) s_wsum[warp] = inc;
        __syncthreads();
        u32 run = inc - sum;
#pragma unroll
        for (int k = 0; k < kWarps; ++k)
            if (k < warp) run += s_wsum[k];
#pragma unroll
        for (int k = 0; k < 8; ++k) h[k] = (v[2 * k] + run) | ((v[2 * k + 1] + run) << 16);
        mine[0] = q[0];
        mine[1] = q[1];
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kPerThread; ++j) {
        if (kPerThread * t + j < cnt) {
            const u32 first = c16[((w[j] >> shift) & 15u) * kThreads + t];
            out[first + r[j]] = w[j];
        }
    }
    __syncthreads();
}

struct Cols {
    int c[kMaxWidth];
};

// (Measured and rejected, 16 M records onto 16 M targets, fold alone 293 us: folding a chunk in ROUNDS
// while its records sit in registers - every pending record bids for its location with its position,
// the earliest one adds itself to the tile, repeat - instead of sorting the chunk.  With shared-memory
// atomicMin as the bid: 210 us, but ATOMS costs 2 cycles per LANE, and locations with 8 records in a row
// or 2+ records per chunk on average got slower (0.77 -> 0.86 ms, 0.61 -> 0.69 ms whole call).  With
// plain stores iterated to the minimum: 283 us, 2.9 warp instructions per record in the bidding loop
// and 1.9 in the apply step, every warp still walking its 8 slots in the late rounds.  The sorted fold
// stays: its cost does not depend on how the records are distributed.)
//
// LANES = false: the WIDTH values of a record go, one after the other, to target[key] (adjacent sites
// on one location).  LANES = true: the target is rows x ncols, key is the ROW and value plane l goes
// to column cols.c[l] of it (sites that name the literal columns of one row: one record instead of
// WIDTH) - different locations, so their mutual order is immaterial, while every location still
// receives its records in queue order.  target_size = number of keys (elements / rows).
template <int WIDTH, bool LANES, int PER>
__global__ void __launch_bounds__(kThreads)
ord_bucket_fold(const u32 *__restrict__ keys_moved, const double *__restrict__ vals_moved,
                const u32 *__restrict__ keys_queue, const double *__restrict__ vals_queue, const u32 *in_order, size_t m,
                double *__restrict__ target, size_t target_size, int ncols, Cols cols, int lb,
                const u32 *__restrict__ start, const u32 *__restrict__ end)
{
    const bool queue = *in_order == kNone;
    const u32 *__restrict__ keys = queue ? keys_queue : keys_moved;
    const double *__restrict__ vals = queue ? vals_queue : vals_moved;
    constexpr int width = WIDTH;
    constexpr int kChunk = kThreads * PER;
    constexpr int kSlotBits = PER == 8 ? 11 : 10;
    const u32 b = blockIdx.x;
    const u32 s0 = start[b];
    if (s0 == kNone) return;
    const size_t t0 = size_t(b) << lb;
    if (t0 >= target_size) return;  // sites that did not execute
    const u32 e0 = end[b];
    const int tn = int(target_size - t0 < (size_t(1) << lb) ? target_size - t0 : (size_t(1) << lb));
    const int tw = LANES ? ncols : 1;  // doubles per key in the tile

    extern __shared__ __align__(16) unsigned char ord_smem[];
    double *tile = reinterpret_cast<double *>(ord_smem);   // [(1 << lb) * tw], padded to 16 bytes
    double *cv = tile + ((((size_t(1) << lb) * tw) + 1) & ~size_t(1));  // [width][kChunk]
    u32 *wa = reinterpret_cast<u32 *>(cv + size_t(width) * kChunk);  // [kChunk]
    u32 *wb = wa + kChunk;                                   // [kChunk]
    unsigned short *c16 = reinterpret_cast<unsigned short *>(wb + kChunk);  // [16][kThreads] ranking counters
    __shared__ u32 s_wsum[kWarps];

    {
        // the first chunk's records: towards L2 while the tile is loaded (one 128-byte line per thread)
        const u32 cnt0 = e0 - s0 < u32(kChunk) ? e0 - s0 : u32(kChunk);
        if (u32(threadIdx.x) * 32u < cnt0) asm volatile("prefetch.global.L2 [%0];" ::"l"(keys + s0 + threadIdx.x * 32u));
        for (int w = 0; w < width; ++w)
            for (u32 q = u32(threadIdx.x) * 16u; q < cnt0; q += kThreads * 16u)
                asm volatile("prefetch.global.L2 [%0];" ::"l"(vals + size_t(w) * m + s0 + q));
    }
    for (int k = threadIdx.x; k < tn * tw; k += kThreads) tile[k] = target[t0 * tw + k];
    const int passes = (lb + kLocalBits - 1) / kLocalBits;  // stable 4-bit passes over the low key bits
    for (u32 c = s0; c < e0; c += kChunk) {
        const int cnt = int(e0 - c < u32(kChunk) ? e0 - c : u32(kChunk));
        __syncthreads();  // the previous chunk's fold is done with wa/wb/cv (and the tile is loaded)
        // A chunk whose keys never decrease (a hot location, a sorted or clustered index map, the
        // restriction stencils) is in fold order as it stands: the local ranking passes are skipped.
        // Every thread first tests ONE pair of neighbours (its first record against the one before it):
        // a random chunk fails that test at once, at the price of one load per thread and no barrier of
        // its own; only when all 256 sampled pairs rise are the remaining pairs compared.
        bool rising = true;
        for (int q = threadIdx.x; q < cnt; q += kThreads) {
            const u32 key = keys[c + q];
            if (q == int(threadIdx.x) && q > 0 && keys[c + q - 1] > key) rising = false;
            u32 kl = key - u32(t0);
            if (kl >= u32(tn)) kl = u32(tn) - 1u;  // cannot happen for keys < target_size: never leave the tile
            wa[q] = (kl << kSlotBits) | u32(q);
#pragma unroll
            for (int w = 0; w < width; ++w) cv[w * kChunk + q] = vals[size_t(w) * m + c + q];
        }
        bool presorted = __syncthreads_and(rising) != 0;
        if (presorted) {
            for (int q = int(threadIdx.x) + kThreads; q < cnt; q += kThreads)
                if ((wa[q - 1] >> kSlotBits) > (wa[q] >> kSlotBits)) rising = false;
            presorted = __syncthreads_and(rising) != 0;
        }
        u32 *fin = wa, *other = wb;
        for (int pass = 0; pass < (presorted ? 0 : passes); ++pass) {
            local_pass4<PER>(fin, other, cnt, kSlotBits + kLocalBits * pass, c16, s_wsum);
            u32 *swap = fin;
            fin = other;
            other = swap;
        }
        // fold: the thread at the head of a run of equal keys adds the run, in order
        for (int q = threadIdx.x; q < cnt; q += kThreads) {
            const u32 k = fin[q] >> kSlotBits;
            if (q > 0 && (fin[q - 1] >> kSlotBits) == k) continue;
            if (LANES) {
                double acc[WIDTH];
#pragma unroll
                for (int w = 0; w < width; ++w) acc[w] = tile[k * tw + cols.c[w]];
                for (int j = q; j < cnt && (fin[j] >> kSlotBits) == k; ++j) {
                    const u32 sl = fin[j] & u32(kChunk - 1);
#pragma unroll
                    for (int w = 0; w < width; ++w) acc[w] = acc[w] + cv[w * kChunk + sl];
                }
#pragma unroll
                for (int w = 0; w < width; ++w) tile[k * tw + cols.c[w]] = acc[w];
                continue;
            }
            double acc = tile[k];
            int j = q;
            // long runs (a hot location): the chain of dependent additions is the definition of the
            // result; the words and values of the NEXT 8 records are fetched while the current 8 are added
            if (width == 1) {
                double v[8];
                bool have = j + 8 <= cnt && (fin[j + 7] >> kSlotBits) == k;
                if (have) {
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = cv[fin[j + u] & u32(kChunk - 1)];
                }
                while (have) {
                    const int jn = j + 8;
                    const bool have_n = jn + 8 <= cnt && (fin[jn + 7] >> kSlotBits) == k;
                    double vn[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) vn[u] = have_n ? cv[fin[jn + u] & u32(kChunk - 1)] : 0.0;
#pragma unroll
                    for (int u = 0; u < 8; ++u) acc = acc + v[u];
#pragma unroll
                    for (int u = 0; u < 8; ++u) v[u] = vn[u];
                    j = jn;
                    have = have_n;
                }
            } else {
                while (j + 8 <= cnt && (fin[j + 7] >> kSlotBits) == k) {
                    u32 sl[8];
#pragma unroll
                    for (int u = 0; u < 8; ++u) sl[u] = fin[j + u] & u32(kChunk - 1);
#pragma unroll
                    for (int u = 0; u < 8; ++u) {
#pragma unroll
                        for (int w = 0; w < width; ++w) acc = acc + cv[w * kChunk + sl[u]];
                    }
                    j += 8;
                }
            }
            while (j < cnt && (fin[j] >> kSlotBits) == k) {
                const u32 sl = fin[j] & u32(kChunk - 1);
#pragma unroll
                for (int w = 0; w < width; ++w) acc = acc + cv[w * kChunk + sl];
                ++j;
            }
            tile[k] = acc;
        }
    }
    __syncthreads();
    for (int k = threadIdx.x; k < tn * tw; k += kThreads) target[t0 * tw + k] = tile[k];
}

#define KRN_BITS_SWITCH(bits, CALL) \
    switch (bits) {                 \
    case 1: CALL(1); break;         \
    case 2: CALL(2); break;         \
    case 3: CALL(3); break;         \
    case 4: CALL(4); break;         \
    case 5: CALL(5); break;         \
    case 6: CALL(6); break;         \
    case 7: CALL(7); break;         \
    case 8: CALL(8); break;         \
    case 9: CALL(9); break;         \
    default: CALL(10); break;       \
    }

cudaError_t launch_hist(int bits, unsigned tiles, cudaStream_t st, const u32 *keys, size_t m, int shift, u32 ntiles,
                        u32 *table, int lb, u32 hmask, u32 *in_order, int check)
{
    cudaError_t e = cudaSuccess;
    const size_t smem = size_t(256) << bits;  // 2^bits rows of 256 byte counters
#define KRN_BYTES(B)                                                                                             \
    do {                                                                                                         \
        e = cudaFuncSetAttribute(ord_hist_bytes<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));     \
        if (e == cudaSuccess)                                                                                    \
            ord_hist_bytes<B><<<tiles, kThreads, smem, st>>>(keys, m, shift, ntiles, table, lb, hmask, in_order, \
                                                             check);                                             \
    } while (0)
    switch (bits) {
    case 1: KRN_BYTES(1); break;
    case 2: KRN_BYTES(2); break;
    case 3: KRN_BYTES(3); break;
    case 4: KRN_BYTES(4); break;
    case 5: KRN_BYTES(5); break;
    case 6: KRN_BYTES(6); break;
    case 7: KRN_BYTES(7); break;
    case 8: KRN_BYTES(8); break;
    case 9: ord_hist<9><<<tiles, kThreads, 0, st>>>(keys, m, shift, ntiles, table, lb, hmask, in_order, check); break;
    default: ord_hist<10><<<tiles, kThreads, 0, st>>>(keys, m, shift, ntiles, table, lb, hmask, in_order, check); break;
    }
#undef KRN_BYTES
    return e;
}

size_t scatter_smem(int bits)
{
    return size_t(kTile) * 16 + (size_t(kWarps + 3) << bits) * 4;
}

cudaError_t launch_scatter(int bits, unsigned tiles, cudaStream_t st, const u32 *keys_in, const double *vals_in,
                           u32 *keys_out, double *vals_out, const u32 *table, size_t m, int shift, u32 ntiles, int width,
                           const u32 *in_order)
{
    const size_t smem = scatter_smem(bits);
    cudaError_t e = cudaSuccess;
#define KRN_CALL(B)                                                                                              \
    do {                                                                                                         \
        e = cudaFuncSetAttribute(ord_scatter<B>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));        \
        if (e == cudaSuccess)                                                                                    \
            ord_scatter<B><<<tiles, kThreads, smem, st>>>(keys_in, vals_in, keys_out, vals_out, table, m, shift, \
                                                          ntiles, width, in_order);                              \
    } while (0)
    KRN_BITS_SWITCH(bits, KRN_CALL)
#undef KRN_CALL
    return e;
}

inline int bit_length(size_t x)
{
    int b = 0;
    while (x) {
        ++b;
        x >>= 1;
    }
    return b;
}

}  // namespace

extern "C" int krn_memset(krn_ctx *ctx, void *d_ptr, int byte, size_t bytes)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (bytes == 0) return KRN_OK;
    KRN_REQUIRE(d_ptr != nullptr, "null pointer");
    KRN_CUDA(cudaMemsetAsync(d_ptr, byte, bytes, ctx->stream));
    return KRN_OK;
}

namespace {
int ordered_impl(krn_ctx *ctx, double *d_target, size_t target_size, int ncols, const int *cols, const uint32_t *d_keys,
                 const double *d_vals, size_t records, int width);
}

extern "C" int krn_ordered_accumulate(krn_ctx *ctx, double *d_target, size_t target_size, const uint32_t *d_keys,
                                      const double *d_vals, size_t records, int width)
{
    return ordered_impl(ctx, d_target, target_size, 0, nullptr, d_keys, d_vals, records, width);
}

extern "C" int krn_ordered_accumulate_rows(krn_ctx *ctx, double *d_target, size_t rows, int ncols, const int *cols,
                                           int planes, const uint32_t *d_keys, const double *d_vals, size_t records)
{
    KRN_REQUIRE(ncols >= 1 && cols != nullptr, "a rows x ncols target needs its column list");
    for (int l = 0; l < planes && l < kMaxWidth; ++l) KRN_REQUIRE(cols[l] >= 0 && cols[l] < ncols, "column outside the target");
    return ordered_impl(ctx, d_target, rows, ncols, cols, d_keys, d_vals, records, planes);
}

namespace {
int ordered_impl(krn_ctx *ctx, double *d_target, size_t target_size, int ncols, const int *cols, const uint32_t *d_keys,
                 const double *d_vals, size_t records, int width)
{
    const bool lanes = cols != nullptr;
    KRN_REQUIRE(ctx != nullptr, "null context");
    KRN_REQUIRE(width >= 1 && width <= kMaxWidth, "width must be 1..4");
    if (records == 0 || target_size == 0) return KRN_OK;
    KRN_REQUIRE(d_target && d_keys && d_vals, "null pointer");
    KRN_REQUIRE(target_size <= 0x80000000ull, "target too large (at most 2^31 elements)");
    KRN_REQUIRE(records < 0xffffffffull, "too many records for 32-bit record numbers");

    // Buckets of 2^lb targets; `high` bits above them are sorted in HBM.  At least 2^10 buckets when
    // the target is large enough (one block per bucket must fill the machine); the all-ones key of a
    // site that did not execute must fall into a bucket beyond the last real one.  (Measured: making lb
    // as large as shared memory allows so that targets of up to 4 M elements need ONE 9-10 bit pass is
    // slower than two balanced 5-6 bit passes - 1 M targets 0.74 against 0.61 ms: a 10-bit pass ranks
    // with ten ballots, leaves the tile in runs of four records, and the fold gets a quarter of the blocks.)
    const int nbits = bit_length(target_size - 1);  // bits of the largest real key
    int lb = nbits - kMaxPassBits;
    if (lb < 0) lb = 0;
    int lb_max = kMaxLocalBits;  // a bucket's targets: 32 KB of shared memory (rows x ncols doubles: 24 KB)
    while (lanes && lb_max > 0 && (size_t(ncols) << lb_max) > 3072) --lb_max;
    if (lb > lb_max) lb = lb_max;
    int high = nbits - lb;
    if (high < 1) high = 1;
    while (((size_t(1) << high) - 1) <= ((target_size - 1) >> lb)) ++high;
    const int passes = (high + kMaxPassBits - 1) / kMaxPassBits;
    const int bits = (high + passes - 1) / passes;
    const size_t buckets = size_t(1) << (bits * passes);  // bucket ids the passes can produce
    const u32 hmask = u32(buckets - 1);
    const size_t tiles = (records + kTile - 1) / kTile;
    const size_t table_len = (size_t(1) << bits) * tiles;
    const size_t sums_len = (table_len + kScanChunk - 1) / kScanChunk;

    auto round256 = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t key_bytes = round256(records * sizeof(u32));
    const size_t val_bytes = round256(records * size_t(width) * sizeof(double));
    const int nbuf = passes > 1 ? 2 : 1;
    const size_t total = nbuf * (key_bytes + val_bytes) + round256(table_len * 4) + round256(sums_len * 4) +
                         2 * round256(buckets * 4) + 256;
    char *ws = nullptr;
    KRN_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&ws), total, ctx->stream));
    char *cursor = ws;
    u32 *key_buf[2] = {nullptr, nullptr};
    double *val_buf[2] = {nullptr, nullptr};
    for (int k = 0; k < nbuf; ++k) {
        key_buf[k] = reinterpret_cast<u32 *>(cursor);
        cursor += key_bytes;
        val_buf[k] = reinterpret_cast<double *>(cursor);
        cursor += val_bytes;
    }
    u32 *table = reinterpret_cast<u32 *>(cursor);
    cursor += round256(table_len * 4);
    u32 *sums = reinterpret_cast<u32 *>(cursor);
    cursor += round256(sums_len * 4);
    u32 *in_order = reinterpret_cast<u32 *>(cursor);  // kNone while no record has been seen out of bucket order
    cursor += 256;
    u32 *start = reinterpret_cast<u32 *>(cursor);  // (directly behind in_order: one memset sets both)
    cursor += round256(buckets * 4);
    u32 *end = reinterpret_cast<u32 *>(cursor);

    int rc = KRN_OK;
    auto fail = [&](cudaError_t e, const char *what) {
        krn_set_error("%s failed: %s", what, cudaGetErrorString(e));
        rc = KRN_E_CUDA;
    };
    cudaError_t e = cudaMemsetAsync(in_order, 0xFF, 256 + buckets * 4, ctx->stream);
    if (e != cudaSuccess) fail(e, "cudaMemsetAsync");
    const u32 *src_keys = d_keys;
    const double *src_vals = d_vals;
    for (int pass = 0; pass < passes && rc == KRN_OK; ++pass) {
        const int shift = lb + pass * bits;
        e = launch_hist(bits, unsigned(tiles), ctx->stream, src_keys, records, shift, u32(tiles), table, lb, hmask,
                        in_order, pass == 0);
        if (e != cudaSuccess) fail(e, "histogram launch");
        ctx->launches++;
        if (table_len <= size_t(kScanChunk) * 32) {
            scan_single<<<1, kThreads, 0, ctx->stream>>>(table, table_len, in_order);
            ctx->launches++;
        } else {
            scan_sums<<<unsigned(sums_len), kThreads, 0, ctx->stream>>>(table, table_len, sums, in_order);
            scan_single<<<1, kThreads, 0, ctx->stream>>>(sums, sums_len, in_order);
            scan_apply<<<unsigned(sums_len), kThreads, 0, ctx->stream>>>(table, table_len, sums, in_order);
            ctx->launches += 3;
        }
        u32 *dst_keys = key_buf[pass & 1];
        double *dst_vals = val_buf[pass & 1];
        e = launch_scatter(bits, unsigned(tiles), ctx->stream, src_keys, src_vals, dst_keys, dst_vals, table, records,
                           shift, u32(tiles), width, in_order);
        ctx->launches++;
        src_keys = dst_keys;
        src_vals = dst_vals;
        if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) fail(e, "partition pass launch");
    }
    if (rc == KRN_OK) {
        const size_t blocks = (records + 4 * kThreads - 1) / (4 * kThreads);
        ord_mark<<<unsigned(blocks), kThreads, 0, ctx->stream>>>(src_keys, d_keys, in_order, records, lb, hmask, start, end);
        const size_t tile_elems = ((size_t(lanes ? ncols : 1) << lb) + 1) & ~size_t(1);
        const size_t chunk = size_t(kThreads) * (width == 1 ? 8 : 4);
        const size_t smem = tile_elems * 8 + size_t(width) * chunk * 8 + 2 * chunk * 4 + size_t(16) * kThreads * 2;
        Cols cc;
        for (int l = 0; l < kMaxWidth; ++l) cc.c[l] = (lanes && l < width) ? cols[l] : 0;
        // real buckets only: ids beyond the last target hold sites that did not execute
        const size_t real = ((target_size - 1) >> lb) + 1;
#define KRN_FOLD(W, L)                                                                                            \
    do {                                                                                                          \
        constexpr int per = W == 1 ? 8 : 4;                                                                       \
        e = cudaFuncSetAttribute(ord_bucket_fold<W, L, per>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
        if (e == cudaSuccess)                                                                                     \
            ord_bucket_fold<W, L, per><<<unsigned(real), kThreads, smem, ctx->stream>>>(                          \
                src_keys, src_vals, d_keys, d_vals, in_order, records, d_target, target_size, ncols, cc, lb,      \
                start, end);                                                                                      \
    } while (0)
        switch (width * 2 + (lanes ? 1 : 0)) {
        case 2: KRN_FOLD(1, false); break;
        case 3: KRN_FOLD(1, true); break;
        case 4: KRN_FOLD(2, false); break;
        case 5: KRN_FOLD(2, true); break;
        case 6: KRN_FOLD(3, false); break;
        case 7: KRN_FOLD(3, true); break;
        case 8: KRN_FOLD(4, false); break;
        default: KRN_FOLD(4, true); break;
        }
#undef KRN_FOLD
        ctx->launches += 2;
        if (e != cudaSuccess || (e = cudaGetLastError()) != cudaSuccess) fail(e, "fold launch");
    }
    cudaFreeAsync(ws, ctx->stream);
    return rc;
}
}  // namespace
