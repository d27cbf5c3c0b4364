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
//     key[r]            = flat offset of the target element (uint32)
//     val[r*width + w]  = the values of the group's sites, program order
// at r = iteration * groups + group, so record order IS the reference's queue
// order.  krn_ordered_accumulate then
//   1. sorts (key, r) by key with a STABLE least-significant-digit radix sort
//      (per pass: per-tile digit histogram -> exclusive scan of the
//      [digit][tile] table -> scatter that ranks equal digits in tile order,
//      through shared memory so that runs leave the SM coalesced),
//   2. folds every run of equal keys, in order, starting from the target's
//      current value, and stores the result with ONE plain store per location.
// No atomics on the target, nothing depends on the schedule: the result is
// bit-identical to the reference and identical from run to run.  Runs longer
// than kLongAfter records (a hot location) are folded by a whole block that
// streams the values through shared memory ahead of the one thread adding
// them; the chain of dependent fp64 additions itself is the definition of the
// result and cannot be shortened.
//
// All kernels are HBM-bound integer/byte work (no tensor-core shape): per pass
// 4 B/record (histogram) + 8 B read + 8 B written; the fold reads 8 B/record of
// (key, r), gathers the values (one 32 B sector per record) and updates the
// target in ascending address order.
#include "krn_common.cuh"
#include "krn_prelude.cuh"

namespace {

typedef unsigned int u32;

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItems = 16;                 // records per thread and tile
constexpr int kTile = kThreads * kItems;   // 4096 records: 32 KB of (key, r) in shared memory
constexpr int kWarpSpan = 32 * kItems;     // consecutive records ranked by one warp
constexpr int kScanChunk = kThreads * 8;
constexpr int kLongAfter = 64;             // a run still open after this many records goes to a block
constexpr int kLongChunk = 1024;           // records a block stages per round of the long fold
constexpr int kMaxWidth = 4;

__device__ __forceinline__ u32 lanemask_lt()
{
    u32 m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// Lanes of the warp holding the same `bits`-bit digit as the caller (valid lanes only): one ballot per
// bit.  (match.any does the same in one instruction but its cost grows with the number of distinct
// values in the warp - measured here: 166 us per 16.7 M-record pass against ballots' constant time.)
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

// ---- pass step 1: digit histogram of every tile ---------------------------------------
// table[digit * tiles + tile]: scanned in this order it yields, for every (digit, tile), the
// number of records with a smaller digit anywhere plus those with the same digit in earlier
// tiles - the stable destination of the tile's first record with that digit.
template <int BITS>
__global__ void __launch_bounds__(kThreads)
ord_hist(const u32 *__restrict__ keys, size_t m, int shift, u32 tiles, u32 *__restrict__ table)
{
    // per-warp counters, bumped by the lowest lane of every group of equal digits with a plain
    // read-modify-write: shared-memory atomics cost 2 cycles per lane and would bound the pass
    constexpr u32 mask = (1u << BITS) - 1u;
    __shared__ u32 s_cnt[kWarps][1 << BITS];
    for (int k = threadIdx.x; k < kWarps << BITS; k += kThreads) (&s_cnt[0][0])[k] = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = size_t(blockIdx.x) * kTile + size_t(warp) * kWarpSpan;
    u32 key[kItems];
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const size_t p = base + size_t(r) * 32 + lane;
        key[r] = p < m ? keys[p] : 0u;
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
    if (threadIdx.x <= mask) {
        u32 total = 0;
#pragma unroll
        for (int w = 0; w < kWarps; ++w) total += s_cnt[w][threadIdx.x];
        table[size_t(threadIdx.x) * tiles + blockIdx.x] = total;
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
__global__ void __launch_bounds__(kThreads) scan_single(u32 *data, size_t count)
{
    u32 carry = 0;
    for (size_t base = 0; base < count; base += kScanChunk) {
        u32 x[8];
        const size_t first = base + size_t(threadIdx.x) * 8;
        load8(data, first, count, x);
        carry += block_scan8(x, carry);
        store8(data, first, count, x);
    }
}

__global__ void __launch_bounds__(kThreads) scan_sums(const u32 *__restrict__ data, size_t count, u32 *__restrict__ sums)
{
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

__global__ void __launch_bounds__(kThreads) scan_apply(u32 *data, size_t count, const u32 *__restrict__ sums)
{
    const size_t first = size_t(blockIdx.x) * kScanChunk + size_t(threadIdx.x) * 8;
    u32 x[8];
    load8(data, first, count, x);
    block_scan8(x, sums[blockIdx.x]);
    store8(data, first, count, x);
}

// ---- pass step 3: stable scatter ------------------------------------------------------------
// Warp w of the tile ranks records [w*512, (w+1)*512) of the tile, 32 consecutive records per
// round: lanes with the same digit find each other (match.any); their rank within the round is
// the number of lower lanes among them, and the warp's running count of the digit (shared
// memory, updated by the lowest lane) orders the rounds.  Tile order = (warp, round, lane), so
// equal digits keep their input order.  The records are then placed in shared memory in digit
// order and leave the tile as runs of consecutive destinations.
template <int BITS>
__global__ void __launch_bounds__(kThreads)
ord_scatter(const u32 *__restrict__ keys_in, const u32 *__restrict__ idx_in, u32 *__restrict__ keys_out,
            u32 *__restrict__ idx_out, const u32 *__restrict__ table, size_t m, int shift, u32 tiles)
{
    constexpr u32 mask = (1u << BITS) - 1u;
    constexpr int kRadix = 1 << BITS;
    __shared__ u32 s_cnt[kWarps][kRadix];  // per-warp digit counts, then the warp's first slot of the digit in the tile
    __shared__ u32 s_first[kRadix];        // first slot of the digit in the sorted tile
    __shared__ u32 s_dest[kRadix];         // global destination of that slot
    __shared__ u32 s_key[kTile];
    __shared__ u32 s_idx[kTile];
    __shared__ u32 s_wsum[kWarps];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const size_t base = size_t(blockIdx.x) * kTile;
    const u32 live = u32(m - base < size_t(kTile) ? m - base : size_t(kTile));  // records of this tile
    for (int k = threadIdx.x; k < kWarps * kRadix; k += kThreads) (&s_cnt[0][0])[k] = 0;
    __syncthreads();

    u32 key[kItems], idx[kItems];
    unsigned short rank[kItems];
    const u32 lt = lanemask_lt();
#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const u32 t = u32(warp) * kWarpSpan + u32(r) * 32 + lane;  // position in the tile
        const bool valid = t < live;
        key[r] = valid ? keys_in[base + t] : 0xffffffffu;
        idx[r] = valid ? (idx_in != nullptr ? idx_in[base + t] : u32(base + t)) : 0u;
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
            before = s_cnt[warp][d];
            s_cnt[warp][d] = before + (u32)__popc(peers);
        }
        before = __shfl_sync(KRN_FULL_MASK, before, leader);
        rank[r] = (unsigned short)(before + (u32)__popc(peers & lt));
        __syncwarp();  // the next round's leader of this digit may be another lane
    }
    __syncthreads();

    // per digit: exclusive prefix over the warps, tile total, then an exclusive scan over the digits
    const u32 d_me = threadIdx.x;  // kThreads >= kRadix
    u32 total = 0;
    if (d_me <= mask) {
#pragma unroll
        for (int w = 0; w < kWarps; ++w) {
            const u32 c = s_cnt[w][d_me];
            s_cnt[w][d_me] = total;
            total += c;
        }
    }
    u32 inc = total;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const u32 t = __shfl_up_sync(KRN_FULL_MASK, inc, o);
        if (lane >= o) inc += t;
    }
    if (lane == 31) s_wsum[warp] = inc;
    __syncthreads();
    u32 wbase = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w)
        if (w < warp) wbase += s_wsum[w];
    if (d_me <= mask) {
        const u32 first = wbase + inc - total;
        s_first[d_me] = first;
        s_dest[d_me] = table[size_t(d_me) * tiles + blockIdx.x];
    }
    __syncthreads();

#pragma unroll
    for (int r = 0; r < kItems; ++r) {
        const u32 t = u32(warp) * kWarpSpan + u32(r) * 32 + lane;
        if (t < live) {
            const u32 d = (key[r] >> shift) & mask;
            const u32 slot = s_first[d] + s_cnt[warp][d] + rank[r];
            s_key[slot] = key[r];
            s_idx[slot] = idx[r];
        }
    }
    __syncthreads();
    for (u32 s = threadIdx.x; s < live; s += kThreads) {
        const u32 k = s_key[s];
        const u32 d = (k >> shift) & mask;
        const size_t g = size_t(s_dest[d]) + (s - s_first[d]);
        keys_out[g] = k;
        idx_out[g] = s_idx[s];
    }
}

// ---- fold --------------------------------------------------------------------------------------
// One thread per sorted position; the thread at the head of a run of equal keys folds the run in
// order, from the target's current value:  acc = target; acc += v(r0, 0); acc += v(r0, 1); ...
__global__ void __launch_bounds__(kThreads)
ord_fold(const u32 *__restrict__ keys, const u32 *__restrict__ idx, const double *__restrict__ vals, int width,
         size_t m, double *target, u32 target_size, u32 *long_list, u32 *long_count)
{
    const size_t p = size_t(blockIdx.x) * kThreads + threadIdx.x;
    if (p >= m) return;
    const u32 key = keys[p];
    if (key >= target_size) return;  // a site that did not execute
    if (p > 0 && keys[p - 1] == key) return;
    double acc = target[key];
    size_t q = p;
    for (int step = 0; step < kLongAfter; ++step) {
        const size_t r = idx[q];
        for (int w = 0; w < width; ++w) acc = acc + vals[r * width + w];
        ++q;
        if (q >= m || keys[q] != key) {
            target[key] = acc;
            return;
        }
    }
    long_list[atomicAdd(long_count, 1u)] = u32(p);  // restarted from the beginning by a block
}

// Long runs: the block stages kLongChunk records per round in shared memory - the loads of the
// next round are in flight while thread 0 adds the current one - and thread 0 performs the fold.
__global__ void __launch_bounds__(kThreads)
ord_fold_long(const u32 *__restrict__ keys, const u32 *__restrict__ idx, const double *__restrict__ vals, int width,
              size_t m, double *target, const u32 *__restrict__ long_list, const u32 *__restrict__ long_count)
{
    __shared__ double s_v[kLongChunk * kMaxWidth];
    constexpr int kPer = kLongChunk / kThreads;
    const u32 runs = *long_count;
    for (u32 s = blockIdx.x; s < runs; s += gridDim.x) {
        const size_t p = long_list[s];
        const u32 key = keys[p];
        double acc = threadIdx.x == 0 ? target[key] : 0.0;
        double v[kPer][kMaxWidth];
        bool same[kPer];
        size_t q0 = p;
        auto fetch = [&](size_t from) {
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                const size_t q = from + threadIdx.x + size_t(j) * kThreads;
                same[j] = q < m && keys[q] == key;
                if (same[j]) {
                    const size_t r = idx[q];
#pragma unroll
                    for (int w = 0; w < kMaxWidth; ++w)
                        if (w < width) v[j][w] = vals[r * width + w];
                }
            }
        };
        fetch(q0);
        for (;;) {
            int count = 0;
#pragma unroll
            for (int j = 0; j < kPer; ++j) {
                if (same[j]) {
#pragma unroll
                    for (int w = 0; w < kMaxWidth; ++w)
                        if (w < width) s_v[(threadIdx.x + j * kThreads) * width + w] = v[j][w];
                }
                count += __syncthreads_count(same[j]);
            }
            q0 += kLongChunk;
            const bool more = count == kLongChunk && q0 < m;  // sorted keys: the run is a prefix of the chunk
            if (more) fetch(q0);
            if (threadIdx.x == 0) {
                const int terms = count * width;
#pragma unroll 8
                for (int k = 0; k < terms; ++k) acc = acc + s_v[k];
            }
            __syncthreads();
            if (!more) break;
        }
        if (threadIdx.x == 0) target[key] = acc;
    }
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
    default: CALL(8); break;        \
    }

void launch_hist(int bits, unsigned tiles, cudaStream_t st, const u32 *keys, size_t m, int shift, u32 ntiles, u32 *table)
{
#define KRN_CALL(B) ord_hist<B><<<tiles, kThreads, 0, st>>>(keys, m, shift, ntiles, table)
    KRN_BITS_SWITCH(bits, KRN_CALL)
#undef KRN_CALL
}

void launch_scatter(int bits, unsigned tiles, cudaStream_t st, const u32 *keys_in, const u32 *idx_in, u32 *keys_out,
                    u32 *idx_out, const u32 *table, size_t m, int shift, u32 ntiles)
{
#define KRN_CALL(B) ord_scatter<B><<<tiles, kThreads, 0, st>>>(keys_in, idx_in, keys_out, idx_out, table, m, shift, ntiles)
    KRN_BITS_SWITCH(bits, KRN_CALL)
#undef KRN_CALL
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

extern "C" int krn_ordered_accumulate(krn_ctx *ctx, double *d_target, size_t target_size, const uint32_t *d_keys,
                                      const double *d_vals, size_t records, int width)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    KRN_REQUIRE(width >= 1 && width <= kMaxWidth, "width must be 1..4");
    if (records == 0 || target_size == 0) return KRN_OK;
    KRN_REQUIRE(d_target && d_keys && d_vals, "null pointer");
    KRN_REQUIRE(target_size < 0xffffffffull, "target too large for 32-bit keys");
    KRN_REQUIRE(records < 0xffffffffull, "too many records for 32-bit record numbers");

    // keys 0..target_size-1 and the all-ones mark of a site that did not execute must stay apart
    // in the bits that are sorted: bit_length(target_size) bits, split evenly over the passes
    const int nbits = bit_length(target_size);
    const int passes = (nbits + 7) / 8;
    const int bits = (nbits + passes - 1) / passes;
    const u32 mask = (1u << bits) - 1u;
    const size_t tiles = (records + kTile - 1) / kTile;
    const size_t table_len = (size_t(mask) + 1) * tiles;
    const size_t sums_len = (table_len + kScanChunk - 1) / kScanChunk;
    const size_t long_cap = records / kLongAfter + 1;

    auto round256 = [](size_t b) { return (b + 255) / 256 * 256; };
    const size_t rec_bytes = round256(records * sizeof(u32));
    const size_t total = 4 * rec_bytes + round256(table_len * 4) + round256(sums_len * 4) + round256(long_cap * 4) + 256;
    char *ws = nullptr;
    KRN_CUDA(cudaMallocAsync(reinterpret_cast<void **>(&ws), total, ctx->stream));
    u32 *key_buf[2] = {reinterpret_cast<u32 *>(ws), reinterpret_cast<u32 *>(ws + rec_bytes)};
    u32 *idx_buf[2] = {reinterpret_cast<u32 *>(ws + 2 * rec_bytes), reinterpret_cast<u32 *>(ws + 3 * rec_bytes)};
    char *cursor = ws + 4 * rec_bytes;
    u32 *table = reinterpret_cast<u32 *>(cursor);
    cursor += round256(table_len * 4);
    u32 *sums = reinterpret_cast<u32 *>(cursor);
    cursor += round256(sums_len * 4);
    u32 *long_list = reinterpret_cast<u32 *>(cursor);
    cursor += round256(long_cap * 4);
    u32 *long_count = reinterpret_cast<u32 *>(cursor);

    int rc = KRN_OK;
    auto fail = [&](cudaError_t e, const char *what) {
        krn_set_error("%s failed: %s", what, cudaGetErrorString(e));
        rc = KRN_E_CUDA;
    };
    const u32 *src_keys = d_keys;
    const u32 *src_idx = nullptr;
    cudaError_t e = cudaMemsetAsync(long_count, 0, sizeof(u32), ctx->stream);
    if (e != cudaSuccess) fail(e, "cudaMemsetAsync");
    for (int pass = 0; pass < passes && rc == KRN_OK; ++pass) {
        const int shift = pass * bits;
        launch_hist(bits, unsigned(tiles), ctx->stream, src_keys, records, shift, u32(tiles), table);
        ctx->launches++;
        if (table_len <= size_t(kScanChunk) * 32) {
            scan_single<<<1, kThreads, 0, ctx->stream>>>(table, table_len);
            ctx->launches++;
        } else {
            scan_sums<<<unsigned(sums_len), kThreads, 0, ctx->stream>>>(table, table_len, sums);
            scan_single<<<1, kThreads, 0, ctx->stream>>>(sums, sums_len);
            scan_apply<<<unsigned(sums_len), kThreads, 0, ctx->stream>>>(table, table_len, sums);
            ctx->launches += 3;
        }
        u32 *dst_keys = key_buf[pass & 1], *dst_idx = idx_buf[pass & 1];
        launch_scatter(bits, unsigned(tiles), ctx->stream, src_keys, src_idx, dst_keys, dst_idx, table, records, shift,
                       u32(tiles));
        ctx->launches++;
        src_keys = dst_keys;
        src_idx = dst_idx;
        if ((e = cudaGetLastError()) != cudaSuccess) fail(e, "radix pass launch");
    }
    if (rc == KRN_OK) {
        const size_t blocks = (records + kThreads - 1) / kThreads;
        ord_fold<<<unsigned(blocks), kThreads, 0, ctx->stream>>>(src_keys, src_idx, d_vals, width, records, d_target,
                                                                u32(target_size), long_list, long_count);
        ord_fold_long<<<unsigned(ctx->sms * 2), kThreads, 0, ctx->stream>>>(src_keys, src_idx, d_vals, width, records,
                                                                            d_target, long_list, long_count);
        ctx->launches += 2;
        if ((e = cudaGetLastError()) != cudaSuccess) fail(e, "fold launch");
    }
    cudaFreeAsync(ws, ctx->stream);
    return rc;
}
