/* krn_b200.h - C ABI of libkrn_b200.so, the B200 (sm_100a) execution path for
 * kernel-language programs: device-resident fp64 Views, the bulk builtins,
 * the fused headline objective/gradient kernels, and a loader for generated
 * parallel_for kernels.
 *
 * The reference package has no FFI: its data path is the Python function
 * `execute(program, fn_name, inputs, cfg)` (reference
 * pkg/src/krn/runtime.py:689-706) and the per-statement numpy operations
 * underneath it.  Each entry point below names the reference operation it
 * replaces.  A reference maintainer binds this header with ctypes
 * (INTEGRATION.md shows the stub); this repo's own binding is
 * paper_2507_13204_b200/_cabi.py.
 *
 * Conventions
 *  - every function returns 0 on success, a KRN_E_* code otherwise;
 *    krn_last_error() gives the message of the calling thread's last failure
 *  - plain pointers and sizes only; `double*` arguments named d_* are DEVICE
 *    pointers, h_* are HOST pointers
 *  - all work is enqueued on the context's CUDA stream and is asynchronous
 *    unless the description says "synchronous"
 *  - fp64 IEEE arithmetic, no FMA contraction (reference SPEC.md:391)
 *  - vectorised paths need 32-byte aligned device pointers (anything from
 *    krn_alloc is 256-byte aligned); unaligned pointers take a scalar path
 */
#ifndef KRN_B200_H
#define KRN_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define KRN_OK 0
#define KRN_E_CUDA 1          /* a CUDA runtime/driver call failed            */
#define KRN_E_ARG 2           /* bad argument                                 */
#define KRN_E_NVRTC 3         /* runtime compilation failed (log in message)  */
#define KRN_E_UNAVAILABLE 4   /* libcuda / libnvrtc could not be loaded       */

/* device status codes written by kernels into the context's status word */
#define KRN_ST_OK 0
#define KRN_ST_OUT_OF_BOUNDS 1   /* reference: OutOfBounds, runtime.py:299-321 */
#define KRN_ST_BAD_INDEX 2       /* NaN/Inf used as an index (int() raises in the reference, runtime.py:335) */

typedef struct krn_ctx krn_ctx;
typedef struct krn_module krn_module;

/* ---- context ------------------------------------------------------------ */

const char *krn_last_error(void);
const char *krn_version(void);
int krn_device_count(int *count);

/* One executor context: a device, a non-blocking stream, a stream-ordered
 * memory pool, a reduction workspace, a status word and scalar slots.
 * Replaces _Interpreter.__init__ (runtime.py:454-466).  `cuda_stream` may be 0
 * (a private stream is created) or an existing cudaStream_t to share. */
int krn_ctx_create(int device, void *cuda_stream, krn_ctx **out);
int krn_ctx_destroy(krn_ctx *ctx);
int krn_sync(krn_ctx *ctx);                    /* synchronous */
int krn_ctx_stream(krn_ctx *ctx, void **cuda_stream);
int krn_ctx_sm_count(krn_ctx *ctx, int *sms);
/* number of kernels this library has launched on the context so far */
int krn_ctx_launch_count(krn_ctx *ctx, uint64_t *launches);

/* ---- View storage (reference: ViewStorage, runtime.py:74-115) ------------ */

int krn_alloc(krn_ctx *ctx, size_t bytes, void **d_ptr);   /* stream-ordered, 256 B aligned */
int krn_free(krn_ctx *ctx, void *d_ptr);
int krn_host_alloc(size_t bytes, void **h_ptr);            /* pinned host memory */
int krn_host_free(void *h_ptr);
int krn_upload(krn_ctx *ctx, void *d_dst, const void *h_src, size_t bytes);    /* async if h_src pinned */
int krn_download(krn_ctx *ctx, void *h_dst, const void *d_src, size_t bytes);  /* synchronous */
int krn_download_async(krn_ctx *ctx, void *h_dst, const void *d_src, size_t bytes);

/* ---- events (device-side timing of the launch sequence; bench_ratio's
 *      perf_counter pair, verify.py:297-306) -------------------------------- */
int krn_event_create(void **event);
int krn_event_destroy(void *event);
int krn_event_record(krn_ctx *ctx, void *event);
int krn_event_elapsed_ms(void *start, void *stop, float *ms);   /* synchronous on stop */

/* ---- auxiliary copy streams: overlap host<->device transfers of one chunk of
 *      rows with the kernels of another (the host-buffer path of execute();
 *      the reference has no counterpart, its Views are host arrays) ------------- */
int krn_stream_create(krn_ctx *ctx, void **stream);
int krn_stream_destroy(void *stream);
int krn_stream_sync(void *stream);                                   /* synchronous */
int krn_upload_on(void *stream, void *d_dst, const void *h_src, size_t bytes);
int krn_download_on(void *stream, void *h_dst, const void *d_src, size_t bytes);
int krn_event_record_on(void *stream, void *event);
int krn_stream_wait_event(void *stream, void *event);
int krn_ctx_wait_event(krn_ctx *ctx, void *event);   /* the context's stream waits */

/* ---- bulk builtins --------------------------------------------------------- */

/* deep_copy(dst, scalar) and DeclView zero-fill   (runtime.py:637-639, 523-535); the
 * scalar is read from device memory at *d_value when d_value != NULL */
int krn_fill(krn_ctx *ctx, double *d_v, size_t n, double value, const double *d_value);
/* deep_copy(dst, src)                              (runtime.py:630-636) */
int krn_copy(krn_ctx *ctx, double *d_dst, const double *d_src, size_t n);
/* parallel_sum(dst_view, scalar): v[i] += s        (runtime.py:662-663); the
 * scalar is read from device memory at *d_s when d_s != NULL, else `s` is used */
int krn_add_scalar(krn_ctx *ctx, double *d_v, size_t n, double s, const double *d_s);
/* parallel_sum(dst_view, src_view): dst[i] += src[i]   (runtime.py:655-661) */
int krn_add_view(krn_ctx *ctx, double *d_dst, const double *d_src, size_t n);
/* dst = parallel_sum(src): *d_out = (accumulate ? *d_out : 0.0) + tree(v)
 * with the reference's adjacent-pair tree, +0.0 padding of odd levels,
 * bit-identical for any n               (pairwise_sum, runtime.py:166-177; gather, 643-651) */
int krn_reduce_pairwise(krn_ctx *ctx, const double *d_v, size_t n, double *d_out, int accumulate);
/* check_finite: *d_flag |= 1 when any element is NaN/Inf   (runtime.py:669-676) */
int krn_check_finite(krn_ctx *ctx, const double *d_v, size_t n, int *d_flag);

/* ---- deferred atomic_add, applied in the reference's order ---------------------------
 * The reference queues every atomic_add of a kernel and applies the queue sorted by
 * (iteration, program order): `flat[offset] += value`, one after the other
 * (runtime.py:430-447, 615-620) - each location is a left fold in a fixed order, hence
 * bit-reproducible.  krn_ordered_accumulate does exactly that for `records` queue entries that
 * are ALREADY in queue order (record r = iteration * groups + group):
 *     d_target[d_keys[r]] += d_vals[0*records + r]; ... += d_vals[(width-1)*records + r];
 * (values are planes of `records` doubles).  Records are partitioned stably by target bucket
 * (radix passes in HBM), each bucket is folded in order inside shared memory, and every
 * location is written with one plain store: no atomics, identical bits on every run.  A key
 * must be < target_size or all ones (krn_memset the key array to 0xFF first): the mark of a
 * site that did not execute.  target_size <= 2^31, records < 2^32 - 1, width 1..4. */
int krn_ordered_accumulate(krn_ctx *ctx, double *d_target, size_t target_size, const uint32_t *d_keys,
                           const double *d_vals, size_t records, int width);
/* The same for a rows x ncols target whose records name a ROW (key) and carry one value per plane for
 * the literal column cols[l] of that row (sites atomic_add(v(r, c0), .), atomic_add(v(r, c1), .), ... of
 * one iteration travel as ONE record): d_target[key*ncols + cols[l]] += d_vals[l*records + r].
 * rows <= 2^31, planes 1..4. */
int krn_ordered_accumulate_rows(krn_ctx *ctx, double *d_target, size_t rows, int ncols, const int *cols, int planes,
                                const uint32_t *d_keys, const double *d_vals, size_t records);
/* cudaMemsetAsync on the context's stream */
int krn_memset(krn_ctx *ctx, void *d_ptr, int byte, size_t bytes);

/* ---- headline objective: normRes1DLaplacianSQ and its generated gradient ----
 * (programs/laplacian.krn; gradient text tests/test_adjoint.py:43-94)
 *
 * One launch each.  `d_x_in` is read, the scaled view 3*x is written to
 * `d_x_out`, which must be a different buffer (the caller swaps the View's
 * storage: an in-place scale would race with the stencil's neighbour reads).
 *
 * Sharding: the kernels process rows [offset, offset + n_local) of a global
 * problem of n_global rows.  d_halo (6 doubles, may be NULL when the shard is
 * the whole problem) holds the ORIGINAL values x[offset-2], x[offset-1],
 * b[offset-1], x[offset+n_local], x[offset+n_local+1], b[offset+n_local];
 * entries outside [0, n_global) are ignored.
 */

/* *d_f = (accumulate ? *d_f : 0.0) + tree(y2) over the local rows.  Bit-identical
 * to the reference when the shard is the whole problem (or, sharded, when
 * offset is a multiple of krn_laplacian_partial_span() and the caller combines
 * the per-block partials in tree order). */
int krn_laplacian_primal(krn_ctx *ctx, const double *d_x_in, double *d_x_out, const double *d_b,
                         size_t n_local, size_t offset, size_t n_global, const double *d_halo,
                         double *d_f, int accumulate);

/* Accumulates the gradient into d_dx / d_db (element-wise read-modify-write).
 * `dx_zero` / `db_zero` != 0 promise that the shadow currently holds +0.0
 * everywhere (ViewStorage.zeros provenance): its read is skipped.  d_db may be
 * NULL when b is not differentiated, d_dx may be NULL when x is not.
 * `seed` is the literal of the generated `_d_sum += seed` statement. */
int krn_laplacian_grad(krn_ctx *ctx, const double *d_x_in, double *d_x_out, const double *d_b,
                       double *d_dx, double *d_db, int dx_zero, int db_zero,
                       size_t n_local, size_t offset, size_t n_global, const double *d_halo,
                       double seed);

/* number of consecutive rows folded into one tree partial by the primal kernel
 * at this problem size (a power of two) */
size_t krn_laplacian_partial_span(size_t n_global);

/* Copies the per-block tree partials of the LAST krn_laplacian_primal launch on this
 * context - ceil(n_local / span) doubles in block order, each the exact node of the
 * reference's tree (pairwise_sum, runtime.py:166-177) over its aligned span of rows - to
 * d_out (device memory), on the context's stream.  Sharded mode: the partials of all shards,
 * concatenated in rank order and folded with krn_reduce_pairwise, give the objective
 * bit-identical to the single-device (and the reference's) result for any number of shards. */
int krn_laplacian_partials(krn_ctx *ctx, double *d_out, size_t count);

/* ---- sharded mode without per-step collectives: peer memory ---------------------------
 * (the reference has no counterpart: its thread pool shares one address space,
 * runtime.py:594-613.)  A rank exports the device allocations holding its x and b once
 * (krn_ipc_export: the 64-byte CUDA IPC handle of the allocation containing d_ptr and d_ptr's
 * offset inside it), hands the 72 bytes to its neighbours by any means (one all_gather at set-up),
 * and each neighbour maps it (krn_ipc_open: peer access over NVLink is enabled by the mapping;
 * two processes on one device work too).  The *_peers kernels then read their halo rows straight
 * from the neighbours' buffers:
 *   d_x_prev_end / d_b_prev_end  one past the LAST row of the previous shard's x / b
 *                                (NULL when offset == 0)
 *   d_x_next / d_b_next          the FIRST row of the next shard's x / b
 *                                (NULL when offset + n_local == n_global)
 * A gradient step is then exactly one launch and no collective.  The caller fences (a barrier
 * across the ranks) only when a neighbour has rewritten the rows being read. */
int krn_ipc_export(krn_ctx *ctx, const void *d_ptr, unsigned char handle[64], size_t *offset);
int krn_ipc_open(krn_ctx *ctx, const unsigned char handle[64], size_t offset, void **d_base, void **d_ptr);
int krn_ipc_close(krn_ctx *ctx, void *d_base);   /* synchronous */
int krn_laplacian_primal_peers(krn_ctx *ctx, const double *d_x_in, double *d_x_out, const double *d_b,
                               size_t n_local, size_t offset, size_t n_global,
                               const double *d_x_prev_end, const double *d_b_prev_end,
                               const double *d_x_next, const double *d_b_next, double *d_f, int accumulate);
int krn_laplacian_grad_peers(krn_ctx *ctx, const double *d_x_in, double *d_x_out, const double *d_b,
                             double *d_dx, double *d_db, int dx_zero, int db_zero, size_t n_local,
                             size_t offset, size_t n_global, const double *d_x_prev_end,
                             const double *d_b_prev_end, const double *d_x_next, const double *d_b_next,
                             double seed);

/* ---- generated kernels (parallel_for bodies compiled from the program tree;
 *      replaces _Compiler/_Interpreter.parallel_for, runtime.py:230-447, 567-624)
 * `cuda_source` is CUDA C++ for sm_100a; it may #include "krn_prelude.cuh"
 * (shipped inside the library).  Compiled with --fmad=false.  Compiled images are
 * cached on disk under $KRN_CACHE_DIR (default ~/.cache/krn_b200; empty = off),
 * keyed by source, prelude, options and NVRTC version. */
int krn_module_compile(krn_ctx *ctx, const char *cuda_source, krn_module **out);
/* which run-time compiler the process ended up with (a Python environment may have loaded an older
 * libnvrtc first) and whether generated kernels use the 256-bit accesses (PTX ISA 8.8, NVRTC >= 12.9) */
int krn_jit_info(int *nvrtc_major, int *nvrtc_minor, int *ld256);
int krn_module_destroy(krn_module *m);
/* launch `name` over `n_iterations` (grid sized by the library: a multiple of
 * the SM count); args = array of pointers to the kernel's arguments */
int krn_module_launch(krn_ctx *ctx, krn_module *m, const char *name, size_t n_iterations,
                      size_t shared_bytes, void **args);
/* launch `name` with exactly `blocks` x `threads_per_block` (tile kernels of fused statement
 * groups: one thread per 4 iterations, and block-level reductions that need every thread; 1 x 1 runs
 * a parallel_for kernel's iterations in order on one thread, for kernels whose result depends on it) */
int krn_module_launch_exact(krn_ctx *ctx, krn_module *m, const char *name, size_t blocks,
                            unsigned threads_per_block, size_t shared_bytes, void **args);
/* registers per thread, local (stack / spill) bytes per thread and static shared memory of a compiled
 * kernel: the host retunes generated kernels with them (occupancy bound of window kernels) */
int krn_module_kernel_info(krn_module *m, const char *name, int *registers, int *local_bytes,
                           int *static_shared_bytes);
/* shared_bytes: dynamic shared memory (<= 48 KB), used by the shared-memory-privatised
 * accumulation policy of atomic_add targets with few rows */

/* ---- status word: 8 x int64 {code, line, view id, index0, index1, 0, 0, 0} of the
 *      first failing access (first error wins) ---- */
int krn_status_reset(krn_ctx *ctx);

/* Start of one execute(): clears the status word AND the context's function-scope scalar slots
 * (reference: `self.scalars = {}` per run, runtime.py:468-479) with a single memset, and returns
 * the slot array (doubles, device memory, owned by the context; `capacity` slots). */
int krn_run_begin(krn_ctx *ctx, double **d_slots, size_t *capacity);

/* The context's reduction workspace for generated kernels that fold a parallel_sum into their
 * epilogue (partials + scratch of at least `blocks` doubles each, arrival ticket kept at zero
 * between launches): no per-launch allocation.  Valid until the next call that needs more. */
int krn_reduce_workspace(krn_ctx *ctx, size_t blocks, double **d_partials, double **d_scratch,
                         unsigned int **d_ticket);
int krn_status_device_ptr(krn_ctx *ctx, long long **d_status);
int krn_status_read(krn_ctx *ctx, long long h_status[8]);      /* synchronous */

#ifdef __cplusplus
}
#endif
#endif /* KRN_B200_H */
