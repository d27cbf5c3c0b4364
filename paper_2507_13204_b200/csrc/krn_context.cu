// Context, View storage, transfers, events, status word.
#include "krn_common.cuh"

static thread_local char g_error[4096] = "";

void krn_set_error(const char *fmt, ...)
{
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_error, sizeof(g_error), fmt, ap);
    va_end(ap);
}

extern "C" const char *krn_last_error(void) { return g_error; }
extern "C" const char *krn_version(void) { return "krn_b200 0.1 (sm_100a)"; }

extern "C" int krn_device_count(int *count)
{
    KRN_REQUIRE(count != nullptr, "null output");
    *count = 0;
    cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
        *count = 0;
        krn_set_error("cudaGetDeviceCount failed: %s", cudaGetErrorString(e));
        return KRN_E_CUDA;
    }
    return KRN_OK;
}

extern "C" int krn_ctx_create(int device, void *cuda_stream, krn_ctx **out)
{
    KRN_REQUIRE(out != nullptr, "null output");
    *out = nullptr;
    KRN_CUDA(cudaSetDevice(device));
    krn_ctx *ctx = new krn_ctx();
    ctx->device = device;
    cudaDeviceProp prop;
    KRN_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        krn_set_error("device %d is sm_%d%d; this library is built for sm_100a only", device, prop.major,
                      prop.minor);
        delete ctx;
        return KRN_E_ARG;
    }
    ctx->sms = prop.multiProcessorCount;
    if (cuda_stream != nullptr) {
        ctx->stream = static_cast<cudaStream_t>(cuda_stream);
    } else {
        KRN_CUDA(cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking));
        ctx->own_stream = true;
    }
    // stream-ordered pool that keeps freed blocks cached: View allocation inside
    // a timed region must not hit the driver
    KRN_CUDA(cudaDeviceGetDefaultMemPool(&ctx->pool, device));
    uint64_t keep = UINT64_MAX;
    KRN_CUDA(cudaMemPoolSetAttribute(ctx->pool, cudaMemPoolAttrReleaseThreshold, &keep));
    KRN_CUDA(cudaMalloc(&ctx->d_ticket, sizeof(unsigned int)));
    KRN_CUDA(cudaMemset(ctx->d_ticket, 0, sizeof(unsigned int)));
    // one block: [status: 8 x int64][scalar slots: KRN_SCALAR_SLOTS doubles], reset by ONE memset
    KRN_CUDA(cudaMalloc(&ctx->d_status, (8 + KRN_SCALAR_SLOTS) * 8));
    KRN_CUDA(cudaMemset(ctx->d_status, 0, (8 + KRN_SCALAR_SLOTS) * 8));
    int rc = krn_reserve_partials(ctx, 4096);
    if (rc) return rc;
    *out = ctx;
    return KRN_OK;
}

extern "C" int krn_ctx_destroy(krn_ctx *ctx)
{
    if (ctx == nullptr) return KRN_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    cudaFree(ctx->d_partials);
    cudaFree(ctx->d_ticket);
    cudaFree(ctx->d_status);
    if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
    delete ctx;
    return KRN_OK;
}

int krn_reserve_partials(krn_ctx *ctx, size_t count)
{
    if (count <= ctx->partial_capacity) return KRN_OK;
    size_t cap = ctx->partial_capacity ? ctx->partial_capacity : 4096;
    while (cap < count) cap *= 2;
    KRN_CUDA(cudaStreamSynchronize(ctx->stream));
    if (ctx->d_partials) KRN_CUDA(cudaFree(ctx->d_partials));
    ctx->d_partials = nullptr;
    ctx->partial_capacity = 0;
    KRN_CUDA(cudaMalloc(&ctx->d_partials, 2 * cap * sizeof(double)));
    ctx->partial_capacity = cap;
    return KRN_OK;
}

extern "C" int krn_sync(krn_ctx *ctx)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    KRN_CUDA(cudaStreamSynchronize(ctx->stream));
    return KRN_OK;
}

extern "C" int krn_ctx_stream(krn_ctx *ctx, void **cuda_stream)
{
    KRN_REQUIRE(ctx && cuda_stream, "null argument");
    *cuda_stream = ctx->stream;
    return KRN_OK;
}

extern "C" int krn_ctx_sm_count(krn_ctx *ctx, int *sms)
{
    KRN_REQUIRE(ctx && sms, "null argument");
    *sms = ctx->sms;
    return KRN_OK;
}

extern "C" int krn_ctx_launch_count(krn_ctx *ctx, uint64_t *launches)
{
    KRN_REQUIRE(ctx && launches, "null argument");
    *launches = ctx->launches;
    return KRN_OK;
}

// ---- View storage ---------------------------------------------------------------

extern "C" int krn_alloc(krn_ctx *ctx, size_t bytes, void **d_ptr)
{
    KRN_REQUIRE(ctx && d_ptr, "null argument");
    *d_ptr = nullptr;
    if (bytes == 0) bytes = 8;  // zero-extent views still get a distinct address
    KRN_CUDA(cudaMallocAsync(d_ptr, bytes, ctx->stream));
    return KRN_OK;
}

extern "C" int krn_free(krn_ctx *ctx, void *d_ptr)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (d_ptr == nullptr) return KRN_OK;
    KRN_CUDA(cudaFreeAsync(d_ptr, ctx->stream));
    return KRN_OK;
}

extern "C" int krn_host_alloc(size_t bytes, void **h_ptr)
{
    KRN_REQUIRE(h_ptr != nullptr, "null output");
    KRN_CUDA(cudaMallocHost(h_ptr, bytes ? bytes : 8));
    return KRN_OK;
}

extern "C" int krn_host_free(void *h_ptr)
{
    if (h_ptr) KRN_CUDA(cudaFreeHost(h_ptr));
    return KRN_OK;
}

extern "C" int krn_upload(krn_ctx *ctx, void *d_dst, const void *h_src, size_t bytes)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (bytes == 0) return KRN_OK;
    KRN_REQUIRE(d_dst && h_src, "null pointer");
    KRN_CUDA(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, ctx->stream));
    return KRN_OK;
}

extern "C" int krn_download_async(krn_ctx *ctx, void *h_dst, const void *d_src, size_t bytes)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (bytes == 0) return KRN_OK;
    KRN_REQUIRE(h_dst && d_src, "null pointer");
    KRN_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, ctx->stream));
    return KRN_OK;
}

extern "C" int krn_download(krn_ctx *ctx, void *h_dst, const void *d_src, size_t bytes)
{
    int rc = krn_download_async(ctx, h_dst, d_src, bytes);
    if (rc) return rc;
    KRN_CUDA(cudaStreamSynchronize(ctx->stream));
    return KRN_OK;
}

// ---- events -----------------------------------------------------------------------

extern "C" int krn_event_create(void **event)
{
    KRN_REQUIRE(event != nullptr, "null output");
    cudaEvent_t e;
    KRN_CUDA(cudaEventCreate(&e));
    *event = e;
    return KRN_OK;
}

extern "C" int krn_event_destroy(void *event)
{
    if (event) KRN_CUDA(cudaEventDestroy(static_cast<cudaEvent_t>(event)));
    return KRN_OK;
}

extern "C" int krn_event_record(krn_ctx *ctx, void *event)
{
    KRN_REQUIRE(ctx && event, "null argument");
    KRN_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), ctx->stream));
    return KRN_OK;
}

extern "C" int krn_event_elapsed_ms(void *start, void *stop, float *ms)
{
    KRN_REQUIRE(start && stop && ms, "null argument");
    KRN_CUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(stop)));
    KRN_CUDA(cudaEventElapsedTime(ms, static_cast<cudaEvent_t>(start), static_cast<cudaEvent_t>(stop)));
    return KRN_OK;
}

// ---- auxiliary copy streams ------------------------------------------------------------

extern "C" int krn_stream_create(krn_ctx *ctx, void **stream)
{
    KRN_REQUIRE(ctx && stream, "null argument");
    KRN_CUDA(cudaSetDevice(ctx->device));
    cudaStream_t s;
    KRN_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    *stream = s;
    return KRN_OK;
}

extern "C" int krn_stream_destroy(void *stream)
{
    if (stream) KRN_CUDA(cudaStreamDestroy(static_cast<cudaStream_t>(stream)));
    return KRN_OK;
}

extern "C" int krn_stream_sync(void *stream)
{
    KRN_REQUIRE(stream != nullptr, "null stream");
    KRN_CUDA(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)));
    return KRN_OK;
}

extern "C" int krn_upload_on(void *stream, void *d_dst, const void *h_src, size_t bytes)
{
    if (bytes == 0) return KRN_OK;
    KRN_REQUIRE(stream && d_dst && h_src, "null argument");
    KRN_CUDA(cudaMemcpyAsync(d_dst, h_src, bytes, cudaMemcpyHostToDevice, static_cast<cudaStream_t>(stream)));
    return KRN_OK;
}

extern "C" int krn_download_on(void *stream, void *h_dst, const void *d_src, size_t bytes)
{
    if (bytes == 0) return KRN_OK;
    KRN_REQUIRE(stream && h_dst && d_src, "null argument");
    KRN_CUDA(cudaMemcpyAsync(h_dst, d_src, bytes, cudaMemcpyDeviceToHost, static_cast<cudaStream_t>(stream)));
    return KRN_OK;
}

extern "C" int krn_event_record_on(void *stream, void *event)
{
    KRN_REQUIRE(stream && event, "null argument");
    KRN_CUDA(cudaEventRecord(static_cast<cudaEvent_t>(event), static_cast<cudaStream_t>(stream)));
    return KRN_OK;
}

extern "C" int krn_stream_wait_event(void *stream, void *event)
{
    KRN_REQUIRE(stream && event, "null argument");
    KRN_CUDA(cudaStreamWaitEvent(static_cast<cudaStream_t>(stream), static_cast<cudaEvent_t>(event), 0));
    return KRN_OK;
}

extern "C" int krn_ctx_wait_event(krn_ctx *ctx, void *event)
{
    KRN_REQUIRE(ctx && event, "null argument");
    KRN_CUDA(cudaStreamWaitEvent(ctx->stream, static_cast<cudaEvent_t>(event), 0));
    return KRN_OK;
}

// ---- status word ---------------------------------------------------------------------

extern "C" int krn_status_reset(krn_ctx *ctx)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    KRN_CUDA(cudaMemsetAsync(ctx->d_status, 0, 8 * sizeof(long long), ctx->stream));
    return KRN_OK;
}

extern "C" int krn_run_begin(krn_ctx *ctx, double **d_slots, size_t *capacity)
{
    KRN_REQUIRE(ctx && d_slots && capacity, "null argument");
    KRN_CUDA(cudaMemsetAsync(ctx->d_status, 0, (8 + KRN_SCALAR_SLOTS) * 8, ctx->stream));
    *d_slots = reinterpret_cast<double *>(ctx->d_status + 8);
    *capacity = KRN_SCALAR_SLOTS;
    return KRN_OK;
}

extern "C" int krn_reduce_workspace(krn_ctx *ctx, size_t blocks, double **d_partials, double **d_scratch,
                                    unsigned int **d_ticket)
{
    KRN_REQUIRE(ctx && d_partials && d_scratch && d_ticket, "null argument");
    int rc = krn_reserve_partials(ctx, blocks);
    if (rc) return rc;
    *d_partials = ctx->d_partials;
    *d_scratch = ctx->d_partials + ctx->partial_capacity;
    *d_ticket = ctx->d_ticket;
    return KRN_OK;
}

extern "C" int krn_status_device_ptr(krn_ctx *ctx, long long **d_status)
{
    KRN_REQUIRE(ctx && d_status, "null argument");
    *d_status = ctx->d_status;
    return KRN_OK;
}

extern "C" int krn_status_read(krn_ctx *ctx, long long h_status[8])
{
    KRN_REQUIRE(ctx && h_status, "null argument");
    KRN_CUDA(cudaMemcpyAsync(h_status, ctx->d_status, 8 * sizeof(long long), cudaMemcpyDeviceToHost,
                             ctx->stream));
    KRN_CUDA(cudaStreamSynchronize(ctx->stream));
    return KRN_OK;
}
