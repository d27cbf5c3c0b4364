// Peer memory between the ranks of a sharded run (one process per GPU): a rank exports the
// allocations that hold its Views once, its neighbours map them (CUDA IPC; peer access over
// NVLink is enabled lazily by the mapping) and the kernels then read the few halo rows they need
// straight from the neighbour's buffer - no pack kernel, no collective, no staging copy per step.
// Two processes on ONE device work the same way (that is how the GPU tests exercise it).
#include "krn_common.cuh"

#include <cuda.h>

namespace {

typedef CUresult (*GetAddressRangeFn)(CUdeviceptr *, size_t *, CUdeviceptr);

int address_range(const void *ptr, void **base, size_t *size)
{
    static GetAddressRangeFn fn = nullptr;
    if (fn == nullptr) {
        void *sym = nullptr;
        cudaDriverEntryPointQueryResult status;
        KRN_CUDA(cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &status));
        if (sym == nullptr || status != cudaDriverEntryPointSuccess) {
            krn_set_error("cuMemGetAddressRange is not available from the driver");
            return KRN_E_UNAVAILABLE;
        }
        fn = reinterpret_cast<GetAddressRangeFn>(sym);
    }
    CUdeviceptr b = 0;
    size_t n = 0;
    CUresult r = fn(&b, &n, reinterpret_cast<CUdeviceptr>(ptr));
    if (r != CUDA_SUCCESS) {
        krn_set_error("cuMemGetAddressRange failed (%d): not a device allocation?", int(r));
        return KRN_E_CUDA;
    }
    *base = reinterpret_cast<void *>(b);
    *size = n;
    return KRN_OK;
}

}  // namespace

static_assert(sizeof(cudaIpcMemHandle_t) == 64, "handle size is part of the C ABI");

extern "C" int krn_ipc_export(krn_ctx *ctx, const void *d_ptr, unsigned char handle[64], size_t *offset)
{
    KRN_REQUIRE(ctx && d_ptr && handle && offset, "null argument");
    KRN_CUDA(cudaSetDevice(ctx->device));
    void *base = nullptr;
    size_t size = 0;
    int rc = address_range(d_ptr, &base, &size);
    if (rc) return rc;
    cudaIpcMemHandle_t h;
    KRN_CUDA(cudaIpcGetMemHandle(&h, base));
    memcpy(handle, &h, 64);
    *offset = size_t(reinterpret_cast<const char *>(d_ptr) - reinterpret_cast<const char *>(base));
    return KRN_OK;
}

extern "C" int krn_ipc_open(krn_ctx *ctx, const unsigned char handle[64], size_t offset, void **d_base, void **d_ptr)
{
    KRN_REQUIRE(ctx && handle && d_base && d_ptr, "null argument");
    KRN_CUDA(cudaSetDevice(ctx->device));
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, 64);
    void *base = nullptr;
    KRN_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
    *d_base = base;
    *d_ptr = static_cast<char *>(base) + offset;
    return KRN_OK;
}

extern "C" int krn_ipc_close(krn_ctx *ctx, void *d_base)
{
    KRN_REQUIRE(ctx != nullptr, "null context");
    if (d_base == nullptr) return KRN_OK;
    KRN_CUDA(cudaSetDevice(ctx->device));
    KRN_CUDA(cudaStreamSynchronize(ctx->stream));
    KRN_CUDA(cudaIpcCloseMemHandle(d_base));
    return KRN_OK;
}
