// Internal declarations shared by the translation units of libkrn_b200.so.
#pragma once

#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <cstring>

#include "../../include/krn_b200.h"

struct krn_ctx {
    int device = 0;
    int sms = 148;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    cudaMemPool_t pool = nullptr;
    // reduction workspace: two ping-pong partial arrays and an arrival ticket
    double *d_partials = nullptr;
    size_t partial_capacity = 0;    // doubles per ping-pong half
    unsigned int *d_ticket = nullptr;
    long long *d_status = nullptr;  // 8 x int64 {code, line, view id, index0, index1, ...}
    uint64_t launches = 0;
};

void krn_set_error(const char *fmt, ...);

#define KRN_CUDA(expr)                                                               \
    do {                                                                             \
        cudaError_t e__ = (expr);                                                    \
        if (e__ != cudaSuccess) {                                                    \
            krn_set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e__),   \
                          __FILE__, __LINE__);                                       \
            (void)cudaGetLastError(); /* reported here: the next launch check must not see it again */ \
            return KRN_E_CUDA;                                                       \
        }                                                                            \
    } while (0)

#define KRN_REQUIRE(cond, msg)                        \
    do {                                              \
        if (!(cond)) {                                \
            krn_set_error("%s: %s", __func__, msg);   \
            return KRN_E_ARG;                         \
        }                                             \
    } while (0)

#define KRN_LAUNCH_CHECK(ctx)            \
    do {                                 \
        (ctx)->launches++;               \
        KRN_CUDA(cudaGetLastError());    \
    } while (0)

// make sure each ping-pong half of the reduction workspace holds `count` doubles
int krn_reserve_partials(krn_ctx *ctx, size_t count);
#define KRN_SCALAR_SLOTS 120  // function-scope scalar slots that live next to the status word

static inline bool krn_aligned32(const void *p) { return (reinterpret_cast<uintptr_t>(p) & 31u) == 0; }
