// common.cuh -- shared helpers of libhexconv (CUDA side only; never included by
// the oracle).  Geometry of the offset-column hex grid lives in geometry.cuh.
#pragma once
#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <atomic>

#include "../../include/hexconv.h"

namespace hexconv {

// Host-side launch counter (hex_launch_count): every kernel launch site calls
// count_launch() right after the <<<>>> / cudaLaunchKernelEx.
extern std::atomic<int64_t> g_launches;
inline void count_launch(int64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

inline hex_status_t last_launch_status() {
    cudaError_t e = cudaGetLastError();
    return e == cudaSuccess ? HEX_OK : HEX_ERR_CUDA;
}

// Element strides (in elements) of a 4-D activation tensor [B, C, H, W] stored
// in `layout`.
struct Strides4 {
    int64_t b, c, h, w;
};
inline Strides4 make_strides(int layout, int C, int H, int W) {
    Strides4 s;
    if (layout == HEX_NCHW) {
        s.w = 1; s.h = W; s.c = (int64_t)H * W; s.b = (int64_t)C * H * W;
    } else {
        s.c = 1; s.w = C; s.h = (int64_t)W * C; s.b = (int64_t)H * W * C;
    }
    return s;
}

template <typename T> __device__ __forceinline__ float to_f32(T v);
template <> __device__ __forceinline__ float to_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ float to_f32<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T> __device__ __forceinline__ T from_f32(float v);
template <> __device__ __forceinline__ float from_f32<float>(float v) { return v; }
template <> __device__ __forceinline__ __nv_bfloat16 from_f32<__nv_bfloat16>(float v) { return __float2bfloat16_rn(v); }

// Kernel-selection switches: the HEXCONV_* environment
// variables are read ONCE, when the library is loaded (abi.cu), never on the dispatch path, so a CUDA graph
// captures the same selection every call sees.  hex_debug_set_switch() overrides one (A/B tests only).
// Every switch picks between kernels that compute the same result (up to the documented summation order).
bool sw_on(const char* name);                      // the variable is set
int sw_int(const char* name, int dflt);            // its integer value, or dflt when unset
double sw_double(const char* name, double dflt);   // its floating value, or dflt when unset

// Timing-experiment modes that skip loads / MMAs / epilogues (results invalid) exist only in builds
// compiled with -DHEXCONV_TIMING_DEBUG=1; in the product library HEX_DBG(x) is the constant 0.
#ifndef HEXCONV_TIMING_DEBUG
#define HEXCONV_TIMING_DEBUG 0
#endif
#define HEX_DBG(x) (HEXCONV_TIMING_DEBUG ? (x) : 0)
inline int debug_mode(const char* name) { return HEXCONV_TIMING_DEBUG ? sw_int(name, 0) : 0; }

inline int ceil_div(int64_t a, int64_t b) { return (int)((a + b - 1) / b); }

inline int num_sms() {
    static int sms = 0;
    if (sms == 0) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

}  // namespace hexconv
