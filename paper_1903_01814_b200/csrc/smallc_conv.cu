// smallc_conv.cu -- single-input-channel hexagonal convolution, bf16 NHWC
// (BASELINE config 5 layer 1: 1 -> 64 channels, n = 2, on 96x96 camera
// images).  With Cin = 1 the layer has no channel contraction, so it is a
// stencil, not a GEMM: each warp owns one output pixel at a time and each lane
// two output channels (bf16x2), the lane's weights live in registers, and the
// T neighbour values are warp-uniform loads.  Stores / dy loads are one
// coalesced 128-byte row per warp per pixel.
//
// Forward:  y[p][co] = relu?(bias[co] + sum_t w[co][t] * x[p + off_t])
// Weight gradient: dw[co][t] = sum_p dy[p][co] * x[p + off_t],
//                  dbias[co] = sum_p dy[p][co]
// (off-grid neighbours contribute 0, A4).  The
// weight gradient reduces per block in a fixed warp order and then across
// blocks in a fixed order: deterministic.
#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {

constexpr int SC_WARPS = 8;
constexpr int SC_WG_BLOCKS = 592;  // 4 x 148 SMs

template <int N>
struct TapsOf {
    static constexpr int T = 3 * N * (N + 1) + 1;
};

// Neighbour value of tap t for a centre (r, c) with column parity p; 0 when off-grid.
template <int N>
__device__ __forceinline__ void gather_taps(const __nv_bfloat16* __restrict__ xb, int H, int W, int r, int c, int p,
                                            float* v) {
    int t = 0;
#pragma unroll
    for (int dc = -N; dc <= N; ++dc) {
        const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
        const int cc = c + dc;
        const bool colok = cc >= 0 && cc < W;
        const int top = r - N + (((dc < 0 ? -dc : dc) + p) >> 1);
#pragma unroll
        for (int k = 0; k < len; ++k, ++t) {
            const int rr = top + k;
            v[t] = (colok && rr >= 0 && rr < H) ? __bfloat162float(xb[rr * W + cc]) : 0.f;
        }
    }
}

// Each warp walks its pixels in batches of 32: lane j computes pixel j's centre
// and gathers its T neighbour values once into shared memory; then the warp
// sweeps the 32 pixels with lanes owning output-channel pairs (uniform LDS of
// the gathered values, one coalesced 128-byte dy load / y store per pixel).
template <int N>
__device__ __forceinline__ void stage_batch(const __nv_bfloat16* __restrict__ x, const Geom& g, int64_t pix0,
                                            int64_t npix, float* sv) {
    constexpr int T = TapsOf<N>::T;
    const int lane = threadIdx.x & 31;
    const int64_t pix = pix0 + lane;
    float v[T + 1];
    if (pix < npix) {
        const int npix_img = g.Ho * g.Wo;
        const int b = (int)(pix / npix_img);
        const int o = (int)(pix - (int64_t)b * npix_img);
        const int R = o / g.Wo, C = o - R * g.Wo;
        const int c = g.s * C;
        const int r = hex_rho(C, g.s, g.parity) + g.s * R;
        gather_taps<N>(x + (int64_t)b * g.H * g.W, g.H, g.W, r, c, (c + g.parity) & 1, v);
        v[T] = 1.f;
    } else {
#pragma unroll
        for (int t = 0; t <= T; ++t) v[t] = 0.f;
    }
#pragma unroll
    for (int t = 0; t <= T; ++t) sv[lane * (T + 1) + t] = v[t];
    __syncwarp();
}

template <int N>
__global__ void __launch_bounds__(SC_WARPS * 32)
smallc_fwd_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ w,
                  const float* __restrict__ bias, __nv_bfloat16* __restrict__ y, Geom g, int Cout, int relu) {
    constexpr int T = TapsOf<N>::T;
    constexpr int NA = T + 1;
    static_assert(NA % 4 == 0, "16-byte tap rows");
    __shared__ __align__(16) float sv_all[SC_WARPS][33 * NA];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sv = sv_all[warp];
    if (lane < NA) sv[32 * NA + lane] = 0.f;
    const int co = blockIdx.y * 64 + 2 * lane;
    float w0[NA], w1[NA];
#pragma unroll
    for (int t = 0; t < T; ++t) {
        w0[t] = __bfloat162float(w[(int64_t)co * T + t]);
        w1[t] = __bfloat162float(w[(int64_t)(co + 1) * T + t]);
    }
    w0[T] = bias ? bias[co] : 0.f;   // the ones column carries the bias
    w1[T] = bias ? bias[co + 1] : 0.f;
    const int64_t npix = (int64_t)g.B * g.Ho * g.Wo;
    const int64_t nbatch = (npix + 31) / 32;
    for (int64_t bt = (int64_t)blockIdx.x * SC_WARPS + warp; bt < nbatch; bt += (int64_t)gridDim.x * SC_WARPS) {
        const int64_t pix0 = bt * 32;
        stage_batch<N>(x, g, pix0, npix, sv);
        const int cnt = (int)min((int64_t)32, npix - pix0);
        // two pixels per iteration (independent FMA chains), 16-byte broadcast smem loads
        for (int j = 0; j < cnt; j += 2) {
            const float4* v0 = reinterpret_cast<const float4*>(sv + j * NA);
            const float4* v1 = reinterpret_cast<const float4*>(sv + (j + 1) * NA);  // row 32 exists (zeros)
            float a0 = 0.f, a1 = 0.f, b0 = 0.f, b1 = 0.f;
#pragma unroll
            for (int q = 0; q < NA / 4; ++q) {
                const float4 u = v0[q], v = v1[q];
                a0 = fmaf(w0[4 * q], u.x, a0); a1 = fmaf(w1[4 * q], u.x, a1);
                b0 = fmaf(w0[4 * q], v.x, b0); b1 = fmaf(w1[4 * q], v.x, b1);
                a0 = fmaf(w0[4 * q + 1], u.y, a0); a1 = fmaf(w1[4 * q + 1], u.y, a1);
                b0 = fmaf(w0[4 * q + 1], v.y, b0); b1 = fmaf(w1[4 * q + 1], v.y, b1);
                a0 = fmaf(w0[4 * q + 2], u.z, a0); a1 = fmaf(w1[4 * q + 2], u.z, a1);
                b0 = fmaf(w0[4 * q + 2], v.z, b0); b1 = fmaf(w1[4 * q + 2], v.z, b1);
                a0 = fmaf(w0[4 * q + 3], u.w, a0); a1 = fmaf(w1[4 * q + 3], u.w, a1);
                b0 = fmaf(w0[4 * q + 3], v.w, b0); b1 = fmaf(w1[4 * q + 3], v.w, b1);
            }
            if (relu) { a0 = fmaxf(a0, 0.f); a1 = fmaxf(a1, 0.f); b0 = fmaxf(b0, 0.f); b1 = fmaxf(b1, 0.f); }
            *reinterpret_cast<__nv_bfloat162*>(y + (pix0 + j) * Cout + co) = __floats2bfloat162_rn(a0, a1);
            if (j + 1 < cnt)
                *reinterpret_cast<__nv_bfloat162*>(y + (pix0 + j + 1) * Cout + co) = __floats2bfloat162_rn(b0, b1);
        }
        __syncwarp();
    }
}

template <int N>
__global__ void __launch_bounds__(SC_WARPS * 32)
smallc_wgrad_kernel(const __nv_bfloat16* __restrict__ x, const __nv_bfloat16* __restrict__ dy,
                    float* __restrict__ part, Geom g, int Cout) {
    constexpr int T = TapsOf<N>::T;
    constexpr int NA = T + 1;  // taps + bias column (ones)
    __shared__ float sv_all[SC_WARPS][32 * NA];
    __shared__ float red[SC_WARPS / 2][NA][64];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float* sv = sv_all[warp];
    const int co = blockIdx.y * 64 + 2 * lane;
    float a0[NA], a1[NA];
#pragma unroll
    for (int t = 0; t < NA; ++t) { a0[t] = 0.f; a1[t] = 0.f; }
    const int64_t npix = (int64_t)g.B * g.Ho * g.Wo;
    const int64_t nbatch = (npix + 31) / 32;
    for (int64_t bt = (int64_t)blockIdx.x * SC_WARPS + warp; bt < nbatch; bt += (int64_t)gridDim.x * SC_WARPS) {
        const int64_t pix0 = bt * 32;
        stage_batch<N>(x, g, pix0, npix, sv);
        const int cnt = (int)min((int64_t)32, npix - pix0);
        for (int j = 0; j < cnt; ++j) {
            const __nv_bfloat162 d2 = *reinterpret_cast<const __nv_bfloat162*>(dy + (pix0 + j) * Cout + co);
            const float d0 = __low2float(d2), d1 = __high2float(d2);
            const float* vj = sv + j * NA;
#pragma unroll
            for (int t = 0; t < NA; ++t) {
                const float vt = vj[t];
                a0[t] = fmaf(d0, vt, a0[t]);
                a1[t] = fmaf(d1, vt, a1[t]);
            }
        }
        __syncwarp();
    }
    // fixed-order reduction over the block's warps: red[k] = acc(warp k+4) + acc(warp k), then sum k
    constexpr int HW_ = SC_WARPS / 2;
    if (warp >= HW_) {
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            red[warp - HW_][t][2 * lane] = a0[t];
            red[warp - HW_][t][2 * lane + 1] = a1[t];
        }
    }
    __syncthreads();
    if (warp < HW_) {
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            red[warp][t][2 * lane] += a0[t];
            red[warp][t][2 * lane + 1] += a1[t];
        }
    }
    __syncthreads();
    // part[block][co][t]
    for (int i = threadIdx.x; i < 64 * NA; i += blockDim.x) {
        const int cl = i / NA, t = i % NA;
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < HW_; ++k) s += red[k][t][cl];
        part[((int64_t)blockIdx.x * Cout + blockIdx.y * 64 + cl) * NA + t] = s;
    }
}

__global__ void smallc_wgrad_reduce_kernel(const float* __restrict__ part, int nblocks, int Cout, int NA,
                                           float* __restrict__ dw, float* __restrict__ dbias, int accumulate) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Cout * NA) return;
    float s = 0.f;
    for (int k = 0; k < nblocks; ++k) s += part[(int64_t)k * Cout * NA + i];
    const int co = i / NA, t = i % NA;
    if (t == NA - 1) {
        if (dbias) dbias[co] = accumulate ? dbias[co] + s : s;
    } else {
        float* d = dw + (int64_t)co * (NA - 1) + t;
        *d = accumulate ? *d + s : s;
    }
}

bool smallc_supported(const Geom& g, int Cin, int Cout) {
    return Cin == 1 && Cout % 64 == 0 && g.n >= 1 && g.n <= 2;
}

// Stride 1 runs on the tensor-core kernels of smallc_mma.cu; the FFMA stencil
// above remains for stride > 1 (HEXCONV_SMALLC_FFMA=1 forces it, for A/B runs).
static bool use_mma(const Geom& g, int Cout) {
    static const bool force_ffma = sw_on("HEXCONV_SMALLC_FFMA");
    return !force_ffma && smallc_mma_supported(g, 1, Cout);
}

size_t smallc_wgrad_ws_bytes(const Geom& g, int Cout) {
    const size_t a = (size_t)SC_WG_BLOCKS * Cout * (g.T + 1) * sizeof(float);
    const size_t b = smallc_mma_wgrad_ws_bytes(g, Cout);
    return a > b ? a : b;
}

hex_status_t smallc_fwd(const void* x, const void* w, const float* bias, void* y, const Geom& g, int Cout, int relu,
                        cudaStream_t st) {
    if (use_mma(g, Cout)) return smallc_mma_fwd(x, w, bias, y, g, Cout, relu, st);
    const int64_t npix = (int64_t)g.B * g.Ho * g.Wo;
    int blocks = (int)((npix + SC_WARPS * 32 * 4 - 1) / (SC_WARPS * 32 * 4));  // ~4 pixel batches per warp
    if (blocks > 148 * 8) blocks = 148 * 8;
    if (blocks < 1) blocks = 1;
    dim3 grid(blocks, Cout / 64);
    const auto* xb = (const __nv_bfloat16*)x;
    const auto* wb = (const __nv_bfloat16*)w;
    auto* yb = (__nv_bfloat16*)y;
    switch (g.n) {
        case 1: smallc_fwd_kernel<1><<<grid, SC_WARPS * 32, 0, st>>>(xb, wb, bias, yb, g, Cout, relu); break;
        default: smallc_fwd_kernel<2><<<grid, SC_WARPS * 32, 0, st>>>(xb, wb, bias, yb, g, Cout, relu); break;
    }
    count_launch();
    return last_launch_status();
}

hex_status_t smallc_wgrad(const void* x, const void* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                          int Cout, void* ws, cudaStream_t st) {
    if (use_mma(g, Cout)) return smallc_mma_wgrad(x, dy, dw, dbias, accumulate, g, Cout, ws, st);
    dim3 grid(SC_WG_BLOCKS, Cout / 64);
    const auto* xb = (const __nv_bfloat16*)x;
    const auto* db = (const __nv_bfloat16*)dy;
    float* part = (float*)ws;
    switch (g.n) {
        case 1: smallc_wgrad_kernel<1><<<grid, SC_WARPS * 32, 0, st>>>(xb, db, part, g, Cout); break;
        default: smallc_wgrad_kernel<2><<<grid, SC_WARPS * 32, 0, st>>>(xb, db, part, g, Cout); break;
    }
    count_launch();
    const int NA = g.T + 1;
    smallc_wgrad_reduce_kernel<<<ceil_div(Cout * NA, 256), 256, 0, st>>>(part, SC_WG_BLOCKS, Cout, NA, dw, dbias,
                                                                         accumulate);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
