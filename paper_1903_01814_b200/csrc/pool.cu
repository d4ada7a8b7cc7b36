// pool.cu -- hexagonal max / average pooling, forward and backward.
//
// pooling replaces the sub-convolutions and the results are
// "combined with aggregation functions, whereas the padding- and
// striding-scheme is identical".  Readings: A8 max ignores
// off-grid cells and avg divides by the in-grid count; A9 ties resolve to the
// first maximal tap in canonical order (strict '>' scan), and the output bits
// are a copy of x at that tap.
//
// HBM-bound stencils.  NHWC tensors with C % 8 == 0 use 16-byte vectors of 8
// channels per thread; everything else one element per thread.  The backward
// pass is a gather over the candidate centres of each input pixel (no
// atomics, deterministic).
#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "pool_tables.cuh"

namespace hexconv {

template <typename T>
__global__ void pool_fwd_kernel(const T* __restrict__ x, T* __restrict__ y, uint8_t* __restrict__ am, Geom g,
                                int Cc, Strides4 sx, Strides4 sy, int mode, int chan_fast) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)g.B * Cc * g.Ho * g.Wo;
    if (idx >= total) return;
    int ch, C, R, b;
    if (chan_fast) {
        ch = (int)(idx % Cc);
        int64_t q = idx / Cc;
        C = (int)(q % g.Wo); q /= g.Wo;
        R = (int)(q % g.Ho);
        b = (int)(q / g.Ho);
    } else {
        C = (int)(idx % g.Wo);
        int64_t q = idx / g.Wo;
        R = (int)(q % g.Ho); q /= g.Ho;
        ch = (int)(q % Cc);
        b = (int)(q / Cc);
    }
    const int c = g.s * C;
    const int r = hex_rho(C, g.s, g.parity) + g.s * R;
    const int p = (c + g.parity) & 1;
    const int n = g.n;
    const T* xp = x + (int64_t)b * sx.b + (int64_t)ch * sx.c;
    int t = 0, best = -1, cnt = 0;
    float bv = 0.f, sum = 0.f;
    T braw = from_f32<T>(0.f);
    for (int dc = -n; dc <= n; ++dc) {
        const int len = 2 * n + 1 - (dc < 0 ? -dc : dc);
        const int cc = c + dc;
        if (cc < 0 || cc >= g.W) { t += len; continue; }
        int rr = r + tap_top(n, dc, p);
        for (int k = 0; k < len; ++k, ++t, ++rr) {
            if (rr < 0 || rr >= g.H) continue;
            const T raw = xp[(int64_t)rr * sx.h + (int64_t)cc * sx.w];
            const float v = to_f32(raw);
            if (mode == HEX_POOL_MAX) {
                if (best < 0 || v > bv) { best = t; bv = v; braw = raw; }
            } else {
                sum += v;
                ++cnt;
            }
        }
    }
    const int64_t yo = (int64_t)b * sy.b + (int64_t)ch * sy.c + (int64_t)R * sy.h + (int64_t)C * sy.w;
    if (mode == HEX_POOL_MAX) {
        y[yo] = braw;
        if (am) am[yo] = (uint8_t)best;
    } else {
        y[yo] = from_f32<T>(sum / (float)(mode == HEX_POOL_AVG_PAD ? g.T : cnt));
    }
}

// NHWC bf16, 8 channels per thread (16-byte loads/stores).
__global__ void pool_fwd_nhwc_bf16x8_kernel(const uint4* __restrict__ x, uint4* __restrict__ y,
                                            uint64_t* __restrict__ am, Geom g, int C8, int mode) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)g.B * C8 * g.Ho * g.Wo;
    if (idx >= total) return;
    const int ch8 = (int)(idx % C8);
    int64_t q = idx / C8;
    const int C = (int)(q % g.Wo); q /= g.Wo;
    const int R = (int)(q % g.Ho);
    const int b = (int)(q / g.Ho);
    const int c = g.s * C;
    const int r = hex_rho(C, g.s, g.parity) + g.s * R;
    const int p = (c + g.parity) & 1;
    const int n = g.n;
    const uint4* xp = x + (int64_t)b * g.H * g.W * C8 + ch8;
    float bv[8], sum[8];
    int best[8];
    __nv_bfloat16 braw[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) { bv[j] = 0.f; sum[j] = 0.f; best[j] = -1; braw[j] = __float2bfloat16_rn(0.f); }
    int t = 0, cnt = 0;
    for (int dc = -n; dc <= n; ++dc) {
        const int len = 2 * n + 1 - (dc < 0 ? -dc : dc);
        const int cc = c + dc;
        if (cc < 0 || cc >= g.W) { t += len; continue; }
        int rr = r + tap_top(n, dc, p);
        for (int k = 0; k < len; ++k, ++t, ++rr) {
            if (rr < 0 || rr >= g.H) continue;
            uint4 v4 = __ldg(xp + ((int64_t)rr * g.W + cc) * C8);
            const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&v4);
            ++cnt;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float f = __bfloat162float(v[j]);
                if (mode == HEX_POOL_MAX) {
                    if (best[j] < 0 || f > bv[j]) { best[j] = t; bv[j] = f; braw[j] = v[j]; }
                } else {
                    sum[j] += f;
                }
            }
        }
    }
    uint4 out;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&out);
    const int64_t yo = (((int64_t)b * g.Ho + R) * g.Wo + C) * C8 + ch8;
    if (mode == HEX_POOL_MAX) {
        uint64_t a = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) { o[j] = braw[j]; a |= (uint64_t)(uint8_t)best[j] << (8 * j); }
        if (am) am[yo] = a;
    } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) o[j] = __float2bfloat16_rn(sum[j] / (float)cnt);
    }
    y[yo] = out;
}

// Number of in-grid taps of the centre at (r, c).
__device__ __forceinline__ int in_grid_count(const Geom& g, int r, int c) {
    const int p = (c + g.parity) & 1;
    int cnt = 0;
    for (int dc = -g.n; dc <= g.n; ++dc) {
        const int cc = c + dc;
        if (cc < 0 || cc >= g.W) continue;
        const int len = 2 * g.n + 1 - (dc < 0 ? -dc : dc);
        const int top = r + tap_top(g.n, dc, p);
        const int lo = max(top, 0), hi = min(top + len, g.H);
        cnt += max(hi - lo, 0);
    }
    return cnt;
}

// Backward: one thread per input element (gather over candidate centres).
template <typename T>
__global__ void pool_bwd_kernel(const T* __restrict__ dy, const uint8_t* __restrict__ am, T* __restrict__ dx,
                                Geom g, int Cc, Strides4 sx, Strides4 sy, int mode, int chan_fast) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)g.B * Cc * g.H * g.W;
    if (idx >= total) return;
    int ch, c, r, b;
    if (chan_fast) {
        ch = (int)(idx % Cc);
        int64_t q = idx / Cc;
        c = (int)(q % g.W); q /= g.W;
        r = (int)(q % g.H);
        b = (int)(q / g.H);
    } else {
        c = (int)(idx % g.W);
        int64_t q = idx / g.W;
        r = (int)(q % g.H); q /= g.H;
        ch = (int)(q % Cc);
        b = (int)(q / Cc);
    }
    const int n = g.n, s = g.s;
    const int64_t ybase = (int64_t)b * sy.b + (int64_t)ch * sy.c;
    float acc = 0.f;
    int t = 0;
    for (int dc = -n; dc <= n; ++dc) {
        const int len = 2 * n + 1 - (dc < 0 ? -dc : dc);
        const int oc = c - dc;
        if (oc < 0 || oc % s != 0 || oc / s >= g.Wo) { t += len; continue; }
        const int Cq = oc / s;
        const int po = (oc + g.parity) & 1;
        const int rho = hex_rho(Cq, s, g.parity);
        const int top = tap_top(n, dc, po);
        for (int k = 0; k < len; ++k, ++t) {
            const int d = r - (top + k) - rho;
            if (d < 0 || d % s != 0) continue;
            const int Rq = d / s;
            if (Rq >= g.Ho) continue;
            const int64_t yo = ybase + (int64_t)Rq * sy.h + (int64_t)Cq * sy.w;
            if (mode == HEX_POOL_MAX) {
                if (am[yo] == t) acc += to_f32(dy[yo]);
            } else {
                const int orow = rho + s * Rq;
                acc += to_f32(dy[yo]) / (float)(mode == HEX_POOL_AVG_PAD ? g.T : in_grid_count(g, orow, oc));
            }
        }
    }
    dx[(int64_t)b * sx.b + (int64_t)ch * sx.c + (int64_t)r * sx.h + (int64_t)c * sx.w] = from_f32<T>(acc);
}

// NHWC bf16 backward, 8 channels per thread.
__global__ void pool_bwd_nhwc_bf16x8_kernel(const uint4* __restrict__ dy, const uint64_t* __restrict__ am,
                                            uint4* __restrict__ dx, Geom g, int C8, int mode) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)g.B * C8 * g.H * g.W;
    if (idx >= total) return;
    const int ch8 = (int)(idx % C8);
    int64_t q = idx / C8;
    const int c = (int)(q % g.W); q /= g.W;
    const int r = (int)(q % g.H);
    const int b = (int)(q / g.H);
    const int n = g.n, s = g.s;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    int t = 0;
    for (int dc = -n; dc <= n; ++dc) {
        const int len = 2 * n + 1 - (dc < 0 ? -dc : dc);
        const int oc = c - dc;
        if (oc < 0 || oc % s != 0 || oc / s >= g.Wo) { t += len; continue; }
        const int Cq = oc / s;
        const int po = (oc + g.parity) & 1;
        const int rho = hex_rho(Cq, s, g.parity);
        const int top = tap_top(n, dc, po);
        for (int k = 0; k < len; ++k, ++t) {
            const int d = r - (top + k) - rho;
            if (d < 0 || d % s != 0) continue;
            const int Rq = d / s;
            if (Rq >= g.Ho) continue;
            const int64_t yo = (((int64_t)b * g.Ho + Rq) * g.Wo + Cq) * C8 + ch8;
            uint4 v4 = __ldg(dy + yo);
            const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&v4);
            if (mode == HEX_POOL_MAX) {
                const uint64_t a = __ldg(am + yo);
#pragma unroll
                for (int j = 0; j < 8; ++j)
                    if ((int)((a >> (8 * j)) & 0xff) == t) acc[j] += __bfloat162float(v[j]);
            } else {
                const float inv = 1.f / (float)in_grid_count(g, rho + s * Rq, oc);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(v[j]) * inv;
            }
        }
    }
    uint4 out;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&out);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = __float2bfloat16_rn(acc[j]);
    dx[(((int64_t)b * g.H + r) * g.W + c) * C8 + ch8] = out;
}

// ---------------------------------------------------------------------------
// Specialised NHWC bf16 x8 kernels: compile-time kernel size N and stride S,
// batch on blockIdx.y, 32-bit index math (no 64-bit division on the hot path).
// ---------------------------------------------------------------------------
template <int N, int S>
__global__ void __launch_bounds__(256)
pool_fwd_nhwc_x8_spec(const uint4* __restrict__ x, uint4* __restrict__ y, uint64_t* __restrict__ am, Geom g, int C8,
                      int mode) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int per_img = g.Ho * g.Wo * C8;
    if (idx >= per_img) return;
    const int b = blockIdx.y;
    const int ch8 = idx % C8;
    const int o = idx / C8;
    const int R = o / g.Wo, C = o - R * g.Wo;
    const int c = S * C;
    const int r = ((S * C + g.parity) >> 1) % S + S * R;
    const int p = (c + g.parity) & 1;
    const uint4* xp = x + (size_t)b * g.H * g.W * C8 + ch8;
    float bv[8], sum[8];
    int best[8];
    uint32_t braw[4] = {0, 0, 0, 0};
#pragma unroll
    for (int j = 0; j < 8; ++j) { bv[j] = -INFINITY; sum[j] = 0.f; best[j] = -1; }
    int t = 0, cnt = 0;
#pragma unroll
    for (int dc = -N; dc <= N; ++dc) {
        const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
        const int cc = c + dc;
        const bool colok = cc >= 0 && cc < g.W;
        const int top = r - N + (((dc < 0 ? -dc : dc) + p) >> 1);
#pragma unroll
        for (int k = 0; k < len; ++k, ++t) {
            const int rr = top + k;
            if (!colok || rr < 0 || rr >= g.H) continue;
            const uint4 v4 = __ldg(xp + (rr * g.W + cc) * C8);
            const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
            ++cnt;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const uint32_t bits = (j & 1) ? (w[j >> 1] & 0xffff0000u) : (w[j >> 1] << 16);
                const float f = __uint_as_float(bits);
                if (mode == HEX_POOL_MAX) {
                    if (best[j] < 0 || f > bv[j]) {
                        best[j] = t;
                        bv[j] = f;
                        const uint32_t h = (j & 1) ? (w[j >> 1] & 0xffff0000u) : (w[j >> 1] & 0xffffu);
                        braw[j >> 1] = (j & 1) ? ((braw[j >> 1] & 0xffffu) | h) : ((braw[j >> 1] & 0xffff0000u) | h);
                    }
                } else {
                    sum[j] += f;
                }
            }
        }
    }
    const size_t yo = ((size_t)b * g.Ho * g.Wo + o) * C8 + ch8;
    if (mode == HEX_POOL_MAX) {
        uint64_t a = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) a |= (uint64_t)(uint8_t)best[j] << (8 * j);
        y[yo] = make_uint4(braw[0], braw[1], braw[2], braw[3]);
        if (am) am[yo] = a;
    } else {
        uint4 out;
        __nv_bfloat16* ob = reinterpret_cast<__nv_bfloat16*>(&out);
        const float inv = 1.f / (float)cnt;
#pragma unroll
        for (int j = 0; j < 8; ++j) ob[j] = __float2bfloat16_rn(sum[j] * inv);
        y[yo] = out;
    }
}

template <int N, int S>
__global__ void __launch_bounds__(256)
pool_bwd_nhwc_x8_spec(const uint4* __restrict__ dy, const uint64_t* __restrict__ am, uint4* __restrict__ dx, Geom g,
                      int C8, int mode) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int per_img = g.H * g.W * C8;
    if (idx >= per_img) return;
    const int b = blockIdx.y;
    const int ch8 = idx % C8;
    const int q = idx / C8;
    const int r = q / g.W, c = q - r * g.W;
    float acc[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) acc[j] = 0.f;
    const size_t ybase = (size_t)b * g.Ho * g.Wo * C8 + ch8;
    int t = 0;
#pragma unroll
    for (int dc = -N; dc <= N; ++dc) {
        const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
        const int oc = c - dc;
        const bool colok = oc >= 0 && (oc % S) == 0 && oc / S < g.Wo;
        const int Cq = oc / S;
        const int po = (oc + g.parity) & 1;
        const int rho = ((S * Cq + g.parity) >> 1) % S;
        const int top = -N + (((dc < 0 ? -dc : dc) + po) >> 1);
#pragma unroll
        for (int k = 0; k < len; ++k, ++t) {
            if (!colok) continue;
            const int d = r - (top + k) - rho;
            if (d < 0 || (d % S) != 0) continue;
            const int Rq = d / S;
            if (Rq >= g.Ho) continue;
            const size_t yo = ybase + (size_t)(Rq * g.Wo + Cq) * C8;
            const uint4 v4 = __ldg(dy + yo);
            const uint32_t w[4] = {v4.x, v4.y, v4.z, v4.w};
            if (mode == HEX_POOL_MAX) {
                const uint64_t a = __ldg(am + yo);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t bits = (j & 1) ? (w[j >> 1] & 0xffff0000u) : (w[j >> 1] << 16);
                    if ((int)((a >> (8 * j)) & 0xff) == t) acc[j] += __uint_as_float(bits);
                }
            } else {
                // in-grid count of the centre (oc, rho + S*Rq)
                const int orow = rho + S * Rq;
                int cnt = 0;
#pragma unroll
                for (int e = -N; e <= N; ++e) {
                    const int ccol = oc + e;
                    if (ccol < 0 || ccol >= g.W) continue;
                    const int l2 = 2 * N + 1 - (e < 0 ? -e : e);
                    const int tp = orow - N + (((e < 0 ? -e : e) + po) >> 1);
                    cnt += max(min(tp + l2, g.H) - max(tp, 0), 0);
                }
                const float inv = 1.f / (float)cnt;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t bits = (j & 1) ? (w[j >> 1] & 0xffff0000u) : (w[j >> 1] << 16);
                    acc[j] += __uint_as_float(bits) * inv;
                }
            }
        }
    }
    uint4 out;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&out);
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = __float2bfloat16_rn(acc[j]);
    dx[(size_t)b * per_img + idx] = out;
}

static bool use_vec8(const PoolArgs& a) {
    return a.dtype == HEX_BF16 && a.layout == HEX_NHWC && (a.C % 8) == 0;
}

static bool use_spec(const PoolArgs& a) {
    return use_vec8(a) && (a.g.n == 1 || a.g.n == 2) && (a.g.s == 1 || a.g.s == 2) && a.g.B <= 65535 &&
           (int64_t)a.g.H * a.g.W * (a.C / 8) < (1ll << 31);
}

template <int N, int S>
static void launch_spec_fwd(const PoolArgs& a, cudaStream_t st) {
    const int C8 = a.C / 8;
    dim3 grid(ceil_div((int64_t)a.g.Ho * a.g.Wo * C8, 256), a.g.B);
    pool_fwd_nhwc_x8_spec<N, S><<<grid, 256, 0, st>>>((const uint4*)a.x, (uint4*)a.y, (uint64_t*)a.argmax, a.g, C8,
                                                      a.mode);
}
template <int N, int S>
static void launch_spec_bwd(const PoolArgs& a, cudaStream_t st) {
    const int C8 = a.C / 8;
    dim3 grid(ceil_div((int64_t)a.g.H * a.g.W * C8, 256), a.g.B);
    pool_bwd_nhwc_x8_spec<N, S><<<grid, 256, 0, st>>>((const uint4*)a.dy, (const uint64_t*)a.argmax_in, (uint4*)a.dx,
                                                      a.g, C8, a.mode);
}


// ---------------------------------------------------------------------------
// Wide NHWC bf16 kernels: each thread owns V x 8 channels of one pixel, so the
// per-pixel index math is shared by 8V channels.  Max pooling compares packed
// bf16x2 pairs (__hgt2_mask, strict '>' keeps the first maximum) and keeps the
// tap index as packed bytes; the backward selects the routed channels with
// SIMD byte compares (__vcmpeq4) and byte-permuted masks.  Exactly the same
// results as the scalar kernels (max: a copy of the selected input; avg and
// backward: fp32 accumulation in canonical tap order).
// ---------------------------------------------------------------------------
template <int N, int S, int V, bool MAXP>  // MAXP: max pooling (else average), fixed at compile time
__global__ void __launch_bounds__(256)
pool_fwd_nhwc_v(const uint4* __restrict__ x, uint4* __restrict__ y, uint2* __restrict__ am, Geom g, int CV,
                int lgcv) {
    // grid: x = (output pixel, channel group) of image b = blockIdx.y
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= g.Ho * g.Wo * CV) return;
    const int b = blockIdx.y;
    const int cv = lgcv >= 0 ? (idx & (CV - 1)) : idx % CV;
    const int o = lgcv >= 0 ? (idx >> lgcv) : idx / CV;
    const int R = o / g.Wo, C = o - R * g.Wo;
    const int c = S * C;
    const int r = ((S * C + g.parity) >> 1) % S + S * R;
    const int p = (c + g.parity) & 1;
    const int C8 = CV * V;
    const uint4* xp = x + (size_t)b * g.H * g.W * C8 + cv * V;
    uint32_t best[4 * V], ix[4 * V];
    float sum[8 * V];
#pragma unroll
    for (int i = 0; i < 4 * V; ++i) { best[i] = 0u; ix[i] = 0u; }
#pragma unroll
    for (int i = 0; i < 8 * V; ++i) sum[i] = 0.f;
    int t = 0, cnt = 0;
#pragma unroll
    for (int dc = -N; dc <= N; ++dc) {
        const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
        const int cc = c + dc;
        const bool colok = cc >= 0 && cc < g.W;
        const int top = r - N + (((dc < 0 ? -dc : dc) + p) >> 1);
#pragma unroll
        for (int k = 0; k < len; ++k, ++t) {
            const int rr = top + k;
            if (!colok || rr < 0 || rr >= g.H) continue;
            const uint4* src = xp + (size_t)(rr * g.W + cc) * C8;
            const uint32_t tt = (uint32_t)t * 0x0101u;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const uint4 q = __ldg(src + v);
                const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const int i = 4 * v + kk;
                    if constexpr (MAXP) {
                        if (cnt == 0) {
                            best[i] = w[kk];
                            ix[i] = tt;
                        } else {
                            const unsigned m = __hgt2_mask(*reinterpret_cast<const __nv_bfloat162*>(&w[kk]),
                                                           *reinterpret_cast<const __nv_bfloat162*>(&best[i]));
                            best[i] = (w[kk] & m) | (best[i] & ~m);
                            const uint32_t bm = __byte_perm(m, 0u, 0x4420);
                            ix[i] = (tt & bm) | (ix[i] & ~bm);
                        }
                    } else {
                        sum[2 * i] += __uint_as_float(w[kk] << 16);
                        sum[2 * i + 1] += __uint_as_float(w[kk] & 0xffff0000u);
                    }
                }
            }
            ++cnt;
        }
    }
    const size_t yo = ((size_t)b * g.Ho * g.Wo + o) * C8 + cv * V;
    if constexpr (MAXP) {
#pragma unroll
        for (int v = 0; v < V; ++v) {
            y[yo + v] = make_uint4(best[4 * v], best[4 * v + 1], best[4 * v + 2], best[4 * v + 3]);
            if (am) am[yo + v] = make_uint2(ix[4 * v] | (ix[4 * v + 1] << 16), ix[4 * v + 2] | (ix[4 * v + 3] << 16));
        }
    } else {
        const float inv = 1.f / (float)cnt;
#pragma unroll
        for (int v = 0; v < V; ++v) {
            uint32_t pk[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                const int i = 4 * v + kk;
                __nv_bfloat162 h = __floats2bfloat162_rn(sum[2 * i] * inv, sum[2 * i + 1] * inv);
                pk[kk] = *reinterpret_cast<uint32_t*>(&h);
            }
            y[yo + v] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
    }
}

template <int N, int S, int V>
__global__ void __launch_bounds__(256)
pool_bwd_nhwc_v(const uint4* __restrict__ dy, const uint2* __restrict__ am, uint4* __restrict__ dx, Geom g, int CV,
                int mode) {
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int per_img = g.H * g.W * CV;
    if (idx >= per_img) return;
    const int b = blockIdx.y;
    const int cv = idx % CV;
    const int q = idx / CV;
    const int r = q / g.W, c = q - r * g.W;
    const int C8 = CV * V;
    float acc[8 * V];
#pragma unroll
    for (int i = 0; i < 8 * V; ++i) acc[i] = 0.f;
    const size_t ybase = (size_t)b * g.Ho * g.Wo * C8 + cv * V;
    int t = 0;
#pragma unroll
    for (int dc = -N; dc <= N; ++dc) {
        const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
        const int oc = c - dc;
        const bool colok = oc >= 0 && (oc % S) == 0 && oc / S < g.Wo;
        const int Cq = oc / S;
        const int po = (oc + g.parity) & 1;
        const int rho = ((S * Cq + g.parity) >> 1) % S;
        const int top = -N + (((dc < 0 ? -dc : dc) + po) >> 1);
#pragma unroll
        for (int k = 0; k < len; ++k, ++t) {
            if (!colok) continue;
            const int d = r - (top + k) - rho;
            if (d < 0 || (d % S) != 0) continue;
            const int Rq = d / S;
            if (Rq >= g.Ho) continue;
            const size_t yo = ybase + (size_t)(Rq * g.Wo + Cq) * C8;
            float inv = 1.f;
            if (mode != HEX_POOL_MAX) {
                const int orow = rho + S * Rq;
                int cntv = 0;
#pragma unroll
                for (int e = -N; e <= N; ++e) {
                    const int ccol = oc + e;
                    if (ccol < 0 || ccol >= g.W) continue;
                    const int l2 = 2 * N + 1 - (e < 0 ? -e : e);
                    const int tp = orow - N + (((e < 0 ? -e : e) + po) >> 1);
                    cntv += max(min(tp + l2, g.H) - max(tp, 0), 0);
                }
                inv = 1.f / (float)cntv;
            }
            const uint32_t tt4 = (uint32_t)t * 0x01010101u;
#pragma unroll
            for (int v = 0; v < V; ++v) {
                const uint4 dq = __ldg(dy + yo + v);
                uint32_t w[4] = {dq.x, dq.y, dq.z, dq.w};
                if (mode == HEX_POOL_MAX) {
                    const uint2 a = __ldg(am + yo + v);
                    const uint32_t mlo = __vcmpeq4(a.x, tt4), mhi = __vcmpeq4(a.y, tt4);
                    w[0] &= __byte_perm(mlo, 0u, 0x1100);
                    w[1] &= __byte_perm(mlo, 0u, 0x3322);
                    w[2] &= __byte_perm(mhi, 0u, 0x1100);
                    w[3] &= __byte_perm(mhi, 0u, 0x3322);
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        acc[8 * v + 2 * kk] += __uint_as_float(w[kk] << 16);
                        acc[8 * v + 2 * kk + 1] += __uint_as_float(w[kk] & 0xffff0000u);
                    }
                } else {
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        acc[8 * v + 2 * kk] += __uint_as_float(w[kk] << 16) * inv;
                        acc[8 * v + 2 * kk + 1] += __uint_as_float(w[kk] & 0xffff0000u) * inv;
                    }
                }
            }
        }
    }
    uint4* out = dx + (size_t)b * per_img * V + (size_t)q * C8 + cv * V;
#pragma unroll
    for (int v = 0; v < V; ++v) {
        uint32_t pk[4];
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
            __nv_bfloat162 h = __floats2bfloat162_rn(acc[8 * v + 2 * kk], acc[8 * v + 2 * kk + 1]);
            pk[kk] = *reinterpret_cast<uint32_t*>(&h);
        }
        out[v] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
}

// ---------------------------------------------------------------------------
// Max-pool backward for the config-5 case n = 1, s = 2 in closed form.  All
// lattice centres sit in even columns 2C with centre parity p = parity & 1 and
// rho(C) = C & 1.  An input pixel (r, c) is reached by:
//   c even: the window of column c/2 -- its centre row r (tap 3) when r - rho is
//           even, else the centres r+1 (tap 2) and r-1 (tap 4);
//   c odd : one window on each side, centres in columns c+1 (taps 0,1; dc = -1)
//           and c-1 (taps 5,6; dc = +1), whose row is the one of
//           {r - top, r - top - 1} on the lattice (top = -1 + ((1 + p) >> 1)).
// At most two candidates (their fp32 sum is order independent), each routed
// per channel with SIMD byte compares of the argmax bytes.  8 channels/thread.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void route_add(const uint4* __restrict__ dy, const uint2* __restrict__ am, size_t yo,
                                          int t, float* acc) {
    const uint4 dq = __ldg(dy + yo);
    const uint2 a = __ldg(am + yo);
    const uint32_t tt4 = (uint32_t)t * 0x01010101u;
    const uint32_t mlo = __vcmpeq4(a.x, tt4), mhi = __vcmpeq4(a.y, tt4);
    const uint32_t w0 = dq.x & __byte_perm(mlo, 0u, 0x1100), w1 = dq.y & __byte_perm(mlo, 0u, 0x3322);
    const uint32_t w2 = dq.z & __byte_perm(mhi, 0u, 0x1100), w3 = dq.w & __byte_perm(mhi, 0u, 0x3322);
    acc[0] += __uint_as_float(w0 << 16); acc[1] += __uint_as_float(w0 & 0xffff0000u);
    acc[2] += __uint_as_float(w1 << 16); acc[3] += __uint_as_float(w1 & 0xffff0000u);
    acc[4] += __uint_as_float(w2 << 16); acc[5] += __uint_as_float(w2 & 0xffff0000u);
    acc[6] += __uint_as_float(w3 << 16); acc[7] += __uint_as_float(w3 & 0xffff0000u);
}

template <int V>
__device__ __forceinline__ void route_add_v(const uint4* __restrict__ dy, const uint2* __restrict__ am, size_t yo,
                                            int t, float* acc) {
#pragma unroll
    for (int v = 0; v < V; ++v) route_add(dy, am, yo + v, t, acc + 8 * v);
}

template <int V>
__global__ void __launch_bounds__(256)
maxpool_bwd_n1s2_kernel(const uint4* __restrict__ dy, const uint2* __restrict__ am, uint4* __restrict__ dx, Geom g,
                        int C8, int lgcv) {
    // grid: x = (input column, channel group) within row r = blockIdx.y of image b = blockIdx.z
    const int CV = C8 / V;
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= g.W * CV) return;
    const int b = blockIdx.z;
    const int r = blockIdx.y;
    const int cv = lgcv >= 0 ? (idx & (CV - 1)) : idx % CV;
    const int ci = lgcv >= 0 ? (idx >> lgcv) : idx / CV;
    // even columns first, then odd ones: a warp never mixes the two closed-form branches
    const int half = (g.W + 1) >> 1;
    const int c = ci < half ? 2 * ci : 2 * (ci - half) + 1;
    const int ch8 = cv * V;
    const int per_img = g.H * g.W * C8;
    const int q = r * g.W + c;
    const size_t ybase = (size_t)b * g.Ho * g.Wo * C8 + ch8;
    float acc[8 * V];
#pragma unroll
    for (int i = 0; i < 8 * V; ++i) acc[i] = 0.f;
    if ((c & 1) == 0) {
        const int C = c >> 1;
        if (C < g.Wo) {
            const int rho = C & 1;
            const int d = r - rho;
            if ((d & 1) == 0) {
                if (d >= 0 && (d >> 1) < g.Ho) route_add_v<V>(dy, am, ybase + (size_t)((d >> 1) * g.Wo + C) * C8, 3, acc);
            } else {
                const int Ra = (d + 1) >> 1;  // centre r + 1, tap 2 (dr = -1)
                if (d + 1 >= 0 && Ra < g.Ho) route_add_v<V>(dy, am, ybase + (size_t)(Ra * g.Wo + C) * C8, 2, acc);
                const int Rb = (d - 1) >> 1;  // centre r - 1, tap 4 (dr = +1)
                if (d - 1 >= 0 && Rb < g.Ho) route_add_v<V>(dy, am, ybase + (size_t)(Rb * g.Wo + C) * C8, 4, acc);
            }
        }
    } else {
        const int p = g.parity & 1;
        const int top = -1 + ((1 + p) >> 1);
        // right centre column c + 1 (dc = -1, taps 0, 1)
        if (c + 1 < g.W) {
            const int C = (c + 1) >> 1;
            if (C < g.Wo) {
                const int rho = C & 1;
                const int k = ((r - top - rho) & 1);  // 0: dr = top is on the lattice, 1: dr = top + 1
                const int ro = r - top - k;
                const int d = ro - rho;
                if (d >= 0 && (d >> 1) < g.Ho) route_add_v<V>(dy, am, ybase + (size_t)((d >> 1) * g.Wo + C) * C8, k, acc);
            }
        }
        // left centre column c - 1 (dc = +1, taps 5, 6)
        {
            const int C = (c - 1) >> 1;
            if (C < g.Wo) {
                const int rho = C & 1;
                const int k = ((r - top - rho) & 1);
                const int ro = r - top - k;
                const int d = ro - rho;
                if (d >= 0 && (d >> 1) < g.Ho)
                    route_add_v<V>(dy, am, ybase + (size_t)((d >> 1) * g.Wo + C) * C8, 5 + k, acc);
            }
        }
    }
#pragma unroll
    for (int v = 0; v < V; ++v) {
        uint4 out;
        uint32_t* o = reinterpret_cast<uint32_t*>(&out);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            __nv_bfloat162 h = __floats2bfloat162_rn(acc[8 * v + 2 * k], acc[8 * v + 2 * k + 1]);
            o[k] = *reinterpret_cast<uint32_t*>(&h);
        }
        dx[(size_t)b * per_img + (size_t)q * C8 + ch8 + v] = out;
    }
}

// ---------------------------------------------------------------------------
// Max-pool backward, n = 1, s = 2, output-block form: one thread owns the 2x2
// input block rows {2R', 2R'+1} x columns {2C, 2C+1} (8 channels).  All of
// the block's candidate windows lie in window columns C, C+1 and rows
// R'-1..R'+1; which (window, tap) reaches which pixel depends only on the
// centre parity P = parity and rho(C) = C & 1 (lattice rho(C) =
// floor((2C + parity) / 2) mod 2), so each of the four (P, rho) cases is a
// compile-time table: every needed window is loaded once (dy 16 B + argmax
// 8 B) and routed to its pixels with SIMD byte compares; a pixel reached by
// two windows adds the two routed values (bf16x2 add = RNE of the exact sum,
// the same value as the fp32 sum rounded once).  Columns are visited even C
// first, then odd C, so rho is warp-uniform.
// ---------------------------------------------------------------------------
// dy masked to the channels whose argmax byte equals `tap`
__device__ __forceinline__ uint4 route_mask(uint4 d, uint2 a, int tap) {
    const uint32_t tt4 = (uint32_t)tap * 0x01010101u;
    const uint32_t mlo = __vcmpeq4(a.x, tt4), mhi = __vcmpeq4(a.y, tt4);
    return make_uint4(d.x & __byte_perm(mlo, 0u, 0x1100), d.y & __byte_perm(mlo, 0u, 0x3322),
                      d.z & __byte_perm(mhi, 0u, 0x1100), d.w & __byte_perm(mhi, 0u, 0x3322));
}
__device__ __forceinline__ uint32_t badd2(uint32_t a, uint32_t b) {
    __nv_bfloat162 r = __hadd2(*reinterpret_cast<__nv_bfloat162*>(&a), *reinterpret_cast<__nv_bfloat162*>(&b));
    return *reinterpret_cast<uint32_t*>(&r);
}

template <int P, int RHO>
__device__ __forceinline__ void maxpool_bwd_blk_body(const uint4* __restrict__ dyb, const uint2* __restrict__ amb,
                                                     uint4* __restrict__ dxb, const Geom& g, int C8, int ch8, int Rp,
                                                     int C) {
    // windows (dC, dR) in {0,1} x {-1,0,1}; unused ones are compiled out
    uint4 d[2][3];
    uint2 a[2][3];
#pragma unroll
    for (int dC = 0; dC < 2; ++dC)
#pragma unroll
        for (int dR = -1; dR <= 1; ++dR) {
            d[dC][dR + 1] = make_uint4(0u, 0u, 0u, 0u);
            a[dC][dR + 1] = make_uint2(0xffffffffu, 0xffffffffu);  // no tap matches
            if (blk_uses(P, RHO, dC, dR)) {
                const int Cw = C + dC, Rw = Rp + dR;
                if (Cw < g.Wo && Rw >= 0 && Rw < g.Ho) {
                    const size_t o = (size_t)(Rw * g.Wo + Cw) * C8 + ch8;
                    d[dC][dR + 1] = __ldg(dyb + o);
                    a[dC][dR + 1] = __ldg(amb + o);
                }
            }
        }
#pragma unroll
    for (int pc = 0; pc < 2; ++pc)
#pragma unroll
        for (int pr = 0; pr < 2; ++pr) {
            const int r = 2 * Rp + pr, c = 2 * C + pc;
            if (r >= g.H || c >= g.W) continue;
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            const Cand c0 = blk_cand(P, RHO, pc, pr, 0), c1 = blk_cand(P, RHO, pc, pr, 1);
            if (c0.tap >= 0) v = route_mask(d[c0.dC][c0.dR + 1], a[c0.dC][c0.dR + 1], c0.tap);
            if (c1.tap >= 0) {
                const uint4 u = route_mask(d[c1.dC][c1.dR + 1], a[c1.dC][c1.dR + 1], c1.tap);
                v = make_uint4(badd2(v.x, u.x), badd2(v.y, u.y), badd2(v.z, u.z), badd2(v.w, u.w));
            }
            dxb[(size_t)(r * g.W + c) * C8 + ch8] = v;
        }
}

template <int P>
__global__ void __launch_bounds__(256)
maxpool_bwd_n1s2_blk_kernel(const uint4* __restrict__ dy, const uint2* __restrict__ am, uint4* __restrict__ dx, Geom g,
                            int C8, int lgc8) {
    // grid: x = (block column in even-then-odd order, channel group), y = block row R', z = image
    const int idx = blockIdx.x * blockDim.x + threadIdx.x;
    const int nC = g.Wo;  // = ceil(W / 2) block columns
    if (idx >= nC * C8) return;
    const int ch8 = lgc8 >= 0 ? (idx & (C8 - 1)) : idx % C8;
    const int ci = lgc8 >= 0 ? (idx >> lgc8) : idx / C8;
    const int half = (nC + 1) >> 1;
    const int C = ci < half ? 2 * ci : 2 * (ci - half) + 1;
    const int b = blockIdx.z, Rp = blockIdx.y;
    const size_t yimg = (size_t)b * g.Ho * g.Wo * C8, ximg = (size_t)b * g.H * g.W * C8;
    if (C & 1)
        maxpool_bwd_blk_body<P, 1>(dy + yimg, am + yimg, dx + ximg, g, C8, ch8, Rp, C);
    else
        maxpool_bwd_blk_body<P, 0>(dy + yimg, am + yimg, dx + ximg, g, C8, ch8, Rp, C);
}

static int ilog2_exact(int v) {  // log2(v) if v is a power of two, else -1
    if (v <= 0 || (v & (v - 1))) return -1;
    int l = 0;
    while ((1 << l) < v) ++l;
    return l;
}

static int pick_v(const PoolArgs& a) {
    int v = a.C % 16 == 0 ? 2 : 1;  // 16 channels/thread measured best (occupancy vs index reuse)
    const int want = sw_int("HEXCONV_POOL_V", 0);  // development override
    if ((want == 1 || want == 2 || want == 4) && a.C % (8 * want) == 0) v = want;
    return v;
}

template <int N, int S, int V>
static void launch_v_fwd(const PoolArgs& a, cudaStream_t st) {
    const int CV = a.C / (8 * V);
    dim3 grid(ceil_div((int64_t)a.g.Ho * a.g.Wo * CV, 256), a.g.B);
    if (a.mode == HEX_POOL_MAX)
        pool_fwd_nhwc_v<N, S, V, true><<<grid, 256, 0, st>>>((const uint4*)a.x, (uint4*)a.y, (uint2*)a.argmax, a.g,
                                                             CV, ilog2_exact(CV));
    else
        pool_fwd_nhwc_v<N, S, V, false><<<grid, 256, 0, st>>>((const uint4*)a.x, (uint4*)a.y, (uint2*)a.argmax, a.g,
                                                              CV, ilog2_exact(CV));
}
template <int N, int S, int V>
static void launch_v_bwd(const PoolArgs& a, cudaStream_t st) {
    const int CV = a.C / (8 * V);
    dim3 grid(ceil_div((int64_t)a.g.H * a.g.W * CV, 256), a.g.B);
    pool_bwd_nhwc_v<N, S, V><<<grid, 256, 0, st>>>((const uint4*)a.dy, (const uint2*)a.argmax_in, (uint4*)a.dx, a.g,
                                                   CV, a.mode);
}
template <int V>
static void dispatch_v(const PoolArgs& a, cudaStream_t st, bool fwd) {
    if (a.g.n == 1) {
        if (a.g.s == 1) { fwd ? launch_v_fwd<1, 1, V>(a, st) : launch_v_bwd<1, 1, V>(a, st); }
        else { fwd ? launch_v_fwd<1, 2, V>(a, st) : launch_v_bwd<1, 2, V>(a, st); }
    } else {
        if (a.g.s == 1) { fwd ? launch_v_fwd<2, 1, V>(a, st) : launch_v_bwd<2, 1, V>(a, st); }
        else { fwd ? launch_v_fwd<2, 2, V>(a, st) : launch_v_bwd<2, 2, V>(a, st); }
    }
}
static bool dispatch_wide(const PoolArgs& a, cudaStream_t st, bool fwd) {
    const int V = pick_v(a);
    if (V == 1) return false;
    if (V == 4) dispatch_v<4>(a, st, fwd);
    else dispatch_v<2>(a, st, fwd);
    return true;
}

hex_status_t pool_fwd(const PoolArgs& a, cudaStream_t st) {
    if (a.mode == HEX_POOL_AVG_PAD) {  // include-pad average: the generic kernel only
        const int64_t total = (int64_t)a.g.B * a.C * a.g.Ho * a.g.Wo;
        const int cf = a.layout == HEX_NHWC;
        if (a.dtype == HEX_F32)
            pool_fwd_kernel<float><<<ceil_div(total, 256), 256, 0, st>>>(
                (const float*)a.x, (float*)a.y, nullptr, a.g, a.C, a.sx, a.sy, a.mode, cf);
        else
            pool_fwd_kernel<__nv_bfloat16><<<ceil_div(total, 256), 256, 0, st>>>(
                (const __nv_bfloat16*)a.x, (__nv_bfloat16*)a.y, nullptr, a.g, a.C, a.sx, a.sy, a.mode, cf);
    } else if (pool_tma_fwd_supported(a)) {
        return pool_tma_fwd(a, st);
    } else if (pool_n1s2_nchw_supported(a)) {
        return pool_n1s2_nchw_fwd(a, st);
    } else if (use_spec(a) && dispatch_wide(a, st, true)) {
    } else if (use_spec(a)) {
        if (a.g.n == 1) { if (a.g.s == 1) launch_spec_fwd<1, 1>(a, st); else launch_spec_fwd<1, 2>(a, st); }
        else { if (a.g.s == 1) launch_spec_fwd<2, 1>(a, st); else launch_spec_fwd<2, 2>(a, st); }
    } else if (pool_plane_fwd(a, st)) {
    } else if (use_vec8(a)) {
        const int C8 = a.C / 8;
        const int64_t total = (int64_t)a.g.B * C8 * a.g.Ho * a.g.Wo;
        pool_fwd_nhwc_bf16x8_kernel<<<ceil_div(total, 256), 256, 0, st>>>(
            (const uint4*)a.x, (uint4*)a.y, (uint64_t*)a.argmax, a.g, C8, a.mode);
    } else {
        const int64_t total = (int64_t)a.g.B * a.C * a.g.Ho * a.g.Wo;
        const int cf = a.layout == HEX_NHWC;
        if (a.dtype == HEX_F32)
            pool_fwd_kernel<float><<<ceil_div(total, 256), 256, 0, st>>>(
                (const float*)a.x, (float*)a.y, a.argmax, a.g, a.C, a.sx, a.sy, a.mode, cf);
        else
            pool_fwd_kernel<__nv_bfloat16><<<ceil_div(total, 256), 256, 0, st>>>(
                (const __nv_bfloat16*)a.x, (__nv_bfloat16*)a.y, a.argmax, a.g, a.C, a.sx, a.sy, a.mode, cf);
    }
    count_launch();
    return last_launch_status();
}

hex_status_t pool_bwd(const PoolArgs& a, cudaStream_t st) {
    // The 8-channel gather measured faster than the wide variant for the backward
    // (round 1: 519 vs 577 us on config-5 pool 1); HEXCONV_POOL_WIDE_BWD selects it.
    if (a.mode == HEX_POOL_AVG_PAD) {
        const int64_t total = (int64_t)a.g.B * a.C * a.g.H * a.g.W;
        const int cf = a.layout == HEX_NHWC;
        if (a.dtype == HEX_F32)
            pool_bwd_kernel<float><<<ceil_div(total, 256), 256, 0, st>>>(
                (const float*)a.dy, nullptr, (float*)a.dx, a.g, a.C, a.sx, a.sy, a.mode, cf);
        else
            pool_bwd_kernel<__nv_bfloat16><<<ceil_div(total, 256), 256, 0, st>>>(
                (const __nv_bfloat16*)a.dy, nullptr, (__nv_bfloat16*)a.dx, a.g, a.C, a.sx, a.sy, a.mode, cf);
    } else if (use_spec(a) && a.mode == HEX_POOL_MAX && a.g.n == 1 && a.g.s == 2 && !sw_on("HEXCONV_POOL_GENERIC") &&
        !sw_on("HEXCONV_POOL_PIXEL_BWD")) {
        const int C8 = a.C / 8;
        dim3 grid(ceil_div((int64_t)a.g.Wo * C8, 256), (a.g.H + 1) / 2, a.g.B);
        if (a.g.parity & 1)
            maxpool_bwd_n1s2_blk_kernel<1><<<grid, 256, 0, st>>>((const uint4*)a.dy, (const uint2*)a.argmax_in,
                                                                 (uint4*)a.dx, a.g, C8, ilog2_exact(C8));
        else
            maxpool_bwd_n1s2_blk_kernel<0><<<grid, 256, 0, st>>>((const uint4*)a.dy, (const uint2*)a.argmax_in,
                                                                 (uint4*)a.dx, a.g, C8, ilog2_exact(C8));
    } else if (use_spec(a) && a.mode == HEX_POOL_MAX && a.g.n == 1 && a.g.s == 2 && !sw_on("HEXCONV_POOL_GENERIC")) {
        const int C8 = a.C / 8;
        const int V = (C8 % 2 == 0 && sw_on("HEXCONV_POOL_BWD_V2")) ? 2 : 1;
        dim3 grid(ceil_div((int64_t)a.g.W * (C8 / V), 256), a.g.H, a.g.B);
        if (V == 2)
            maxpool_bwd_n1s2_kernel<2><<<grid, 256, 0, st>>>((const uint4*)a.dy, (const uint2*)a.argmax_in,
                                                             (uint4*)a.dx, a.g, C8, ilog2_exact(C8 / 2));
        else
            maxpool_bwd_n1s2_kernel<1><<<grid, 256, 0, st>>>((const uint4*)a.dy, (const uint2*)a.argmax_in,
                                                             (uint4*)a.dx, a.g, C8, ilog2_exact(C8));
    } else if (use_spec(a) && sw_on("HEXCONV_POOL_WIDE_BWD") && dispatch_wide(a, st, false)) {
    } else if (use_spec(a)) {
        if (a.g.n == 1) { if (a.g.s == 1) launch_spec_bwd<1, 1>(a, st); else launch_spec_bwd<1, 2>(a, st); }
        else { if (a.g.s == 1) launch_spec_bwd<2, 1>(a, st); else launch_spec_bwd<2, 2>(a, st); }
    } else if (pool_plane_bwd(a, st)) {
    } else if (use_vec8(a)) {
        const int C8 = a.C / 8;
        const int64_t total = (int64_t)a.g.B * C8 * a.g.H * a.g.W;
        pool_bwd_nhwc_bf16x8_kernel<<<ceil_div(total, 256), 256, 0, st>>>(
            (const uint4*)a.dy, (const uint64_t*)a.argmax_in, (uint4*)a.dx, a.g, C8, a.mode);
    } else {
        const int64_t total = (int64_t)a.g.B * a.C * a.g.H * a.g.W;
        const int cf = a.layout == HEX_NHWC;
        if (a.dtype == HEX_F32)
            pool_bwd_kernel<float><<<ceil_div(total, 256), 256, 0, st>>>(
                (const float*)a.dy, a.argmax_in, (float*)a.dx, a.g, a.C, a.sx, a.sy, a.mode, cf);
        else
            pool_bwd_kernel<__nv_bfloat16><<<ceil_div(total, 256), 256, 0, st>>>(
                (const __nv_bfloat16*)a.dy, a.argmax_in, (__nv_bfloat16*)a.dx, a.g, a.C, a.sx, a.sy, a.mode, cf);
    }
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
