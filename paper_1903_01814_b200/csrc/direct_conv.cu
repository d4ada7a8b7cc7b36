// direct_conv.cu -- CUDA-core ("stencil") hexagonal convolution kernels.
//
// Used for the small-channel layers (BASELINE configs 1-3 in fp32, config 5
// layer 1 in bf16) and for every shape the tcgen05 path does not take.  Any
// dtype (fp32 / bf16), layout (NCHW / NHWC), kernel size n, stride s and
// parity.  fp32 accumulation, no TF32 (A13).  Deterministic.
//
// Semantics (A3/A4): cross-correlation
// over the hexagonal neighbourhood of each lattice centre, off-grid = 0.
#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {

// ---------------------------------------------------------------------------
// Forward: one thread per output pixel, COB output channels in registers,
// weights of the channel block staged in shared memory as [ci][t][COB]
// (warp-uniform broadcast reads).
// ---------------------------------------------------------------------------
template <typename T, int COB>
__global__ void __launch_bounds__(128)
conv_fwd_direct_kernel(const T* __restrict__ x, const T* __restrict__ w, const float* __restrict__ bias,
                       T* __restrict__ y, Geom g, int Cin, int Cout, Strides4 sx, Strides4 sy,
                       int ci_chunk, int relu) {
    extern __shared__ float wsm[];
    const int co0 = blockIdx.y * COB;
    const int64_t npix = (int64_t)g.B * g.Ho * g.Wo;
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = pix < npix;
    int C = 0, R = 0, b = 0;
    if (active) {
        C = (int)(pix % g.Wo);
        int64_t q = pix / g.Wo;
        R = (int)(q % g.Ho);
        b = (int)(q / g.Ho);
    }
    const int c = g.s * C;
    const int r = hex_rho(C, g.s, g.parity) + g.s * R;
    const int p = (c + g.parity) & 1;
    const int n = g.n, NT = g.T;

    float acc[COB];
#pragma unroll
    for (int j = 0; j < COB; ++j) acc[j] = 0.f;

    for (int ci0 = 0; ci0 < Cin; ci0 += ci_chunk) {
        const int nci = min(ci_chunk, Cin - ci0);
        __syncthreads();
        for (int i = threadIdx.x; i < nci * NT * COB; i += blockDim.x) {
            int j = i % COB;
            int rest = i / COB;
            int t = rest % NT;
            int ci = rest / NT;
            int co = co0 + j;
            wsm[i] = co < Cout ? to_f32(w[((int64_t)co * Cin + ci0 + ci) * NT + t]) : 0.f;
        }
        __syncthreads();
        if (active) {
            for (int ci = 0; ci < nci; ++ci) {
                const T* xp = x + (int64_t)b * sx.b + (int64_t)(ci0 + ci) * sx.c;
                int t = 0;
                for (int dc = -n; dc <= n; ++dc) {
                    const int len = 2 * n + 1 - (dc < 0 ? -dc : dc);
                    const int cc = c + dc;
                    if (cc < 0 || cc >= g.W) { t += len; continue; }
                    int rr = r + tap_top(n, dc, p);
                    for (int k = 0; k < len; ++k, ++t, ++rr) {
                        if (rr < 0 || rr >= g.H) continue;
                        const float v = to_f32(xp[(int64_t)rr * sx.h + (int64_t)cc * sx.w]);
                        const float* wp = wsm + (ci * NT + t) * COB;
#pragma unroll
                        for (int j = 0; j < COB; ++j) acc[j] = fmaf(v, wp[j], acc[j]);
                    }
                }
            }
        }
    }
    if (!active) return;
    T* yp = y + (int64_t)b * sy.b + (int64_t)R * sy.h + (int64_t)C * sy.w;
#pragma unroll
    for (int j = 0; j < COB; ++j) {
        const int co = co0 + j;
        if (co < Cout) {
            float v = acc[j] + (bias ? bias[co] : 0.f);
            if (relu) v = fmaxf(v, 0.f);
            yp[(int64_t)co * sy.c] = from_f32<T>(v);
        }
    }
}

// ---------------------------------------------------------------------------
// Backward-data (gather form, any stride): one thread per INPUT pixel, CIB
// input channels in registers.  For tap t=(dc, k) the only output centre that
// could have touched this pixel sits in column c-dc; its parity fixes the
// tap's row offset, and it must lie on the stride lattice.
// ---------------------------------------------------------------------------
template <typename T, int CIB>
__global__ void __launch_bounds__(128)
conv_bwd_data_direct_kernel(const T* __restrict__ dy, const T* __restrict__ w, const T* __restrict__ relu_y,
                            T* __restrict__ dx, Geom g, int Cin, int Cout, Strides4 sdy, Strides4 sdx,
                            int co_chunk) {
    extern __shared__ float wsm[];  // [co][t][CIB]
    const int ci0 = blockIdx.y * CIB;
    const int64_t npix = (int64_t)g.B * g.H * g.W;
    const int64_t pix = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const bool active = pix < npix;
    int c = 0, r = 0, b = 0;
    if (active) {
        c = (int)(pix % g.W);
        int64_t q = pix / g.W;
        r = (int)(q % g.H);
        b = (int)(q / g.H);
    }
    const int n = g.n, NT = g.T, s = g.s;

    float acc[CIB];
#pragma unroll
    for (int j = 0; j < CIB; ++j) acc[j] = 0.f;

    for (int co0 = 0; co0 < Cout; co0 += co_chunk) {
        const int nco = min(co_chunk, Cout - co0);
        __syncthreads();
        for (int i = threadIdx.x; i < nco * NT * CIB; i += blockDim.x) {
            int j = i % CIB;
            int rest = i / CIB;
            int t = rest % NT;
            int co = rest / NT;
            int ci = ci0 + j;
            wsm[i] = ci < Cin ? to_f32(w[((int64_t)(co0 + co) * Cin + ci) * NT + t]) : 0.f;
        }
        __syncthreads();
        if (active) {
            int t = 0;
            for (int dc = -n; dc <= n; ++dc) {
                const int len = 2 * n + 1 - (dc < 0 ? -dc : dc);
                const int oc = c - dc;  // centre column
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
                    const T* dyp = dy + (int64_t)b * sdy.b + (int64_t)Rq * sdy.h + (int64_t)Cq * sdy.w +
                                   (int64_t)co0 * sdy.c;
                    for (int co = 0; co < nco; ++co) {
                        const float gv = to_f32(dyp[(int64_t)co * sdy.c]);
                        const float* wp = wsm + (co * NT + t) * CIB;
#pragma unroll
                        for (int j = 0; j < CIB; ++j) acc[j] = fmaf(gv, wp[j], acc[j]);
                    }
                }
            }
        }
    }
    if (!active) return;
    const int64_t base = (int64_t)b * sdx.b + (int64_t)r * sdx.h + (int64_t)c * sdx.w;
#pragma unroll
    for (int j = 0; j < CIB; ++j) {
        const int ci = ci0 + j;
        if (ci < Cin) {
            float v = acc[j];
            const int64_t off = base + (int64_t)ci * sdx.c;
            if (relu_y && !(to_f32(relu_y[off]) > 0.f)) v = 0.f;
            dx[off] = from_f32<T>(v);
        }
    }
}

// ---------------------------------------------------------------------------
// Backward-weight: a GEMM  dW[co][j] = sum_k dy[k][co] * X[k][j]  with
// k = output pixel (b,R,C), j = (ci, t) and one extra column j = Cin*T of
// ones that yields dbias.  64x64 block tile, 4x4 per thread, K staged 32
// pixels at a time through shared memory.  Split-K over fixed pixel chunks:
// partial sums go to ws[chunk][Cout][N], reduced in chunk order afterwards.
// ---------------------------------------------------------------------------
constexpr int WG_BM = 64, WG_BN = 64, WG_BK = 32;

template <typename T>
__global__ void __launch_bounds__(256)
conv_wgrad_direct_kernel(const T* __restrict__ x, const T* __restrict__ dy, float* __restrict__ part,
                         Geom g, int Cin, int Cout, Strides4 sx, Strides4 sdy, int64_t chunk_len) {
    __shared__ float dys[WG_BK][WG_BM + 4];
    __shared__ float xgs[WG_BK][WG_BN + 4];
    const int N = Cin * g.T + 1;
    const int m0 = blockIdx.x * WG_BM;
    const int n0 = blockIdx.y * WG_BN;
    const int chunk = blockIdx.z;
    const int64_t K = (int64_t)g.B * g.Ho * g.Wo;
    const int64_t kbeg = (int64_t)chunk * chunk_len;
    const int64_t kend = min(K, kbeg + chunk_len);
    const int tid = threadIdx.x;
    const int tm = tid / 16, tn = tid % 16;
    float acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0.f;
    const bool dy_chan_fast = (sdy.c == 1);

    for (int64_t k0 = kbeg; k0 < kend; k0 += WG_BK) {
        __syncthreads();
        // stage dy[k][m]
        for (int i = tid; i < WG_BK * WG_BM; i += 256) {
            int kk, mm;
            if (dy_chan_fast) { mm = i % WG_BM; kk = i / WG_BM; }
            else { kk = i % WG_BK; mm = i / WG_BK; }
            const int64_t k = k0 + kk;
            const int co = m0 + mm;
            float v = 0.f;
            if (k < kend && co < Cout) {
                const int C = (int)(k % g.Wo);
                const int64_t q = k / g.Wo;
                const int R = (int)(q % g.Ho);
                const int b = (int)(q / g.Ho);
                v = to_f32(dy[(int64_t)b * sdy.b + (int64_t)co * sdy.c + (int64_t)R * sdy.h + (int64_t)C * sdy.w]);
            }
            dys[kk][mm] = v;
        }
        // stage gathered x[k][j]
        for (int i = tid; i < WG_BK * WG_BN; i += 256) {
            const int kk = i % WG_BK, nn = i / WG_BK;
            const int64_t k = k0 + kk;
            const int j = n0 + nn;
            float v = 0.f;
            if (k < kend && j < N) {
                if (j == N - 1) {
                    v = 1.f;
                } else {
                    const int ci = j / g.T, t = j % g.T;
                    const int C = (int)(k % g.Wo);
                    const int64_t q = k / g.Wo;
                    const int R = (int)(q % g.Ho);
                    const int b = (int)(q / g.Ho);
                    const int c = g.s * C;
                    const int r = hex_rho(C, g.s, g.parity) + g.s * R;
                    int dc, dr;
                    tap_offset(g.n, (c + g.parity) & 1, t, &dc, &dr);
                    const int rr = r + dr, cc = c + dc;
                    if (rr >= 0 && rr < g.H && cc >= 0 && cc < g.W)
                        v = to_f32(x[(int64_t)b * sx.b + (int64_t)ci * sx.c + (int64_t)rr * sx.h + (int64_t)cc * sx.w]);
                }
            }
            xgs[kk][nn] = v;
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < WG_BK; ++kk) {
            float a[4], bb[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = dys[kk][tm * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) bb[j] = xgs[kk][tn * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], bb[j], acc[i][j]);
        }
    }
    float* pp = part + (int64_t)chunk * Cout * N;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int co = m0 + tm * 4 + i;
        if (co >= Cout) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int jj = n0 + tn * 4 + j;
            if (jj < N) pp[(int64_t)co * N + jj] = acc[i][j];
        }
    }
}

// Fixed-order reduction of the split-K partials.
__global__ void wgrad_reduce_kernel(const float* __restrict__ part, int nchunks, int Cout, int N,
                                    float* __restrict__ dw, float* __restrict__ dbias, int accumulate) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)Cout * N;
    if (idx >= total) return;
    float s = 0.f;
    for (int ch = 0; ch < nchunks; ++ch) s += part[(int64_t)ch * total + idx];
    const int co = (int)(idx / N), j = (int)(idx % N);
    if (j == N - 1) {
        if (dbias) dbias[co] = accumulate ? dbias[co] + s : s;
    } else {
        float* d = dw + (int64_t)co * (N - 1) + j;
        *d = accumulate ? *d + s : s;
    }
}

// ---------------------------------------------------------------------------
// Host launchers
// ---------------------------------------------------------------------------
template <typename T>
static hex_status_t launch_fwd_T(const DirectConvArgs& a, cudaStream_t st) {
    const int taps = a.g.T;
    int cob = a.Cout <= 4 ? 4 : a.Cout <= 8 ? 8 : a.Cout <= 16 ? 16 : a.Cout <= 32 ? 32 : 64;
    if (sizeof(T) == 4 && cob > 32) cob = 32;
    int ci_chunk = (48 * 1024 / 4) / (taps * cob);
    if (ci_chunk < 1) ci_chunk = 1;
    if (ci_chunk > a.Cin) ci_chunk = a.Cin;
    const size_t smem = (size_t)ci_chunk * taps * cob * sizeof(float);
    const int64_t npix = (int64_t)a.g.B * a.g.Ho * a.g.Wo;
    dim3 grid(ceil_div(npix, 128), ceil_div(a.Cout, cob));
    const T* x = (const T*)a.x;
    const T* w = (const T*)a.w;
    T* y = (T*)a.y;
#define HEX_LAUNCH_FWD(CB)                                                                              \
    conv_fwd_direct_kernel<T, CB><<<grid, 128, smem, st>>>(x, w, a.bias, y, a.g, a.Cin, a.Cout, a.sx, \
                                                           a.sy, ci_chunk, a.relu)
    switch (cob) {
        case 4: HEX_LAUNCH_FWD(4); break;
        case 8: HEX_LAUNCH_FWD(8); break;
        case 16: HEX_LAUNCH_FWD(16); break;
        case 32: HEX_LAUNCH_FWD(32); break;
        default: HEX_LAUNCH_FWD(64); break;
    }
#undef HEX_LAUNCH_FWD
    count_launch();
    return last_launch_status();
}

hex_status_t direct_conv_fwd(const DirectConvArgs& a, cudaStream_t st) {
    return a.dtype == HEX_F32 ? launch_fwd_T<float>(a, st) : launch_fwd_T<__nv_bfloat16>(a, st);
}

template <typename T>
static hex_status_t launch_bwd_data_T(const DirectConvArgs& a, cudaStream_t st) {
    const int taps = a.g.T;
    int cib = a.Cin <= 4 ? 4 : a.Cin <= 8 ? 8 : a.Cin <= 16 ? 16 : 32;
    int co_chunk = (48 * 1024 / 4) / (taps * cib);
    if (co_chunk < 1) co_chunk = 1;
    if (co_chunk > a.Cout) co_chunk = a.Cout;
    const size_t smem = (size_t)co_chunk * taps * cib * sizeof(float);
    const int64_t npix = (int64_t)a.g.B * a.g.H * a.g.W;
    dim3 grid(ceil_div(npix, 128), ceil_div(a.Cin, cib));
    const T* dy = (const T*)a.dy;
    const T* w = (const T*)a.w;
    const T* ry = (const T*)a.relu_y;
    T* dx = (T*)a.dx;
#define HEX_LAUNCH_BWD(CB)                                                                           \
    conv_bwd_data_direct_kernel<T, CB><<<grid, 128, smem, st>>>(dy, w, ry, dx, a.g, a.Cin, a.Cout, \
                                                                a.sy, a.sx, co_chunk)
    switch (cib) {
        case 4: HEX_LAUNCH_BWD(4); break;
        case 8: HEX_LAUNCH_BWD(8); break;
        case 16: HEX_LAUNCH_BWD(16); break;
        default: HEX_LAUNCH_BWD(32); break;
    }
#undef HEX_LAUNCH_BWD
    count_launch();
    return last_launch_status();
}

hex_status_t direct_conv_bwd_data(const DirectConvArgs& a, cudaStream_t st) {
    return a.dtype == HEX_F32 ? launch_bwd_data_T<float>(a, st) : launch_bwd_data_T<__nv_bfloat16>(a, st);
}

// Split-K plan: a deterministic function of the problem shape only.
void direct_wgrad_plan(const Geom& g, int Cin, int Cout, int* nchunks, int64_t* chunk_len) {
    const int N = Cin * g.T + 1;
    const int64_t K = (int64_t)g.B * g.Ho * g.Wo;
    const int tiles = ceil_div(Cout, WG_BM) * ceil_div(N, WG_BN);
    int64_t want = (592 + tiles - 1) / tiles;  // ~4 waves of 148 SMs
    int64_t maxch = (K + 255) / 256;          // at least 256 pixels per chunk
    if (want > maxch) want = maxch;
    if (want < 1) want = 1;
    int64_t len = (K + want - 1) / want;
    len = (len + WG_BK - 1) / WG_BK * WG_BK;
    *chunk_len = len;
    *nchunks = (int)((K + len - 1) / len);
}

size_t direct_wgrad_ws_bytes(const Geom& g, int Cin, int Cout) {
    int nch;
    int64_t len;
    direct_wgrad_plan(g, Cin, Cout, &nch, &len);
    return (size_t)nch * Cout * (Cin * g.T + 1) * sizeof(float);
}

template <typename T>
static hex_status_t launch_wgrad_T(const DirectConvArgs& a, float* ws, cudaStream_t st) {
    int nch;
    int64_t len;
    direct_wgrad_plan(a.g, a.Cin, a.Cout, &nch, &len);
    const int N = a.Cin * a.g.T + 1;
    dim3 grid(ceil_div(a.Cout, WG_BM), ceil_div(N, WG_BN), nch);
    conv_wgrad_direct_kernel<T><<<grid, 256, 0, st>>>((const T*)a.x, (const T*)a.dy, ws, a.g, a.Cin, a.Cout,
                                                      a.sx, a.sy, len);
    count_launch();
    const int64_t total = (int64_t)a.Cout * N;
    wgrad_reduce_kernel<<<ceil_div(total, 256), 256, 0, st>>>(ws, nch, a.Cout, N, a.dw, a.dbias, a.accumulate);
    count_launch();
    return last_launch_status();
}

hex_status_t direct_conv_bwd_weight(const DirectConvArgs& a, void* ws, cudaStream_t st) {
    return a.dtype == HEX_F32 ? launch_wgrad_T<float>(a, (float*)ws, st)
                              : launch_wgrad_T<__nv_bfloat16>(a, (float*)ws, st);
}

// Gather-map test hook kernel.
__global__ void gather_map_kernel(int32_t* map, Geom g) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)g.Ho * g.Wo * g.T;
    if (idx >= total) return;
    const int t = (int)(idx % g.T);
    const int64_t o = idx / g.T;
    const int C = (int)(o % g.Wo), R = (int)(o / g.Wo);
    const int c = g.s * C;
    const int r = hex_rho(C, g.s, g.parity) + g.s * R;
    int dc, dr;
    tap_offset(g.n, (c + g.parity) & 1, t, &dc, &dr);
    const int rr = r + dr, cc = c + dc;
    map[idx] = (rr >= 0 && rr < g.H && cc >= 0 && cc < g.W) ? rr * g.W + cc : -1;
}

hex_status_t launch_gather_map(int32_t* map, const Geom& g, cudaStream_t st) {
    const int64_t total = (int64_t)g.Ho * g.Wo * g.T;
    gather_map_kernel<<<ceil_div(total, 256), 256, 0, st>>>(map, g);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
