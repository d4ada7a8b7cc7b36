// plane_kernels.cu -- NCHW kernels that stage whole (image, channel) planes in
// shared memory: hexagonal max / avg pooling (forward, backward) for any dtype,
// and the single-input-channel fp32 convolution (forward, weight gradient) of
// BASELINE config 3 (40x40 camera images, 1 -> 16 channels).
//
// These layers are HBM-bound: every input element is read once from HBM into
// shared memory with coalesced 16-byte loads, every output element written
// once, and the hexagonal neighbourhood gathers (pooling
// PAPER.md:202-205) run against shared memory.  The per-element index work of
// the generic kernels (div/mod decode, per-tap bounds checks against global
// memory) is what kept them at a few percent of HBM bandwidth.
//
// Semantics are those of the generic kernels (A4, A8, A9): conv is a
// cross-correlation with off-grid taps = 0; max pooling takes the first strict
// maximum in canonical tap order and stores its tap index; average pooling
// divides by the number of in-grid taps; backward passes gather over the
// candidate centres (no atomics).
#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "pool_tables.cuh"

namespace hexconv {

namespace {

constexpr int PL_THREADS = 256;
constexpr int PL_MAX_ELEMS = 12288;  // plane elements staged (48 KB of fp32)

template <typename T>
__device__ __forceinline__ void stage_plane(const T* __restrict__ src, float* dst, int n) {
    if (sizeof(T) == 4 && (n & 3) == 0 && ((uintptr_t)src & 15) == 0) {
        const float4* s4 = reinterpret_cast<const float4*>(src);
        for (int i = threadIdx.x; i < (n >> 2); i += blockDim.x) reinterpret_cast<float4*>(dst)[i] = __ldg(s4 + i);
    } else {
        for (int i = threadIdx.x; i < n; i += blockDim.x) dst[i] = to_f32(src[i]);
    }
}

// number of in-grid taps of the window centred at (r, c)
__device__ __forceinline__ int window_count(int n, int H, int W, int parity, int r, int c) {
    const int p = (c + parity) & 1;
    int cnt = 0;
    for (int dc = -n; dc <= n; ++dc) {
        const int cc = c + dc;
        if (cc < 0 || cc >= W) continue;
        const int len = 2 * n + 1 - (dc < 0 ? -dc : dc);
        const int top = r + tap_top(n, dc, p);
        cnt += max(min(top + len, H) - max(top, 0), 0);
    }
    return cnt;
}

}  // namespace

// ---------------------------------------------------------------------------
// Pool forward: grid-stride over planes; per plane the input is staged, every
// thread computes output pixels from shared memory.
// ---------------------------------------------------------------------------
template <typename T, int N, int S>
__global__ void __launch_bounds__(PL_THREADS)
pool_fwd_plane_kernel(const T* __restrict__ x, T* __restrict__ y, uint8_t* __restrict__ am, Geom g, int planes,
                      int pb, int mode) {
    // pb consecutive planes are staged per iteration (more bytes in flight per block)
    extern __shared__ float xs[];
    const int HW = g.H * g.W, HoWo = g.Ho * g.Wo;
    const int ngroups = (planes + pb - 1) / pb;
    for (int grp = blockIdx.x; grp < ngroups; grp += gridDim.x) {
        const int pl0 = grp * pb;
        const int np = min(pb, planes - pl0);
        __syncthreads();
        stage_plane<T>(x + (int64_t)pl0 * HW, xs, np * HW);
        __syncthreads();
        for (int i = threadIdx.x; i < np * HoWo; i += blockDim.x) {
            const int pp = i / HoWo, o = i - pp * HoWo;
            const float* xp = xs + pp * HW;
            const int R = o / g.Wo, C = o - R * g.Wo;
            const int c = S * C;
            const int r = hex_rho(C, S, g.parity) + S * R;
            const int p = (c + g.parity) & 1;
            int t = 0, best = -1, cnt = 0;
            float bv = 0.f, sum = 0.f;
#pragma unroll
            for (int dc = -N; dc <= N; ++dc) {
                const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
                const int cc = c + dc;
                const int top = r + tap_top(N, dc, p);
#pragma unroll
                for (int k = 0; k < len; ++k, ++t) {
                    const int rr = top + k;
                    if (cc < 0 || cc >= g.W || rr < 0 || rr >= g.H) continue;
                    const float v = xp[rr * g.W + cc];
                    if (mode == HEX_POOL_MAX) {
                        if (best < 0 || v > bv) { best = t; bv = v; }
                    } else {
                        sum += v;
                        ++cnt;
                    }
                }
            }
            const int64_t yo = (int64_t)pl0 * HoWo + i;
            if (mode == HEX_POOL_MAX) {
                y[yo] = from_f32<T>(bv);  // exact: staged values are the inputs (fp32 or widened bf16)
                if (am) am[yo] = (uint8_t)best;
            } else {
                y[yo] = from_f32<T>(sum / (float)cnt);
            }
        }
    }
}

// ---------------------------------------------------------------------------
// Pool backward: dy (avg: pre-divided by the window's in-grid count) and the
// argmax plane are staged; every thread gathers its input pixels' candidates.
// ---------------------------------------------------------------------------
template <typename T, int N, int S>
__global__ void __launch_bounds__(PL_THREADS)
pool_bwd_plane_kernel(const T* __restrict__ dy, const uint8_t* __restrict__ am, T* __restrict__ dx, Geom g,
                      int planes, int mode) {
    extern __shared__ float ds[];
    uint8_t* as = reinterpret_cast<uint8_t*>(ds + g.Ho * g.Wo);
    const int HW = g.H * g.W, HoWo = g.Ho * g.Wo;
    constexpr int s = S;
    for (int pl = blockIdx.x; pl < planes; pl += gridDim.x) {
        __syncthreads();
        for (int o = threadIdx.x; o < HoWo; o += blockDim.x) {
            float v = to_f32(dy[(int64_t)pl * HoWo + o]);
            if (mode == HEX_POOL_MAX) {
                as[o] = am[(int64_t)pl * HoWo + o];
            } else {
                const int R = o / g.Wo, C = o - R * g.Wo;
                v = v / (float)window_count(N, g.H, g.W, g.parity, hex_rho(C, s, g.parity) + s * R, s * C);
            }
            ds[o] = v;
        }
        __syncthreads();
        for (int q = threadIdx.x; q < HW; q += blockDim.x) {
            const int r = q / g.W, c = q - r * g.W;
            float acc = 0.f;
            int t = 0;
#pragma unroll
            for (int dc = -N; dc <= N; ++dc) {
                const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
                const int oc = c - dc;  // candidate centre column
                const bool colok = oc >= 0 && oc % s == 0 && oc / s < g.Wo;
                const int Cq = oc / s;
                const int po = (oc + g.parity) & 1;
                const int rho = colok ? hex_rho(Cq, s, g.parity) : 0;
                const int top = tap_top(N, dc, po);
#pragma unroll
                for (int k = 0; k < len; ++k, ++t) {
                    if (!colok) continue;
                    const int d = r - (top + k) - rho;
                    if (d < 0 || d % s != 0) continue;
                    const int Rq = d / s;
                    if (Rq >= g.Ho) continue;
                    const int o = Rq * g.Wo + Cq;
                    if (mode == HEX_POOL_MAX) {
                        if (as[o] == t) acc += ds[o];
                    } else {
                        acc += ds[o];
                    }
                }
            }
            dx[(int64_t)pl * HW + q] = from_f32<T>(acc);
        }
    }
}

// ---------------------------------------------------------------------------
// Pool backward for n = 1, stride 2 (configs 2 and 3), NCHW: one thread per 2x2
// input block of one plane; its candidate windows come from the compile-time
// (parity, rho) tables of pool_tables.cuh and are read straight from global
// memory (neighbouring threads read neighbouring windows: coalesced, L1 reuse).
// max: routed where the stored argmax equals the tap; avg: dy / in-grid count.
// ---------------------------------------------------------------------------
template <typename T, int P, int RHO, bool MAX, bool MASK>
__device__ __forceinline__ void pool_bwd_blk_nchw(const T* __restrict__ dyp, const uint8_t* __restrict__ amp,
                                                  const T* __restrict__ mp, T* __restrict__ dxp, const Geom& g,
                                                  int Rp, int C, float* VOUT = nullptr) {
    float v[2][3];
    int a[2][3];
#pragma unroll
    for (int dC = 0; dC < 2; ++dC)
#pragma unroll
        for (int dR = -1; dR <= 1; ++dR) {
            v[dC][dR + 1] = 0.f;
            a[dC][dR + 1] = -1;
            if (blk_uses(P, RHO, dC, dR)) {
                const int Cw = C + dC, Rw = Rp + dR;
                if (Cw < g.Wo && Rw >= 0 && Rw < g.Ho) {
                    const int o = Rw * g.Wo + Cw;
                    float d = to_f32(dyp[o]);
                    if (MAX) {
                        a[dC][dR + 1] = amp[o];
                    } else {
                        const int rho = Cw & 1;  // = hex_rho(Cw, 2, parity) for parity in {0, 1}
                        const int rc = rho + 2 * Rw, cc = 2 * Cw;
                        // interior windows (the usual case) have all 7 taps in the grid
                        const bool interior = rc >= 1 && rc + 1 < g.H && cc >= 1 && cc + 1 < g.W;
                        // dy / count as dy * (1 / count): one multiply for interior windows (an IEEE division
                        // per window made this kernel instruction-bound); <= 1 ulp from the quotient (A14)
                        d *= interior ? (1.f / 7.f) : 1.f / (float)window_count(1, g.H, g.W, g.parity, rc, cc);
                    }
                    v[dC][dR + 1] = d;
                }
            }
        }
    float out[2][2];
#pragma unroll
    for (int pr = 0; pr < 2; ++pr)
#pragma unroll
        for (int pc = 0; pc < 2; ++pc) {
            float acc = 0.f;
#pragma unroll
            for (int k = 0; k < 2; ++k) {
                const Cand cd = blk_cand(P, RHO, pc, pr, k);
                if (cd.tap < 0) continue;
                const float d = v[cd.dC][cd.dR + 1];
                if (!MAX || a[cd.dC][cd.dR + 1] == cd.tap) acc += d;
            }
            out[pr][pc] = acc;
        }
    if (VOUT) {
#pragma unroll
        for (int pr = 0; pr < 2; ++pr)
#pragma unroll
            for (int pc = 0; pc < 2; ++pc) VOUT[pr * 2 + pc] = out[pr][pc];
        return;
    }
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
        const int r = 2 * Rp + pr;
        if (r >= g.H) continue;
#pragma unroll
        for (int pc = 0; pc < 2; ++pc) {
            const int c = 2 * C + pc;
            if (c >= g.W) continue;
            float acc = out[pr][pc];
            if (MASK && !(to_f32(__ldg(mp + r * g.W + c)) > 0.f)) acc = 0.f;
            dxp[r * g.W + c] = from_f32<T>(acc);
        }
    }
}

// fp32, W % 4 == 0: one thread per pair of 2x2 blocks (window columns C = 2k, 2k + 1 -> input columns
// 4k .. 4k + 3): two float4 stores (and mask loads) per thread instead of four strided scalars
template <int P, bool MAX, bool MASK>
__global__ void __launch_bounds__(PL_THREADS)
pool_bwd_n1s2_nchw_v4_kernel(const float* __restrict__ dy, const uint8_t* __restrict__ am,
                             const float* __restrict__ relu_y, float* __restrict__ dx, Geom g) {
    const int nk = g.W >> 2, nR = (g.H + 1) / 2;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nR * nk) return;
    const int64_t pl = blockIdx.y;
    const int Rp = i / nk, k = i - Rp * nk;
    const float* dyp = dy + pl * g.Ho * g.Wo;
    const uint8_t* amp = MAX ? am + pl * g.Ho * g.Wo : nullptr;
    float e[4], o[4];
    pool_bwd_blk_nchw<float, P, 0, MAX, false>(dyp, amp, nullptr, nullptr, g, Rp, 2 * k, e);
    pool_bwd_blk_nchw<float, P, 1, MAX, false>(dyp, amp, nullptr, nullptr, g, Rp, 2 * k + 1, o);
#pragma unroll
    for (int pr = 0; pr < 2; ++pr) {
        const int r = 2 * Rp + pr;
        if (r >= g.H) break;
        const int64_t off = (pl * g.H + r) * g.W + 4 * k;
        float4 val = make_float4(e[2 * pr], e[2 * pr + 1], o[2 * pr], o[2 * pr + 1]);
        if (MASK) {
            const float4 m = __ldg(reinterpret_cast<const float4*>(relu_y + off));
            val.x = m.x > 0.f ? val.x : 0.f;
            val.y = m.y > 0.f ? val.y : 0.f;
            val.z = m.z > 0.f ? val.z : 0.f;
            val.w = m.w > 0.f ? val.w : 0.f;
        }
        *reinterpret_cast<float4*>(dx + off) = val;
    }
}

template <typename T, int P, bool MAX, bool MASK>
__global__ void __launch_bounds__(PL_THREADS)
pool_bwd_n1s2_nchw_kernel(const T* __restrict__ dy, const uint8_t* __restrict__ am, const T* __restrict__ relu_y,
                          T* __restrict__ dx, Geom g) {
    // grid: (block tiles of one plane, planes); thread = one 2x2 input block (even C first, then odd C)
    const int nC = g.Wo, nR = (g.H + 1) / 2;
    const int half = (nC + 1) >> 1;  // block columns: even C first, then odd C (rho warp-uniform)
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nR * nC) return;
    const int64_t pl = blockIdx.y;
    const int Rp = i / nC, ci = i - Rp * nC;
    const int C = ci < half ? 2 * ci : 2 * (ci - half) + 1;
    const T* dyp = dy + pl * g.Ho * g.Wo;
    const uint8_t* amp = MAX ? am + pl * g.Ho * g.Wo : nullptr;
    const T* mp = MASK ? relu_y + pl * g.H * g.W : nullptr;
    T* dxp = dx + pl * g.H * g.W;
    if (C & 1) pool_bwd_blk_nchw<T, P, 1, MAX, MASK>(dyp, amp, mp, dxp, g, Rp, C);
    else pool_bwd_blk_nchw<T, P, 0, MAX, MASK>(dyp, amp, mp, dxp, g, Rp, C);
}

template <typename T>
static bool launch_bwd_n1s2(const PoolArgs& a, const void* relu_y, cudaStream_t st) {
    const int64_t planes = (int64_t)a.g.B * a.C;
    if (planes > 65535) return false;
    if (sizeof(T) == 4 && (a.g.W & 3) == 0 && a.g.Wo * 2 == a.g.W &&
        (((uintptr_t)a.dx | (uintptr_t)relu_y) & 15) == 0) {  // vectorised pair-of-blocks kernel
        const int per_plane = ((a.g.H + 1) / 2) * (a.g.W / 4);
        dim3 grid(ceil_div(per_plane, PL_THREADS), (unsigned)planes);
        const float* dy = (const float*)a.dy;
        const float* m = (const float*)relu_y;
        float* dx = (float*)a.dx;
        const bool mx = a.mode == HEX_POOL_MAX;
#define HEX_BW4(PP, MX, MK) \
    pool_bwd_n1s2_nchw_v4_kernel<PP, MX, MK><<<grid, PL_THREADS, 0, st>>>(dy, MX ? a.argmax_in : nullptr, m, dx, a.g)
        if (a.g.parity & 1) {
            if (mx) { if (m) HEX_BW4(1, true, true); else HEX_BW4(1, true, false); }
            else { if (m) HEX_BW4(1, false, true); else HEX_BW4(1, false, false); }
        } else {
            if (mx) { if (m) HEX_BW4(0, true, true); else HEX_BW4(0, true, false); }
            else { if (m) HEX_BW4(0, false, true); else HEX_BW4(0, false, false); }
        }
#undef HEX_BW4
        return true;
    }
    const int per_plane = ((a.g.H + 1) / 2) * a.g.Wo;
    dim3 grid(ceil_div(per_plane, PL_THREADS), (unsigned)planes);
    const bool mx = a.mode == HEX_POOL_MAX;
    const T* dy = (const T*)a.dy;
    const T* m = (const T*)relu_y;
    T* dx = (T*)a.dx;
#define HEX_BW(PP, MX, MK) \
    pool_bwd_n1s2_nchw_kernel<T, PP, MX, MK><<<grid, PL_THREADS, 0, st>>>(dy, MX ? a.argmax_in : nullptr, m, dx, a.g)
    if (a.g.parity & 1) {
        if (mx) { if (m) HEX_BW(1, true, true); else HEX_BW(1, true, false); }
        else { if (m) HEX_BW(1, false, true); else HEX_BW(1, false, false); }
    } else {
        if (mx) { if (m) HEX_BW(0, true, true); else HEX_BW(0, true, false); }
        else { if (m) HEX_BW(0, false, true); else HEX_BW(0, false, false); }
    }
#undef HEX_BW
    return true;
}

static bool plane_pool_ok(const PoolArgs& a) {
    if (a.layout != HEX_NCHW || (a.g.n != 1 && a.g.n != 2) || (a.g.s != 1 && a.g.s != 2) || sw_on("HEXCONV_NO_PLANE"))
        return false;
    const int64_t HW = (int64_t)a.g.H * a.g.W;
    return HW <= PL_MAX_ELEMS;
}

static int plane_grid(int64_t planes) {
    const int64_t cap = (int64_t)num_sms() * 8;
    return (int)(planes < cap ? planes : cap);
}

template <typename T, int N, int S>
static void launch_pool_fwd(const PoolArgs& a, cudaStream_t st) {
    const int planes = a.g.B * a.C;
    const int HW = a.g.H * a.g.W;
    int pb = PL_MAX_ELEMS / HW;  // planes staged per iteration (<= 48 KB)
    if (pb > 4) pb = 4;
    if (pb < 1) pb = 1;
    const size_t smem = (size_t)pb * HW * sizeof(float);
    pool_fwd_plane_kernel<T, N, S><<<plane_grid((planes + pb - 1) / pb), PL_THREADS, smem, st>>>(
        (const T*)a.x, (T*)a.y, a.argmax, a.g, planes, pb, a.mode);
}

template <typename T, int N, int S>
static void launch_pool_bwd(const PoolArgs& a, cudaStream_t st) {
    const int planes = a.g.B * a.C;
    const size_t smem = (size_t)a.g.Ho * a.g.Wo * (sizeof(float) + 1) + 16;
    pool_bwd_plane_kernel<T, N, S><<<plane_grid(planes), PL_THREADS, smem, st>>>(
        (const T*)a.dy, a.argmax_in, (T*)a.dx, a.g, planes, a.mode);
}

template <typename T>
static void dispatch_plane(const PoolArgs& a, cudaStream_t st, bool fwd) {
#define HEX_PL(NN, SS) (fwd ? launch_pool_fwd<T, NN, SS>(a, st) : launch_pool_bwd<T, NN, SS>(a, st))
    if (a.g.n == 1) {
        if (a.g.s == 1) HEX_PL(1, 1); else HEX_PL(1, 2);
    } else {
        if (a.g.s == 1) HEX_PL(2, 1); else HEX_PL(2, 2);
    }
#undef HEX_PL
}

bool pool_plane_fwd(const PoolArgs& a, cudaStream_t st) {
    if (!plane_pool_ok(a)) return false;
    if (a.dtype == HEX_F32) dispatch_plane<float>(a, st, true);
    else dispatch_plane<__nv_bfloat16>(a, st, true);
    return true;
}

bool pool_plane_bwd_n1s2(const PoolArgs& a, const void* relu_y, cudaStream_t st) {
    if (a.layout != HEX_NCHW || a.g.n != 1 || a.g.s != 2 || a.mode == HEX_POOL_AVG_PAD ||
        !(a.g.parity == 0 || a.g.parity == 1) || sw_on("HEXCONV_NO_PLANE"))
        return false;
    return a.dtype == HEX_F32 ? launch_bwd_n1s2<float>(a, relu_y, st) : launch_bwd_n1s2<__nv_bfloat16>(a, relu_y, st);
}

bool pool_plane_bwd(const PoolArgs& a, cudaStream_t st) {
    if (!plane_pool_ok(a)) return false;
    if (pool_plane_bwd_n1s2(a, nullptr, st)) return true;
    if (a.dtype == HEX_F32) dispatch_plane<float>(a, st, false);
    else dispatch_plane<__nv_bfloat16>(a, st, false);
    return true;
}

// ---------------------------------------------------------------------------
// Single-input-channel fp32 convolution, stride 1 (config 3 layer 1).
// The layer is small (7 or 19 FMAs per output element) and its tensors live in
// L2, so both kernels are instruction-bound: the design keeps the per-pixel
// instruction count near the FMA count.  A block stages one zero-padded band of
// x (rb rows + an n-row / n-column halo) in shared memory; its 256 threads form
// two channel groups of 128 threads (warp-uniform), each thread holding its
// group's COB channels' taps in registers and walking the band's pixels with
// stride 128 (incremental row / column, no per-pixel division).
//   forward: per pixel T shared-memory taps, COB x T FMAs, COB coalesced stores
//            (one per output plane, 128 consecutive pixels per warp group).
//   weight gradient: persistent blocks over bands; per pixel COB coalesced dy
//            loads, T taps, COB x (T + 1) FMAs into registers (the + 1 is
//            dbias); a fixed xor-shuffle tree per warp, the 4 warps of a group
//            in warp order, then blocks in block order (c1_wgrad_reduce):
//            deterministic.
// ---------------------------------------------------------------------------
constexpr int C1_THREADS = 256;
constexpr int C1_TPG = 128;    // threads per channel group (2 groups per block)
constexpr int C1_MAX_RB = 32;  // rows per forward band (at most)

template <int N>
struct C1Cfg {
    static constexpr int T = 3 * N * (N + 1) + 1;
    static constexpr int COB = N == 1 ? 8 : 4;  // channels per group (registers: COB x T weights / sums)
};

// zero-padded band [(rows + 2N) x (W + 2N)] of image b, rows r0 - N .. r0 + rows + N - 1
template <int N>
__device__ __forceinline__ void c1_stage(const float* __restrict__ x, float* xs, int b, int r0, int rows, int H,
                                         int W) {
    const int Wp = W + 2 * N, nr = rows + 2 * N;
    const float* xb = x + (int64_t)b * H * W;
    for (int rr = threadIdx.x / 32; rr < nr; rr += C1_THREADS / 32) {  // one warp per staged row
        const int r = r0 - N + rr;
        const bool rok = r >= 0 && r < H;
        for (int cc = threadIdx.x % 32; cc < Wp; cc += 32) {
            const int c = cc - N;
            xs[rr * Wp + cc] = (rok && c >= 0 && c < W) ? __ldg(xb + (int64_t)r * W + c) : 0.f;
        }
    }
}

template <int N>
__global__ void __launch_bounds__(C1_THREADS, 2)
c1_fwd_kernel(const float* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
              float* __restrict__ y, int B, int H, int W, int parity, int Cout, int relu, int rb) {
    constexpr int T = C1Cfg<N>::T, COB = C1Cfg<N>::COB;
    extern __shared__ float xs[];  // [(rb + 2N) x (W + 2N)]
    __shared__ float wsh[2 * COB * T + 2 * COB];
    const int Wp = W + 2 * N;
    const int nb = (H + rb - 1) / rb;
    const int b = blockIdx.x / nb, r0 = (blockIdx.x - b * nb) * rb;
    const int rows = min(rb, H - r0);
    const int grp = threadIdx.x / C1_TPG, tg = threadIdx.x % C1_TPG;
    const int cb = blockIdx.y * 2 * COB;  // first channel of the block
    for (int i = threadIdx.x; i < 2 * COB * T; i += C1_THREADS)
        wsh[i] = cb + i / T < Cout ? __ldg(w + (int64_t)cb * T + i) : 0.f;
    if (threadIdx.x < 2 * COB)
        wsh[2 * COB * T + threadIdx.x] = (bias && cb + (int)threadIdx.x < Cout) ? __ldg(bias + cb + threadIdx.x) : 0.f;
    c1_stage<N>(x, xs, b, r0, rows, H, W);
    __syncthreads();
    const int co0 = cb + grp * COB;
    if (co0 >= Cout) return;
    const int nco = min(COB, Cout - co0);
    float wr[T][COB], br[COB];
#pragma unroll
    for (int j = 0; j < COB; ++j) {
        br[j] = wsh[2 * COB * T + grp * COB + j];
#pragma unroll
        for (int t = 0; t < T; ++t) wr[t][j] = wsh[(grp * COB + j) * T + t];
    }
    const int64_t plane = (int64_t)H * W;
    float* yb = y + ((int64_t)b * Cout + co0) * plane + (int64_t)r0 * W;
    const int npx = rows * W;
    int rl = tg / W, c = tg - rl * W;
    const int dq = C1_TPG / W, dcc = C1_TPG - dq * W;
    for (int q = tg; q < npx; q += C1_TPG) {
        const int p = (c + parity) & 1;
        float acc[COB];
#pragma unroll
        for (int j = 0; j < COB; ++j) acc[j] = br[j];
        const float* xc = xs + (rl + N) * Wp + (c + N);
        int t = 0;
#pragma unroll
        for (int dc = -N; dc <= N; ++dc) {
            const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
            const float* xcol = xc + dc + tap_top(N, dc, p) * Wp;
#pragma unroll
            for (int k = 0; k < len; ++k, ++t) {
                const float v = xcol[k * Wp];
#pragma unroll
                for (int j = 0; j < COB; ++j) acc[j] = fmaf(v, wr[t][j], acc[j]);
            }
        }
        if (nco == COB) {
#pragma unroll
            for (int j = 0; j < COB; ++j) yb[j * plane + q] = relu ? fmaxf(acc[j], 0.f) : acc[j];
        } else {
#pragma unroll
            for (int j = 0; j < COB; ++j)
                if (j < nco) yb[j * plane + q] = relu ? fmaxf(acc[j], 0.f) : acc[j];
        }
        rl += dq;
        c += dcc;
        if (c >= W) { c -= W; ++rl; }
    }
}

template <int N>
__global__ void __launch_bounds__(C1_THREADS, 2)
c1_wgrad_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* __restrict__ part, int B, int H,
                int W, int parity, int Cout, int rb) {
    constexpr int T = C1Cfg<N>::T, COB = C1Cfg<N>::COB, NA = T + 1;
    extern __shared__ float sm[];
    const int Wp = W + 2 * N;
    float* xs = sm;                       // [(rb + 2N) x Wp]
    float* red = xs + (rb + 2 * N) * Wp;  // [8 warps][COB * NA]
    const int grp = threadIdx.x / C1_TPG, tg = threadIdx.x % C1_TPG;
    const int co0 = blockIdx.y * 2 * COB + grp * COB;
    const int nco = max(0, min(COB, Cout - co0));
    const int nb = (H + rb - 1) / rb;
    const int64_t plane = (int64_t)H * W;
    const int dq = C1_TPG / W, dcc = C1_TPG - dq * W;
    float acc[COB][NA];
#pragma unroll
    for (int j = 0; j < COB; ++j)
#pragma unroll
        for (int t = 0; t < NA; ++t) acc[j][t] = 0.f;
    for (int band = blockIdx.x; band < B * nb; band += gridDim.x) {
        const int b = band / nb, r0 = (band - b * nb) * rb;
        const int rows = min(rb, H - r0);
        __syncthreads();
        c1_stage<N>(x, xs, b, r0, rows, H, W);
        __syncthreads();
        if (nco == 0) continue;
        const float* dyb = dy + ((int64_t)b * Cout + co0) * plane + (int64_t)r0 * W;
        const int npx = rows * W;
        int rl = tg / W, c = tg - rl * W;
#pragma unroll 2
        for (int q = tg; q < npx; q += C1_TPG) {
            const int p = (c + parity) & 1;
            float g[COB];
#pragma unroll
            for (int j = 0; j < COB; ++j) g[j] = j < nco ? __ldg(dyb + j * plane + q) : 0.f;
            const float* xc = xs + (rl + N) * Wp + (c + N);
            int t = 0;
#pragma unroll
            for (int dc = -N; dc <= N; ++dc) {
                const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
                const float* xcol = xc + dc + tap_top(N, dc, p) * Wp;
#pragma unroll
                for (int k = 0; k < len; ++k, ++t) {
                    const float v = xcol[k * Wp];
#pragma unroll
                    for (int j = 0; j < COB; ++j) acc[j][t] = fmaf(g[j], v, acc[j][t]);
                }
            }
#pragma unroll
            for (int j = 0; j < COB; ++j) acc[j][T] += g[j];
            rl += dq;
            c += dcc;
            if (c >= W) { c -= W; ++rl; }
        }
    }
    // fixed xor-shuffle tree within the warp, then the group's 4 warps in warp order
#pragma unroll
    for (int j = 0; j < COB; ++j)
#pragma unroll
        for (int t = 0; t < NA; ++t) {
            float v = acc[j][t];
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
            acc[j][t] = v;
        }
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    __syncthreads();
    if (lane == 0)
#pragma unroll
        for (int j = 0; j < COB; ++j)
#pragma unroll
            for (int t = 0; t < NA; ++t) red[warp * COB * NA + j * NA + t] = acc[j][t];
    __syncthreads();
    constexpr int WPG = C1_TPG / 32;  // warps per group
    for (int i = threadIdx.x; i < 2 * COB * NA; i += C1_THREADS) {
        const int gi = i / (COB * NA), e = i - gi * (COB * NA);
        const int co = blockIdx.y * 2 * COB + gi * COB + e / NA;
        if (co >= Cout) continue;
        float s = 0.f;
#pragma unroll
        for (int k = 0; k < WPG; ++k) s += red[(gi * WPG + k) * COB * NA + e];
        part[((int64_t)blockIdx.x * Cout + co) * NA + (e % NA)] = s;
    }
}

// One block per output (dw[co][t] or dbias[co]): thread k sums partials k, k + 256, ... and the block
// combines the 256 sums in a fixed shared-memory tree (deterministic).
constexpr int C1R_THREADS = 256;
__global__ void __launch_bounds__(C1R_THREADS)
c1_wgrad_reduce_kernel(const float* __restrict__ part, int nblocks, int Cout, int NA, float* __restrict__ dw,
                       float* __restrict__ dbias, int accumulate) {
    __shared__ float red[C1R_THREADS];
    const int o = blockIdx.x, total = Cout * NA;
    float s = 0.f;
#pragma unroll 4
    for (int k = threadIdx.x; k < nblocks; k += C1R_THREADS) s += part[(int64_t)k * total + o];
    red[threadIdx.x] = s;
    __syncthreads();
    for (int h = C1R_THREADS / 2; h > 0; h >>= 1) {
        if ((int)threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
        __syncthreads();
    }
    if (threadIdx.x != 0) return;
    s = red[0];
    const int co = o / NA, t = o - co * NA;
    if (t == NA - 1) {
        if (dbias) dbias[co] = accumulate ? dbias[co] + s : s;
    } else {
        float* d = dw + (int64_t)co * (NA - 1) + t;
        *d = accumulate ? *d + s : s;
    }
}

static int c1_cgy(const Geom& g, int Cout) { return ceil_div(Cout, 2 * (g.n == 1 ? C1Cfg<1>::COB : C1Cfg<2>::COB)); }

// forward rows per band: about two blocks per SM slot where the batch allows
static int c1_rows(const Geom& g, int cgy) {
    const int64_t slots = (int64_t)num_sms() * 2;
    int nb = (int)((2 * slots + (int64_t)g.B * cgy - 1) / ((int64_t)g.B * cgy));
    if (nb < 1) nb = 1;
    if (nb > g.H) nb = g.H;
    int rb = (g.H + nb - 1) / nb;
    if (rb < 4 && g.H >= 4) rb = 4;
    return rb < C1_MAX_RB ? rb : C1_MAX_RB;
}

static int c1_band_rows(const Geom& g) { return g.H < 16 ? g.H : 16; }  // weight gradient

bool c1_conv_supported(const Geom& g, int Cin, int Cout, int dtype, int layout) {
    if (sw_on("HEXCONV_NO_PLANE")) return false;
    if (dtype != HEX_F32 || layout != HEX_NCHW || Cin != 1 || g.s != 1 || (g.n != 1 && g.n != 2)) return false;
    if (g.B > 65535 * 8 || Cout > 65535) return false;
    const int64_t band = (int64_t)(C1_MAX_RB + 2 * g.n) * (g.W + 2 * g.n);  // the tallest band
    return band * 4 + 8 * 8 * 20 * 4 <= 200 * 1024;
}

static int c1_wgrad_blocks(const Geom& g, int Cout) {
    const int64_t bands = (int64_t)g.B * ((g.H + c1_band_rows(g) - 1) / c1_band_rows(g));
    const int64_t cap = (int64_t)num_sms() * 2 / c1_cgy(g, Cout);
    const int64_t nb = bands < cap ? bands : cap;
    return (int)(nb > 0 ? nb : 1);
}

size_t c1_wgrad_ws_bytes(const Geom& g, int Cout) {
    return (size_t)c1_wgrad_blocks(g, Cout) * Cout * (g.T + 1) * 4;
}

hex_status_t c1_conv_fwd(const float* x, const float* w, const float* bias, float* y, const Geom& g, int Cout,
                         int relu, cudaStream_t st) {
    const int cgy = c1_cgy(g, Cout);
    const int rb = c1_rows(g, cgy);
    const size_t smem = (size_t)(rb + 2 * g.n) * (g.W + 2 * g.n) * 4;
    dim3 grid(g.B * ceil_div(g.H, rb), cgy);
    if (g.n == 1) {
        if (smem > 40 * 1024)
            cudaFuncSetAttribute(c1_fwd_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        c1_fwd_kernel<1><<<grid, C1_THREADS, smem, st>>>(x, w, bias, y, g.B, g.H, g.W, g.parity, Cout, relu, rb);
    } else {
        if (smem > 40 * 1024)
            cudaFuncSetAttribute(c1_fwd_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        c1_fwd_kernel<2><<<grid, C1_THREADS, smem, st>>>(x, w, bias, y, g.B, g.H, g.W, g.parity, Cout, relu, rb);
    }
    count_launch();
    return last_launch_status();
}

hex_status_t c1_conv_wgrad(const float* x, const float* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                           int Cout, void* ws, cudaStream_t st) {
    const int nb = c1_wgrad_blocks(g, Cout);
    const int rb = c1_band_rows(g);
    const int COB = g.n == 1 ? C1Cfg<1>::COB : C1Cfg<2>::COB;
    const size_t smem = ((size_t)(rb + 2 * g.n) * (g.W + 2 * g.n) + (size_t)8 * COB * (g.T + 1)) * 4;
    float* part = (float*)ws;
    dim3 grid(nb, c1_cgy(g, Cout));
    if (g.n == 1) {
        if (smem > 40 * 1024)
            cudaFuncSetAttribute(c1_wgrad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        c1_wgrad_kernel<1><<<grid, C1_THREADS, smem, st>>>(x, dy, part, g.B, g.H, g.W, g.parity, Cout, rb);
    } else {
        if (smem > 40 * 1024)
            cudaFuncSetAttribute(c1_wgrad_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        c1_wgrad_kernel<2><<<grid, C1_THREADS, smem, st>>>(x, dy, part, g.B, g.H, g.W, g.parity, Cout, rb);
    }
    count_launch();
    const int NA = g.T + 1;
    c1_wgrad_reduce_kernel<<<Cout * NA, C1R_THREADS, 0, st>>>(part, nb, Cout, NA, dw, dbias, accumulate);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
