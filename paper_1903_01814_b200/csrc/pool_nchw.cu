// pool_nchw.cu -- hexagonal max / average pooling forward with kernel size n = 1 and stride 2 on NCHW
// tensors (BASELINE configs 2 and 3: fp32 planes of 48x48 / 40x40), one thread per output, consecutive
// threads on consecutive output columns.  HBM-bound: each element moves once; the neighbouring re-reads hit
// L1.  (The backward is the 2x2-block candidate-table kernel of plane_kernels.cu.)
//
// Geometry (A5, A8, A9).  Output (R, C) is centred at input
// (rho + 2R, 2C) with rho = rho(C) = C & 1 (the stride-2 lattice for either parity), and the centre
// column parity is the grid parity P.  Its 7 taps in canonical order (columns left to right, rows top to
// bottom) are
//   t0 (rc + a, cc - 1), t1 (rc + a + 1, cc - 1), t2 (rc - 1, cc), t3 (rc, cc), t4 (rc + 1, cc),
//   t5 (rc + a, cc + 1), t6 (rc + a + 1, cc + 1),          a = -1 for P = 0, 0 for P = 1.
// Max: first strict maximum over the in-grid taps (uint8 tap index); avg: in-grid sum / in-grid count.
#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {
namespace {

constexpr int PN_THREADS = 128;

template <int P>
__device__ __forceinline__ int win_count(int rc, int cc, int H, int W) {
    constexpr int a = P ? 0 : -1;
    int n = (rc - 1 >= 0) + 1 + (rc + 1 < H);
    const int side = (rc + a >= 0 && rc + a < H) + (rc + a + 1 >= 0 && rc + a + 1 < H);
    n += (cc - 1 >= 0 ? side : 0) + (cc + 1 < W ? side : 0);
    return n;
}

template <typename T>
__device__ __forceinline__ float ld(const T* p) { return to_f32(__ldg(p)); }

template <typename T, int P, bool MAX>
__global__ void __launch_bounds__(PN_THREADS)
pool_n1s2_fwd_nchw(const T* __restrict__ x, T* __restrict__ y, uint8_t* __restrict__ am, int H, int W, int Ho,
                   int Wo) {
    constexpr int a = P ? 0 : -1;
    const int pl = blockIdx.y;
    const int o = blockIdx.x * PN_THREADS + threadIdx.x;
    if (o >= Ho * Wo) return;
    const int R = o / Wo, C = o - R * Wo;
    const int rc = (C & 1) + 2 * R, cc = 2 * C;
    const T* xp = x + (int64_t)pl * H * W;
    const int rr[7] = {rc + a, rc + a + 1, rc - 1, rc, rc + 1, rc + a, rc + a + 1};
    const int cl[7] = {cc - 1, cc - 1, cc, cc, cc, cc + 1, cc + 1};
    float best = 0.f, sum = 0.f;
    int bt = -1, cnt = 0;
#pragma unroll
    for (int t = 0; t < 7; ++t) {
        if ((unsigned)rr[t] >= (unsigned)H || (unsigned)cl[t] >= (unsigned)W) continue;
        const float v = ld(xp + rr[t] * W + cl[t]);
        if (MAX) {
            if (bt < 0 || v > best) { best = v; bt = t; }
        } else {
            sum += v;
            ++cnt;
        }
    }
    const int64_t yo = (int64_t)pl * Ho * Wo + o;
    if (MAX) {
        y[yo] = from_f32<T>(best);
        if (am) am[yo] = (uint8_t)bt;
    } else {
        y[yo] = from_f32<T>(sum / (float)cnt);
    }
}

template <typename T, int P>
void launch_fwd(const PoolArgs& a, cudaStream_t st) {
    dim3 grid(ceil_div((int64_t)a.g.Ho * a.g.Wo, PN_THREADS), a.g.B * a.C);
    if (a.mode == HEX_POOL_MAX)
        pool_n1s2_fwd_nchw<T, P, true><<<grid, PN_THREADS, 0, st>>>((const T*)a.x, (T*)a.y, a.argmax, a.g.H, a.g.W,
                                                                     a.g.Ho, a.g.Wo);
    else
        pool_n1s2_fwd_nchw<T, P, false><<<grid, PN_THREADS, 0, st>>>((const T*)a.x, (T*)a.y, nullptr, a.g.H, a.g.W,
                                                                      a.g.Ho, a.g.Wo);
}

}  // namespace

bool pool_n1s2_nchw_supported(const PoolArgs& a) {
    return a.layout == HEX_NCHW && a.g.n == 1 && a.g.s == 2 && a.mode != HEX_POOL_AVG_PAD &&
           (int64_t)a.g.B * a.C <= 65535 && !sw_on("HEXCONV_POOL_GENERIC");
}

hex_status_t pool_n1s2_nchw_fwd(const PoolArgs& a, cudaStream_t st) {
    if (a.dtype == HEX_F32) {
        if (a.g.parity & 1) launch_fwd<float, 1>(a, st); else launch_fwd<float, 0>(a, st);
    } else {
        if (a.g.parity & 1) launch_fwd<__nv_bfloat16, 1>(a, st); else launch_fwd<__nv_bfloat16, 0>(a, st);
    }
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
