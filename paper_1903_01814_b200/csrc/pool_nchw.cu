// pool_nchw.cu -- hexagonal max / average pooling forward with kernel size n = 1 and stride 2 on NCHW
// tensors (BASELINE configs 2 and 3: fp32 planes of 48x48 / 40x40): one thread per output pair with
// float4 row loads (fp32, W % 4 == 0), else one thread per output, consecutive threads on consecutive
// output columns.  HBM-bound: each element moves once; the neighbouring re-reads hit L1.  (The backward
// is the 2x2-block candidate-table kernel of plane_kernels.cu.)
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
constexpr int PN_V4_MAX = 512;  // output-pair kernel: a whole plane per block up to this many threads

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

// fp32, W % 4 == 0 (so Wo = W / 2 is even): one thread per output pair (R, 2k), (R, 2k + 1), whose 14 taps
// lie in input rows 2R-1 .. 2R+2 and columns 4k-1 .. 4k+3: four coalesced float4 row loads (columns
// 4k .. 4k+3) and two scalar loads of column 4k-1 instead of 14 strided scalars; float2 / 2-byte stores.
// Row 2R-1+j is v[j]; with a = -1 (P = 0) or 0 (P = 1):
//   C = 2k   (centre (2R, 4k)):     t0,t1 = col 4k-1 rows 2R+a, 2R+a+1; t2..t4 = v[0..2].x;
//                                   t5,t6 = v[1+a].y, v[2+a].y
//   C = 2k+1 (centre (2R+1, 4k+2)): t0,t1 = v[2+a].y, v[3+a].y; t2..t4 = v[1..3].z;
//                                   t5,t6 = v[2+a].w, v[3+a].w
template <bool MAX>
__device__ __forceinline__ void reduce7(const float* v, const bool* ok, float* out, int* idx) {
    float best = 0.f, sum = 0.f;
    int bt = -1, cnt = 0;
#pragma unroll
    for (int t = 0; t < 7; ++t) {
        if (!ok[t]) continue;
        if (MAX) {
            if (bt < 0 || v[t] > best) { best = v[t]; bt = t; }
        } else {
            sum += v[t];
            ++cnt;
        }
    }
    *out = MAX ? best : sum * (cnt == 7 ? 1.f / 7.f : 1.f / (float)cnt);  // (A8, <= 1 ulp from sum / cnt)
    *idx = bt;
}

template <int P, bool MAX>
__global__ void __launch_bounds__(PN_V4_MAX)
pool_n1s2_fwd_nchw_v4(const float* __restrict__ x, float* __restrict__ y, uint8_t* __restrict__ am, int H, int W,
                      int Ho, int Wo) {
    constexpr int a = P ? 0 : -1;
    const int nk = Wo >> 1;
    const int pl = blockIdx.y;
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= Ho * nk) return;
    const int R = i / nk, k = i - R * nk;
    const float* xp = x + (int64_t)pl * H * W;
    float4 v[4];
    bool rv[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const int r = 2 * R - 1 + j;
        rv[j] = r >= 0 && r < H;
        v[j] = rv[j] ? __ldg(reinterpret_cast<const float4*>(xp + (int64_t)r * W + 4 * k))
                     : make_float4(0.f, 0.f, 0.f, 0.f);
    }
    const bool lok = k > 0;
    const bool l0 = lok && rv[1 + a], l1 = lok && rv[2 + a];
    const float lv0 = l0 ? __ldg(xp + (int64_t)(2 * R + a) * W + 4 * k - 1) : 0.f;
    const float lv1 = l1 ? __ldg(xp + (int64_t)(2 * R + a + 1) * W + 4 * k - 1) : 0.f;
    const float ve[7] = {lv0, lv1, v[0].x, v[1].x, v[2].x, v[1 + a].y, v[2 + a].y};
    const bool oe[7] = {l0, l1, rv[0], rv[1], rv[2], rv[1 + a], rv[2 + a]};
    const float vo[7] = {v[2 + a].y, v[3 + a].y, v[1].z, v[2].z, v[3].z, v[2 + a].w, v[3 + a].w};
    const bool oo[7] = {rv[2 + a], rv[3 + a], rv[1], rv[2], rv[3], rv[2 + a], rv[3 + a]};
    float re, ro;
    int ie, io;
    reduce7<MAX>(ve, oe, &re, &ie);
    reduce7<MAX>(vo, oo, &ro, &io);
    const int64_t yo = ((int64_t)pl * Ho + R) * Wo + 2 * k;
    *reinterpret_cast<float2*>(y + yo) = make_float2(re, ro);
    if (MAX && am) *reinterpret_cast<uint16_t*>(am + yo) = (uint16_t)((uint32_t)ie | ((uint32_t)io << 8));
}

template <typename T, int P>
void launch_fwd(const PoolArgs& a, cudaStream_t st) {
    if (sizeof(T) == 4 && (a.g.W & 3) == 0 && ((uintptr_t)a.x & 15) == 0 && ((uintptr_t)a.y & 7) == 0 &&
        ((uintptr_t)a.argmax & 1) == 0) {
        const int per_plane = a.g.Ho * (a.g.Wo >> 1);
        const int threads = per_plane <= PN_V4_MAX ? (per_plane + 31) / 32 * 32 : PN_THREADS;
        dim3 grid(ceil_div(per_plane, threads), a.g.B * a.C);
        if (a.mode == HEX_POOL_MAX)
            pool_n1s2_fwd_nchw_v4<P, true><<<grid, threads, 0, st>>>((const float*)a.x, (float*)a.y, a.argmax, a.g.H,
                                                                      a.g.W, a.g.Ho, a.g.Wo);
        else
            pool_n1s2_fwd_nchw_v4<P, false><<<grid, threads, 0, st>>>((const float*)a.x, (float*)a.y, nullptr,
                                                                       a.g.H, a.g.W, a.g.Ho, a.g.Wo);
        return;
    }
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
