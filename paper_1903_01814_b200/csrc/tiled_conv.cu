// tiled_conv.cu -- register-blocked fp32 hexagonal convolution for small
// channel counts (BASELINE configs 2-3), stride 1, NCHW.
//
// Forward:  y[b,co,r,c] = bias[co] + sum_ci sum_t w[co,ci,t] x[b,ci,(r,c)+off_t(p)]
// Backward-data at stride 1 is the same computation on dy with
// W'[ci][co][t] = W[co][ci][T-1-t] (oracle pin P18), applied while the weights are
// staged, plus the fused ReLU-backward mask.  fp32 FFMA throughout (no TF32,
// DESIGN.md A13); off-grid neighbours are the zero-filled halo (A4).
//
// Block = output tile of TR x TC pixels (one image) x COB output channels.  Per
// chunk of CIC input channels the zero-padded input tile (TR + 2n rows, TC + 2n
// columns, column-major) and the weight slice [ci][t][co] are staged in shared
// memory.  Each thread owns PR consecutive rows of ONE column (so a single
// column parity and tap table) and CO output channels: per (ci, tap) it issues
// PR scalar + CO/4 vector shared loads for PR*CO FMAs.
#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {

constexpr int TT_CO = 8;

// Tile shapes: TT_TR rows x TT_TC columns, TT_PR rows per thread, NCG groups of 8 output
// channels (COB = 8 NCG).  Chosen per call so the tiles cover the grid (and Cout) without
// idle threads: 8x32 (default), 8x40 (40-wide grids), 20x20 (20x20 grids); NCG = 2 / 4.
template <int N, bool TRANSPOSE, int TT_TR, int TT_TC, int TT_PR, int NCG>
__global__ void __launch_bounds__((TT_TR / TT_PR) * TT_TC * NCG)
tiled_conv_s1_kernel(const float* __restrict__ x, const float* __restrict__ w, const float* __restrict__ bias,
                     const float* __restrict__ relu_y, float* __restrict__ y, int B, int Cin, int Cout, int H, int W,
                     int parity, int relu) {
    constexpr int T = 3 * N * (N + 1) + 1;
    constexpr int TT_THREADS = (TT_TR / TT_PR) * TT_TC * NCG;
    constexpr int TT_COB = NCG * TT_CO;
    constexpr int TT_CIC = N >= 3 ? 4 : 8;  // input channels per staged chunk (static smem < 48 KB)
    constexpr int RH = TT_TR + 2 * N;  // staged rows
    constexpr int CW = TT_TC + 2 * N;  // staged columns
    __shared__ float xs[TT_CIC][CW][RH + 1];               // column-major (+1: bank spread)
    __shared__ __align__(16) float ws[TT_CIC][T][TT_COB];  // [ci][t][co]

    const int tiles_c = (W + TT_TC - 1) / TT_TC;
    const int tile = blockIdx.x;
    const int r0 = (tile / tiles_c) * TT_TR;
    const int c0 = (tile % tiles_c) * TT_TC;
    const int co0 = blockIdx.y * TT_COB;
    const int b = blockIdx.z;

    const int tid = threadIdx.x;
    const int col = tid % TT_TC;                    // output column within the tile
    const int rg = (tid / TT_TC) % (TT_TR / TT_PR); // row group
    const int cg = tid / (TT_TC * (TT_TR / TT_PR)); // channel group (0..NCG-1)
    const int c = c0 + col;
    const int rbase = rg * TT_PR;                   // first output row (tile-relative)
    const int p = (c + parity) & 1;

    float acc[TT_PR][TT_CO];
#pragma unroll
    for (int i = 0; i < TT_PR; ++i)
#pragma unroll
        for (int j = 0; j < TT_CO; ++j) acc[i][j] = 0.f;

    const int64_t plane = (int64_t)H * W;
    for (int ci0 = 0; ci0 < Cin; ci0 += TT_CIC) {
        const int nci = min(TT_CIC, Cin - ci0);
        __syncthreads();
        // stage the zero-padded input tile, column-major
        for (int i = tid; i < nci * RH * CW; i += TT_THREADS) {
            const int cc = i % CW;
            const int rest = i / CW;
            const int rr = rest % RH;
            const int ci = rest / RH;
            const int gr = r0 - N + rr, gc = c0 - N + cc;
            float v = 0.f;
            if (gr >= 0 && gr < H && gc >= 0 && gc < W)
                v = x[((int64_t)b * Cin + ci0 + ci) * plane + (int64_t)gr * W + gc];
            xs[ci][cc][rr] = v;
        }
        // stage the weight slice [ci][t][co]
        for (int i = tid; i < nci * T * TT_COB; i += TT_THREADS) {
            const int co = i % TT_COB;
            const int rest = i / TT_COB;
            const int t = rest % T;
            const int ci = rest / T;
            const int gco = co0 + co, gci = ci0 + ci;
            float v = 0.f;
            if (gco < Cout) {
                if (TRANSPOSE)  // W'[gco][gci][t] = W[gci][gco][T-1-t]; stored W is [Cin'][Cout'][T] = [Cout][Cin][T]
                    v = w[((int64_t)gci * Cout + gco) * T + (T - 1 - t)];
                else
                    v = w[((int64_t)gco * Cin + gci) * T + t];
            }
            ws[ci][t][co] = v;
        }
        __syncthreads();
        for (int ci = 0; ci < nci; ++ci) {
            int t = 0;
#pragma unroll
            for (int dc = -N; dc <= N; ++dc) {
                const int len = 2 * N + 1 - (dc < 0 ? -dc : dc);
                const int top = -N + (((dc < 0 ? -dc : dc) + p) >> 1);
                const float* xcol = &xs[ci][col + N + dc][rbase + N + top];
#pragma unroll
                for (int k = 0; k < len; ++k, ++t) {
                    float xv[TT_PR];
#pragma unroll
                    for (int i = 0; i < TT_PR; ++i) xv[i] = xcol[k + i];
                    const float4 wa = *reinterpret_cast<const float4*>(&ws[ci][t][cg * TT_CO]);
                    const float4 wb = *reinterpret_cast<const float4*>(&ws[ci][t][cg * TT_CO + 4]);
                    const float wv[8] = {wa.x, wa.y, wa.z, wa.w, wb.x, wb.y, wb.z, wb.w};
#pragma unroll
                    for (int i = 0; i < TT_PR; ++i)
#pragma unroll
                        for (int j = 0; j < TT_CO; ++j) acc[i][j] = fmaf(xv[i], wv[j], acc[i][j]);
                }
            }
        }
    }
    if (c >= W) return;
#pragma unroll
    for (int j = 0; j < TT_CO; ++j) {
        const int co = co0 + cg * TT_CO + j;
        if (co >= Cout) continue;
        const float bv = bias ? bias[co] : 0.f;
#pragma unroll
        for (int i = 0; i < TT_PR; ++i) {
            const int r = r0 + rbase + i;
            if (r >= H) continue;
            const int64_t off = ((int64_t)b * Cout + co) * plane + (int64_t)r * W + c;
            float v = acc[i][j] + bv;
            if (relu) v = fmaxf(v, 0.f);
            if (relu_y && !(relu_y[off] > 0.f)) v = 0.f;
            y[off] = v;
        }
    }
}

bool tiled_supported(const Geom& g, int dtype, int layout) {
    return dtype == HEX_F32 && layout == HEX_NCHW && g.s == 1 && g.n <= 3 && !sw_on("HEXCONV_NO_TILED");
}

namespace {
template <int TR, int TC, int PR, int NCG>
hex_status_t launch_tiled(const float* x, const float* w, const float* bias, const float* relu_y, float* y,
                          const Geom& g, int Cin, int Cout, int relu, int transpose, cudaStream_t st) {
    constexpr int threads = (TR / PR) * TC * NCG;
    const int tiles = ceil_div(g.H, TR) * ceil_div(g.W, TC);
    dim3 grid(tiles, ceil_div(Cout, NCG * TT_CO), g.B);
#define HEX_TILED(NN)                                                                                          \
    if (transpose)                                                                                             \
        tiled_conv_s1_kernel<NN, true, TR, TC, PR, NCG><<<grid, threads, 0, st>>>(x, w, bias, relu_y, y, g.B,  \
                                                                                  Cin, Cout, g.H, g.W,         \
                                                                                  g.parity, relu);             \
    else                                                                                                       \
        tiled_conv_s1_kernel<NN, false, TR, TC, PR, NCG><<<grid, threads, 0, st>>>(x, w, bias, relu_y, y, g.B, \
                                                                                   Cin, Cout, g.H, g.W,        \
                                                                                   g.parity, relu);
    switch (g.n) {
        case 0: HEX_TILED(0); break;
        case 1: HEX_TILED(1); break;
        case 2: HEX_TILED(2); break;
        default: HEX_TILED(3); break;
    }
#undef HEX_TILED
    count_launch();
    return last_launch_status();
}

// fraction of computed outputs that are real (tile padding of rows, columns and channels)
double tile_fill(int H, int W, int Cout, int TR, int TC, int COB) {
    return (double)H / (ceil_div(H, TR) * TR) * W / (ceil_div(W, TC) * TC) * Cout / (ceil_div(Cout, COB) * COB);
}
}  // namespace

// transpose = 0: forward (x, w[Cout][Cin][T]); 1: backward-data at stride 1 (x = dy,
// Cin = original Cout, Cout = original Cin, w = the original weights).
hex_status_t tiled_conv(const float* x, const float* w, const float* bias, const float* relu_y, float* y,
                        const Geom& g, int Cin, int Cout, int relu, int transpose, cudaStream_t st) {
    // candidate shapes (rows, cols, channel groups); pick the best-filled, ties -> listed order
    struct Shape { int tr, tc, ncg; };
    const Shape cand[] = {{8, 32, 4}, {8, 40, 4}, {20, 20, 4}, {8, 32, 2}, {8, 40, 2}, {20, 20, 2}};
    int best = 0;
    double bf = -1.0;
    for (int i = 0; i < 6; ++i) {
        const double f = tile_fill(g.H, g.W, Cout, cand[i].tr, cand[i].tc, 8 * cand[i].ncg);
        if (f > bf + 1e-9) { bf = f; best = i; }
    }
    switch (best) {
        case 0: return launch_tiled<8, 32, 4, 4>(x, w, bias, relu_y, y, g, Cin, Cout, relu, transpose, st);
        case 1: return launch_tiled<8, 40, 4, 4>(x, w, bias, relu_y, y, g, Cin, Cout, relu, transpose, st);
        case 2: return launch_tiled<20, 20, 5, 4>(x, w, bias, relu_y, y, g, Cin, Cout, relu, transpose, st);
        case 3: return launch_tiled<8, 32, 4, 2>(x, w, bias, relu_y, y, g, Cin, Cout, relu, transpose, st);
        case 4: return launch_tiled<8, 40, 4, 2>(x, w, bias, relu_y, y, g, Cin, Cout, relu, transpose, st);
        default: return launch_tiled<20, 20, 5, 2>(x, w, bias, relu_y, y, g, Cin, Cout, relu, transpose, st);
    }
}

}  // namespace hexconv
