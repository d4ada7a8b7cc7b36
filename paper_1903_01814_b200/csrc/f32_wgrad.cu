// f32_wgrad.cu -- fp32 NCHW hexagonal-convolution weight gradient for the
// small/mid channel layers of BASELINE configs 2-3 (CUDA-core FFMA, stride 1).
//
//   dW[co][ci][t] = sum_px dy[co][px] * x[ci][px + off_t(parity(px))],
//   dbias[co]     = sum_px dy[co][px]
// (off-grid taps = 0, A4; pure fp32 FFMA, A13).
//
// The taps of one kernel column dc are consecutive rows of input column c + dc.
// A thread owns one (input channel, kernel column) pair and CO = 8 output
// channels; it walks each pixel column of a staged band top to bottom, keeping
// the column's 2n+1 tap values in a register sliding window (one new shared
// load per pixel) while the 8 dy values of the pixel arrive as two broadcast
// 16-byte shared loads: 8 x (2n+1) FFMAs per ~3 shared loads.  dbias is a
// separate plane-sum pass (f32_dbias_partial_kernel).  Blocks are
// persistent over image bands; each thread's accumulators are its own outputs,
// written once per block as partials and summed over blocks in a fixed order
// (deterministic).
#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {

namespace {
constexpr int FW_RB = 8;   // rows per band
constexpr int FW_CO = 8;   // output channels per thread
}  // namespace

// grid = (blocks, co tiles); block threads = CIC * (2N+1) * (COT / 8)
template <int N>
__global__ void __launch_bounds__(384, 2)
f32_wgrad_kernel(const float* __restrict__ x, const float* __restrict__ dy, float* __restrict__ part,
                 float* __restrict__ db_part, int B, int Cin, int Cout, int H, int W, int parity, int COT) {
    constexpr int L = 2 * N + 1;  // taps per column slot (short columns compute and drop the extra rows)
    constexpr int T = 3 * N * (N + 1) + 1;
    extern __shared__ __align__(16) float sm[];
    const int RBp = FW_RB + 2 * N;        // staged rows
    const int Wp = W + 2 * N;             // staged columns
    const int xs_ci = Wp * RBp + 1;       // per-channel stride (odd: spreads banks)
    float* xs = sm;                       // [Cin][Wp][RBp] column-major
    float* ds = sm + ((Cin * xs_ci + 3) & ~3);  // [FW_RB * W][COT], 16-byte aligned (integer offset from the
                                                 // shared array keeps the accesses LDS/STS, not generic)

    const int co0 = blockIdx.y * COT;
    const int per_cs = Cin * L;
    const int cs = threadIdx.x / per_cs;            // co subset
    const int rem = threadIdx.x - cs * per_cs;
    const int ci = rem / L, dcs = rem - ci * L;     // kernel column slot dc = dcs - N
    const int dc = dcs - N;
    const int len = L - (dc < 0 ? -dc : dc);
    const int nthreads = blockDim.x;

    float acc[FW_CO][L];
#pragma unroll
    for (int j = 0; j < FW_CO; ++j)
#pragma unroll
        for (int k = 0; k < L; ++k) acc[j][k] = 0.f;

    const int nb = (H + FW_RB - 1) / FW_RB;
    const int64_t HW = (int64_t)H * W;
    for (int band = blockIdx.x; band < B * nb; band += gridDim.x) {
        const int b = band / nb, r0 = (band - b * nb) * FW_RB;
        const int rows = min(FW_RB, H - r0);
        __syncthreads();
        // stage x rows r0-N .. r0+FW_RB-1+N (zero outside), column-major per channel: 4-byte cp.async
        // (zero fill off the grid), all in flight at once instead of one load round trip per element
        const uint32_t xs_s = (uint32_t)__cvta_generic_to_shared(xs);
        for (int i = threadIdx.x; i < Cin * RBp * Wp; i += nthreads) {
            const int c_ = i / (RBp * Wp);
            const int q = i - c_ * RBp * Wp;
            const int rr = q / Wp, cc = q - rr * Wp;  // row-major walk of global memory (coalesced)
            const int r = r0 - N + rr, c = cc - N;
            const bool ok = r >= 0 && r < H && c >= 0 && c < W;
            const float* src = x + ((int64_t)b * Cin + c_) * HW + (ok ? (int64_t)r * W + c : 0);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(xs_s + 4u * (c_ * xs_ci + cc * RBp + rr)),
                         "l"(src), "r"(ok ? 4 : 0)
                         : "memory");
        }
        // stage dy rows r0 .. r0+rows-1 transposed to [pixel][co] (rows beyond the image: 0).  The
        // 16-byte chunks of a pixel row are XOR-swizzled by the pixel index so that consecutive pixels
        // of one channel land in different banks (fewer store conflicts than a plain transpose).
        const uint32_t ds_s = (uint32_t)__cvta_generic_to_shared(ds);
        for (int i = threadIdx.x; i < COT * FW_RB * W; i += nthreads) {
            const int co = i / (FW_RB * W);
            const int q = i - co * FW_RB * W;  // pixel within the band (row-major)
            const int rl = q / W;
            const bool ok = rl < rows && co0 + co < Cout;
            const float* src = dy + ((int64_t)b * Cout + (ok ? co0 + co : 0)) * HW + (ok ? (int64_t)r0 * W + q : 0);
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(
                             ds_s + 4u * (q * COT + ((((co >> 2) ^ q) & (COT / 4 - 1)) << 2) + (co & 3))),
                         "l"(src), "r"(ok ? 4 : 0)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
        __syncthreads();
        const float* xc0 = xs + ci * xs_ci;
        for (int c = 0; c < W; ++c) {
            const int p = (c + parity) & 1;
            const int top = -N + (((dc < 0 ? -dc : dc) + p) >> 1);
            // staged row of image row r0 + rl + top + k is rl + top + k + N
            const float* col = xc0 + (c + dc + N) * RBp + top + N;
            // the column's FW_RB + L - 1 staged values; with the row loop fully unrolled the sliding
            // window is pure register renaming (no moves)
            float colv[FW_RB + L - 1];
#pragma unroll
            for (int k = 0; k < FW_RB + L - 1; ++k) colv[k] = col[k];
#pragma unroll
            for (int rl = 0; rl < FW_RB; ++rl) {
                const int q = rl * W + c;
                const float* dq = ds + q * COT;
                const float4 g0 = *reinterpret_cast<const float4*>(dq + ((((2 * cs) ^ q) & (COT / 4 - 1)) << 2));
                const float4 g1 = *reinterpret_cast<const float4*>(dq + ((((2 * cs + 1) ^ q) & (COT / 4 - 1)) << 2));
                const float g[FW_CO] = {g0.x, g0.y, g0.z, g0.w, g1.x, g1.y, g1.z, g1.w};
#pragma unroll
                for (int j = 0; j < FW_CO; ++j)
#pragma unroll
                    for (int k = 0; k < L; ++k) acc[j][k] = fmaf(g[j], colv[rl + k], acc[j][k]);
            }
        }
    }
    // partials: part[blk][co][ci][t] for this thread's (8 co) x (column taps); dbias from the (ci 0, dc 0) threads
    const int blk = blockIdx.x;
    int tb = 0;
    for (int c_ = -N; c_ < dc; ++c_) tb += L - (c_ < 0 ? -c_ : c_);
#pragma unroll
    for (int j = 0; j < FW_CO; ++j) {
        const int co = co0 + cs * FW_CO + j;
        if (co >= Cout) continue;
        float* pp = part + (((int64_t)blk * Cout + co) * Cin + ci) * T + tb;
#pragma unroll
        for (int k = 0; k < L; ++k)
            if (k < len) pp[k] = acc[j][k];
    }
    (void)db_part;
}

// dbias partials: block (blk, co) sums the dy planes of channel co of images blk, blk + nblk, ...
// (float4 loads, fixed-order block reduction) -> db_part[blk][co], reduced with the dW partials.
__global__ void __launch_bounds__(256)
f32_dbias_partial_kernel(const float* __restrict__ dy, float* __restrict__ db_part, int B, int Cout, int HW,
                         int nblk) {
    __shared__ float red[256];
    const int blk = blockIdx.x, co = blockIdx.y;
    float s = 0.f;
    for (int b = blk; b < B; b += nblk) {
        const float* pl = dy + ((int64_t)b * Cout + co) * HW;
        if ((HW & 3) == 0 && ((uintptr_t)pl & 15) == 0) {
            for (int i = threadIdx.x; i < (HW >> 2); i += blockDim.x) {
                const float4 v = __ldg(reinterpret_cast<const float4*>(pl) + i);
                s += (v.x + v.y) + (v.z + v.w);
            }
        } else {
            for (int i = threadIdx.x; i < HW; i += blockDim.x) s += __ldg(pl + i);
        }
    }
    red[threadIdx.x] = s;
    __syncthreads();
    for (int w = 128; w > 0; w >>= 1) {
        if (threadIdx.x < w) red[threadIdx.x] += red[threadIdx.x + w];
        __syncthreads();
    }
    if (threadIdx.x == 0) db_part[(int64_t)blk * Cout + co] = red[0];
}

// dw[co][ci][t] (+)= sum_blk part[blk][co][ci][t]; dbias likewise (fixed block order)
__global__ void f32_wgrad_reduce_kernel(const float* __restrict__ part, const float* __restrict__ db_part,
                                        int nblk, int64_t n_w, int Cout, float* __restrict__ dw,
                                        float* __restrict__ dbias, int accumulate) {
    const int64_t gid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t o = gid >> 3;
    const int sub = (int)(gid & 7);
    const int64_t total = n_w + (dbias ? Cout : 0);
    float s = 0.f;
    if (o < total) {
        if (o < n_w)
            for (int k = sub; k < nblk; k += 8) s += part[(int64_t)k * n_w + o];
        else
            for (int k = sub; k < nblk; k += 8) s += db_part[(int64_t)k * Cout + (o - n_w)];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (o >= total || sub != 0) return;
    if (o < n_w) dw[o] = accumulate ? dw[o] + s : s;
    else dbias[o - n_w] = accumulate ? dbias[o - n_w] + s : s;
}

// ------------------------------------------------------------------ host side
struct FwPlan {
    int COT, co_tiles, threads, blocks;
    size_t smem;
};

static FwPlan fw_plan(const Geom& g, int Cin, int Cout) {
    FwPlan p{};
    const int L = 2 * g.n + 1;
    p.COT = 0;
    for (int cot = 128; cot >= 8; cot /= 2) {  // largest power-of-two co tile (>= 8) within 512 threads
        if (Cin * L * (cot / 8) <= 384 && Cout % cot == 0) { p.COT = cot; break; }
    }
    if (p.COT == 0) return p;
    p.co_tiles = Cout / p.COT;
    p.threads = Cin * L * (p.COT / 8);
    const int RBp = FW_RB + 2 * g.n, Wp = g.W + 2 * g.n;
    p.smem = ((size_t)Cin * (Wp * RBp + 1) + 4 + (size_t)FW_RB * g.W * p.COT) * sizeof(float);
    const int64_t bands = (int64_t)g.B * ((g.H + FW_RB - 1) / FW_RB);
    int per_sm = (int)((200 * 1024) / (p.smem + 1024));
    if (per_sm < 1) per_sm = 1;
    if (per_sm > 2) per_sm = 2;
    int64_t blocks = (int64_t)num_sms() * per_sm / p.co_tiles;
    if (blocks < 1) blocks = 1;
    if (blocks > bands) blocks = bands;
    p.blocks = (int)blocks;
    return p;
}

bool f32_wgrad_supported(const Geom& g, int Cin, int Cout, int dtype, int layout) {
    if (sw_on("HEXCONV_NO_F32_WGRAD")) return false;
    if (dtype != HEX_F32 || layout != HEX_NCHW || g.s != 1 || (g.n != 1 && g.n != 2)) return false;
    if (Cout % 8 || Cin < 2) return false;
    const FwPlan p = fw_plan(g, Cin, Cout);
    return p.COT > 0 && p.threads >= 64 && p.smem <= 200 * 1024;
}

size_t f32_wgrad_ws_bytes(const Geom& g, int Cin, int Cout) {
    const FwPlan p = fw_plan(g, Cin, Cout);
    return (size_t)p.blocks * ((size_t)Cout * Cin * g.T + Cout) * sizeof(float);
}

hex_status_t f32_wgrad(const float* x, const float* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                       int Cin, int Cout, void* ws, cudaStream_t st) {
    const FwPlan p = fw_plan(g, Cin, Cout);
    float* part = (float*)ws;
    const int64_t n_w = (int64_t)Cout * Cin * g.T;
    float* db_part = part + (int64_t)p.blocks * n_w;
    dim3 grid(p.blocks, p.co_tiles);
    if (g.n == 1) {
        cudaFuncSetAttribute(f32_wgrad_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        cudaFuncSetAttribute(f32_wgrad_kernel<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        f32_wgrad_kernel<1><<<grid, p.threads, p.smem, st>>>(x, dy, part, db_part, g.B, Cin, Cout, g.H, g.W, g.parity,
                                                              p.COT);
    } else {
        cudaFuncSetAttribute(f32_wgrad_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)p.smem);
        cudaFuncSetAttribute(f32_wgrad_kernel<2>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        f32_wgrad_kernel<2><<<grid, p.threads, p.smem, st>>>(x, dy, part, db_part, g.B, Cin, Cout, g.H, g.W, g.parity,
                                                              p.COT);
    }
    count_launch();
    if (dbias) {
        f32_dbias_partial_kernel<<<dim3(p.blocks, Cout), 256, 0, st>>>(dy, db_part, g.B, Cout, g.H * g.W, p.blocks);
        count_launch();
    }
    // the partials of different co tiles were written by different grid.y blocks into the same
    // part[blk] slab (disjoint co ranges), so the reduction runs over grid.x blocks only
    const int64_t outs = n_w + (dbias ? Cout : 0);
    f32_wgrad_reduce_kernel<<<ceil_div(outs * 8, 256), 256, 0, st>>>(part, db_part, p.blocks, n_w, Cout, dw, dbias,
                                                                     accumulate);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
