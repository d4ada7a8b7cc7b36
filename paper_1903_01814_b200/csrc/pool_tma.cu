// pool_tma.cu -- hexagonal max pool n = 1, s = 2 (bf16 NHWC, C % 64 == 0) with TMA-staged input
// (the pooling replaces the sub-convolutions, same padding and striding; DESIGN.md
// A8 off-grid cells ignored, A9 first strict maximum in canonical tap order).
//
// The stencil kernels in pool.cu read every input pixel from L2 about 1.75 times with 16-byte loads
// and stall on load latency (ncu: long-scoreboard, 44 % warps active, 61 % of HBM on C5 pool 2).
// Here (grids at least 64 wide) a persistent CTA walks work units (image, 64-channel chunk, band of RB output rows): ONE TMA
// box brings the band's 2RB+2 input rows x (W+2) columns (one -inf column each side) into shared
// memory, double-buffered so the next unit's box streams in while this one is reduced; the windows
// are then reduced from shared memory (3-input VHMNMX, first equal tap = first strict maximum, value
// bits taken from that tap) and written straight to HBM (128 B of y + 64 B of argmax per window).
// Off-grid cells: TMA zero-fills out-of-bounds pixels, so the box's outer columns and any rows
// outside the image are overwritten with -inf before the reduction (a window's centre is in-grid, so
// -inf never wins).  SWIZZLE_128B keeps the 16-byte group reads conflict-free.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hexconv {
namespace {

constexpr int PT_THREADS = 256;
constexpr uint32_t PT_NEG_INF2 = 0xFF80FF80u;

struct PtParams {
    int B, H, W, C, Ho, Wo, parity;
    int RB, nbands, kchunks, units, nbuf;  // nbuf: ring of boxes, nbuf - 1 units prefetched
    int box_rows, box_cols;  // 2RB+2, W+2
    uint16_t* y;
    uint8_t* am;
};

// byte offset of 16-byte group i of box pixel (row, col): TMA SWIZZLE_128B (pixel = one 128-byte row)
__device__ __forceinline__ uint32_t pt_off(int row, int col, int ncols, int i) {
    const uint32_t m = (uint32_t)(row * ncols + col);
    return m * 128u + (((uint32_t)i ^ (m & 7u)) << 4);
}

__global__ void __launch_bounds__(PT_THREADS, 1)
pool_tma_fwd_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ PtParams p, int buf_bytes,
                    uint32_t box_bytes) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* bar = (uint64_t*)(base + p.nbuf * buf_bytes);
    const int tid = threadIdx.x;
    if (tid == 0) {
        for (int i = 0; i < p.nbuf; ++i) ptx::mbar_init(&bar[i], 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x);
    }
    __syncthreads();
    const int pcen = p.parity & 1;
    const int top1 = -1 + pcen;  // first row of the dc = +-1 taps relative to the centre row (tap_top(1, 1, p))
    auto issue = [&](int u, int bi) {
        const int band = u % p.nbands, rest = u / p.nbands;
        const int kc = rest % p.kchunks, b = rest / p.kchunks;
        ptx::mbar_arrive_expect_tx(&bar[bi], box_bytes);
        ptx::tma_load_5d(&map_x, &bar[bi], base + bi * buf_bytes, 0, -1, 2 * band * p.RB - 1, kc, b);
    };
    if (tid == 0)  // prologue: the first nbuf - 1 units of this CTA
        for (int j = 0; j < p.nbuf - 1; ++j) {
            const int u = blockIdx.x + j * gridDim.x;
            if (u < p.units) issue(u, j);
        }
    int it = 0;
    for (int u = blockIdx.x; u < p.units; u += gridDim.x, ++it) {
        const int bi = it % p.nbuf;
        const int nu = u + (p.nbuf - 1) * gridDim.x;
        if (tid == 0 && nu < p.units) {
            ptx::fence_proxy_async();  // generic-proxy reads / -inf writes of that buffer are done
            issue(nu, (it + p.nbuf - 1) % p.nbuf);
        }
        const int band = u % p.nbands, rest = u / p.nbands;
        const int kc = rest % p.kchunks, b = rest / p.kchunks;
        const int r0 = 2 * band * p.RB - 1;  // image row of box row 0
        uint8_t* bx = base + bi * buf_bytes;
        ptx::mbar_wait(&bar[bi], (uint32_t)((it / p.nbuf) & 1));
        // off-grid cells -> -inf: box columns 0 (image column -1) and W+1 (image column W), and rows
        // outside the image
        const uint4 ninf = make_uint4(PT_NEG_INF2, PT_NEG_INF2, PT_NEG_INF2, PT_NEG_INF2);
        for (int e = tid; e < p.box_rows * 2 * 8; e += PT_THREADS) {
            const int i = e & 7, side = (e >> 3) & 1, row = e >> 4;
            *reinterpret_cast<uint4*>(bx + pt_off(row, side ? p.box_cols - 1 : 0, p.box_cols, i)) = ninf;
        }
        for (int row = 0; row < p.box_rows; ++row) {
            const int ir = r0 + row;
            if (ir >= 0 && ir < p.H) continue;
            for (int e = tid; e < p.box_cols * 8; e += PT_THREADS)
                *reinterpret_cast<uint4*>(bx + pt_off(row, e >> 3, p.box_cols, e & 7)) = ninf;
        }
        __syncthreads();
        // windows (R, C), R in [band*RB, band*RB + RB), C in [0, Wo); 8 channels per item
        const int nitems = p.RB * p.Wo * 8;
        for (int w = tid; w < nitems; w += PT_THREADS) {
            const int cg = w & 7, wi = w >> 3;
            const int C = wi % p.Wo, lr = wi / p.Wo;
            const int R = band * p.RB + lr;
            if (R >= p.Ho) continue;
            const int cr = 2 * R + (C & 1);   // centre row (rho(C) = C mod 2 for s = 2)
            const int brow = cr - r0;         // box row of the centre
            const int bcol = 2 * C + 1;       // box column of the centre (box column 0 = image column -1)
            // canonical taps: 0,1 column 2C-1 rows cr+top1, +1; 2,3,4 column 2C rows cr-1..cr+1;
            // 5,6 column 2C+1 rows cr+top1, +1
            uint4 tv[7];
            tv[0] = *reinterpret_cast<const uint4*>(bx + pt_off(brow + top1, bcol - 1, p.box_cols, cg));
            tv[1] = *reinterpret_cast<const uint4*>(bx + pt_off(brow + top1 + 1, bcol - 1, p.box_cols, cg));
            tv[2] = *reinterpret_cast<const uint4*>(bx + pt_off(brow - 1, bcol, p.box_cols, cg));
            tv[3] = *reinterpret_cast<const uint4*>(bx + pt_off(brow, bcol, p.box_cols, cg));
            tv[4] = *reinterpret_cast<const uint4*>(bx + pt_off(brow + 1, bcol, p.box_cols, cg));
            tv[5] = *reinterpret_cast<const uint4*>(bx + pt_off(brow + top1, bcol + 1, p.box_cols, cg));
            tv[6] = *reinterpret_cast<const uint4*>(bx + pt_off(brow + top1 + 1, bcol + 1, p.box_cols, cg));
            uint32_t best[4], ix[4];
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {
                __nv_bfloat162 mx =
                    *reinterpret_cast<const __nv_bfloat162*>(reinterpret_cast<const uint32_t*>(&tv[0]) + kk);
#pragma unroll
                for (int t = 1; t < 7; ++t)
                    mx = __hmax2(mx, *reinterpret_cast<const __nv_bfloat162*>(
                                         reinterpret_cast<const uint32_t*>(&tv[t]) + kk));
                // the first tap equal to the maximum is the first strict maximum; its bits are the value
                best[kk] = reinterpret_cast<const uint32_t*>(&tv[6])[kk];
                ix[kk] = 6u * 0x00010001u;
#pragma unroll
                for (int t = 5; t >= 0; --t) {
                    const uint32_t wv = reinterpret_cast<const uint32_t*>(&tv[t])[kk];
                    const uint32_t mk = __heq2_mask(*reinterpret_cast<const __nv_bfloat162*>(&wv), mx);
                    best[kk] = (wv & mk) | (best[kk] & ~mk);
                    ix[kk] = ((uint32_t)t * 0x00010001u & mk) | (ix[kk] & ~mk);
                }
            }
            const int64_t o = (((int64_t)b * p.Ho + R) * p.Wo + C) * p.C + kc * 64 + cg * 8;
            *reinterpret_cast<uint4*>(p.y + o) = make_uint4(best[0], best[1], best[2], best[3]);
            if (p.am)
                *reinterpret_cast<uint2*>(p.am + o) =
                    make_uint2(__byte_perm(ix[0], ix[1], 0x6420), __byte_perm(ix[2], ix[3], 0x6420));
        }
        ptx::fence_proxy_async();  // this thread's generic accesses precede the next TMA write here
        __syncthreads();           // this buffer is free for the unit after next
    }
}

PFN_cuTensorMapEncodeTiled_v12000 pt_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    return fn;
}

// output rows per unit: the largest band whose double buffer fits, capped at 8
int pt_buf_bytes(int rb, int W) { return (((2 * rb + 2) * (W + 2) * 128) + 1023) & ~1023; }
constexpr int PT_SMEM = 227 * 1024 - 1024 - 128;
// output rows per unit: the largest band (<= 8) whose double buffer fits.  Measured (C5 pools, B200):
// 96-wide grids 174 us with 2 buffers of RB = 3 (stencil 189 us; a 3-box ring of RB = 2 186 us); 48-wide
// grids stay on the stencil kernel (104 us vs 108-121 us here), hence the width threshold.
int pt_band(int W, int* nbuf) {
    *nbuf = 2;
    for (int rb = 8; rb >= 1; --rb)
        if (2 * pt_buf_bytes(rb, W) <= PT_SMEM) return rb;
    return 0;
}

}  // namespace

bool pool_tma_fwd_supported(const PoolArgs& a) {
    if (sw_on("HEXCONV_NO_POOL_TMA") || !pt_encode()) return false;
    const Geom& g = a.g;
    if (a.dtype != HEX_BF16 || a.layout != HEX_NHWC || a.mode != HEX_POOL_MAX || g.n != 1 || g.s != 2) return false;
    const int min_w = sw_int("HEXCONV_POOL_TMA_MIN_W", 64);
    if (a.C % 64 || g.W < min_w || g.W < 2 || g.W + 2 > 256 || g.B < 1) return false;
    if (((uintptr_t)a.x & 15) || ((uintptr_t)a.y & 15) || ((uintptr_t)a.argmax & 7)) return false;
    int nb;
    return pt_band(g.W, &nb) > 0;
}

hex_status_t pool_tma_fwd(const PoolArgs& a, cudaStream_t st) {
    const Geom& g = a.g;
    PtParams p{};
    p.B = g.B; p.H = g.H; p.W = g.W; p.C = a.C; p.Ho = g.Ho; p.Wo = g.Wo; p.parity = g.parity;
    p.RB = pt_band(g.W, &p.nbuf);
    if (p.RB > g.Ho) p.RB = g.Ho;
    p.nbands = ceil_div(g.Ho, p.RB);
    p.kchunks = a.C / 64;
    p.units = g.B * p.kchunks * p.nbands;
    p.box_rows = 2 * p.RB + 2;
    p.box_cols = g.W + 2;
    p.y = (uint16_t*)a.y;
    p.am = a.argmax;
    const int buf_bytes = pt_buf_bytes(p.RB, g.W);
    const int smem = p.nbuf * buf_bytes + 1024 + 64;
    // x as {64 channels, W, H, C/64, B}; box {64, W+2, 2RB+2, 1, 1} from column -1 (zero fill outside)
    CUtensorMap m;
    cuuint64_t dims[5] = {64, (cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)(a.C / 64), (cuuint64_t)g.B};
    cuuint64_t strides[4] = {(cuuint64_t)a.C * 2, (cuuint64_t)g.W * a.C * 2, 128, (cuuint64_t)g.H * g.W * a.C * 2};
    cuuint32_t box[5] = {64, (cuuint32_t)p.box_cols, (cuuint32_t)p.box_rows, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    const CUresult er = pt_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, (void*)a.x, dims, strides, box, es,
                                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (er != CUDA_SUCCESS) {
        if (sw_on("HEXCONV_DEBUG")) fprintf(stderr, "pool_tma: tensor map encode failed (%d)\n", (int)er);
        return HEX_ERR_CUDA;
    }
    if (cudaFuncSetAttribute(pool_tma_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return HEX_ERR_CUDA;
    const int grid = p.units < num_sms() ? p.units : num_sms();
    pool_tma_fwd_kernel<<<grid, PT_THREADS, smem, st>>>(m, p, buf_bytes, (uint32_t)(p.box_rows * p.box_cols * 128));
    count_launch();
    if (sw_on("HEXCONV_DEBUG")) {
        const cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) fprintf(stderr, "pool_tma: launch failed: %s\n", cudaGetErrorString(e));
        return e == cudaSuccess ? HEX_OK : HEX_ERR_CUDA;
    }
    return last_launch_status();
}

}  // namespace hexconv
