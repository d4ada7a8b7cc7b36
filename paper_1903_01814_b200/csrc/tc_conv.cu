// tc_conv.cu -- tcgen05 / TMEM / TMA implicit-GEMM hexagonal convolution for
// sm_100a (bf16 NHWC activations, fp32 accumulation in tensor memory).
//
// Method: y = bias + sum_ci sum_t w[co,ci,t] x[nb_t].
// The paper realises it as n+1 dilated rectangular sub-convolutions per
// column parity; here it is ONE implicit GEMM per column-parity class:
//
//   M = 128 output pixels of one column parity P (a box of RB rows x JB
//       sub-columns x BB images of the parity view P = tensor columns P::2),
//   N = output channels (64/128/256 per tile),
//   K = (tap t, input channel).
//
// For a tile of parity P every tap t = (dc, dr) reads ONE constant-offset box
// of one input parity view P' = (P+dc) mod 2, at sub-column offset
// floor((P+dc)/2) and row offset dr (the tap row offset depends only on the
// centre parity, constant over the tile).  TMA loads that box (64 channels x
// 128 pixels, SWIZZLE_128B, zero fill for off-grid neighbours = DESIGN.md A4)
// straight into the K-major A operand layout; weights are pre-packed
// tap-major [T][Cout][Cin] and loaded as the K-major B operand.
//
// Forward kernel: persistent, warp specialised (warp 0 TMA producer, warp 1
// MMA issuer, warps 2-5 epilogue), 4-8 stage smem ring, two TMEM accumulators
// so the epilogue of tile i overlaps the MMAs of tile i+1.  The epilogue adds
// bias, applies ReLU or a ReLU-backward mask, rounds to bf16 (RNE) and stores
// NHWC rows.  Backward-data at stride 1 is the same kernel on dy with
// W'[ci][co][t] = W[co][ci][T-1-t] (pin P18).
//
// Weight-gradient kernel: per (Cout tile of 128, Cin tile N, tap group,
// pixel chunk) accumulate dW_t = dy^T * shift_t(x) over the chunk with both
// operands MN-major (pixels are K), then a fixed-order split-K reduction.
#include <cudaTypedefs.h>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hexconv {

constexpr int TC_BM = 128;  // output pixels per tile (UMMA M)
constexpr int TC_BK = 64;   // channels per K block = one 128-byte swizzle row
constexpr int TC_MAXT = 37; // taps supported on the tensor-core path (n <= 3)
constexpr int TC_EPI_THREADS = 256;              // 8 epilogue warps (2 per TMEM lane quadrant)
constexpr int TC_FWD_THREADS = 64 + TC_EPI_THREADS;

// ------------------------------------------------------------------ host: TMA descriptors
static PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = (PFN_cuTensorMapEncodeTiled_v12000)p;
    }
    return fn;
}

// NHWC bf16 tensor [B][H][W][C] viewed as parity view P (columns P, P+2, ...):
// dims {C, H, ceil((W-P)/2), B}, box {64, RB, JB, BB}.
static bool make_view_map(CUtensorMap* m, const void* base, int B, int H, int W, int C, int P, int RB, int JB,
                          int BB) {
    auto enc = get_encode();
    if (!enc) return false;
    const int Wp = (W - P + 1) / 2;
    if (Wp < 1) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)H, (cuuint64_t)Wp, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)W * C * 2, (cuuint64_t)2 * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {(cuuint32_t)TC_BK, (cuuint32_t)RB, (cuuint32_t)JB, (cuuint32_t)BB};
    cuuint32_t es[4] = {1, 1, 1, 1};
    void* addr = (void*)((const char*)base + (size_t)P * C * 2);
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, addr, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The same parity view with the channel axis split into 64-channel chunks as an
// OUTER dimension: dims {64, H, Wp, B, C/64}, box {64, RB, JB, BB, KC}.  One TMA op
// then fills KC consecutive canonical SW128 blocks (one per 64-channel chunk).
// estride = s > 1: rows and view sub-columns traversed with element stride s (strided forward / weight gradient,
// lattice_box)
static bool make_view_map5(CUtensorMap* m, const void* base, int B, int H, int W, int C, int P, int RB, int JB,
                           int BB, int KC, int estride = 1) {
    auto enc = get_encode();
    if (!enc) return false;
    const int Wp = (W - P + 1) / 2;
    if (Wp < 1 || C % 64) return false;
    cuuint64_t dims[5] = {64, (cuuint64_t)H, (cuuint64_t)Wp, (cuuint64_t)B, (cuuint64_t)(C / 64)};
    cuuint64_t strides[4] = {(cuuint64_t)W * C * 2, (cuuint64_t)2 * C * 2, (cuuint64_t)H * W * C * 2, 128};
    cuuint32_t box[5] = {64, (cuuint32_t)(RB * estride), (cuuint32_t)(JB * estride), (cuuint32_t)BB, (cuuint32_t)KC};
    cuuint32_t es[5] = {1, (cuuint32_t)estride, (cuuint32_t)estride, 1, 1};
    void* addr = (void*)((const char*)base + (size_t)P * C * 2);
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, addr, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// packed weights [T][N][K] as dims {64, N, K/64, T}, box {64, BN, KC, 1}: KC blocks of [BN][64]
static bool make_weight_map4(CUtensorMap* m, const void* base, int T, int N, int K, int BN, int KC) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {64, (cuuint64_t)N, (cuuint64_t)(K / 64), (cuuint64_t)T};
    cuuint64_t strides[3] = {(cuuint64_t)K * 2, 128, (cuuint64_t)N * K * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)BN, (cuuint32_t)KC, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// packed weights [T][N][K] bf16, box {64, BN, 1}
static bool make_weight_map(CUtensorMap* m, const void* base, int T, int N, int K, int BN) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {(cuuint64_t)K, (cuuint64_t)N, (cuuint64_t)T};
    cuuint64_t strides[2] = {(cuuint64_t)K * 2, (cuuint64_t)N * K * 2};
    cuuint32_t box[3] = {(cuuint32_t)TC_BK, (cuuint32_t)BN, 1};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, (void*)base, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// Pixel box (RB x JB x BB = npix) minimising the number of tiles over both views.
static void choose_box(int B, int H, int W, int npix, int* RB, int* JB, int* BB, int es = 1) {
    long best = -1;
    for (int rb = 1; rb <= npix; rb *= 2)
        for (int jb = 1; rb * jb <= npix; jb *= 2) {
            const int bb = npix / (rb * jb);
            if (rb * es > 256 || jb * es > 256 || bb > 256) continue;  // TMA box extents (element stride es)
            long tiles = 0;
            for (int P = 0; P < 2; ++P) {
                const int Wp = (W - P + 1) / 2;
                if (Wp < 1) continue;
                tiles += (long)ceil_div(H, rb) * ceil_div(Wp, jb) * ceil_div(B, bb);
            }
            // prefer fewer tiles, then taller row boxes (vertical halo reuse in L2)
            if (best < 0 || tiles < best || (tiles == best && rb > *RB)) {
                best = tiles;
                *RB = rb; *JB = jb; *BB = bb;
            }
        }
}

// ------------------------------------------------------------------ forward kernel
struct TcFwdParams {
    int B, H, W, Cin, Cout, T, parity;
    int s;  // 1, 2 or 3: output column-parity classes P = C mod 2 read element-stride-s input boxes (lattice_box)
    int RB, JB, BB;
    int rt, bt, jt0, jt1;  // tiles along rows, batch, and sub-columns of view 0 / view 1
    int tiles0;            // m tiles of view 0
    int n_tiles, total_tiles, kblocks;
    int m_total, pair_tiles;  // m tiles over both views; (n tile, m-tile pair) work items of the 2-CTA kernel
    int relu, has_mask;
    const float* bias;
    int8_t tap_dc[2][TC_MAXT];
    int8_t tap_dr[2][TC_MAXT];
};

struct TileCoord {
    int P, r0, j0, b0, n0;
};

__device__ __forceinline__ TileCoord decode_fwd_tile(const TcFwdParams& p, int tile, int BN) {
    TileCoord tc;
    const int nt = tile % p.n_tiles;
    int m = tile / p.n_tiles;
    tc.n0 = nt * BN;
    int jt;
    if (p.jt0 == p.jt1) {  // interleave the two parity views: both passes over a region run together (L2 reuse)
        tc.P = m & 1; m >>= 1; jt = p.jt0;
    } else if (m < p.tiles0) { tc.P = 0; jt = p.jt0; }
    else { tc.P = 1; m -= p.tiles0; jt = p.jt1; }
    const int rti = m % p.rt;
    m /= p.rt;
    const int jti = m % jt;
    const int bti = m / jt;
    tc.r0 = rti * p.RB;
    tc.j0 = jti * p.JB;
    tc.b0 = bti * p.BB;
    return tc;
}

// 2-CTA kernel: work item = (n tile, pair of consecutive m tiles); CTA `rank` of the
// pair takes m tile 2*mpair + rank.  A missing odd tile gets r0 = H: its loads are
// out of bounds (zero fill) and its TMA stores are clipped entirely.
__device__ __forceinline__ TileCoord decode_pair_tile(const TcFwdParams& p, int ptile, int BN, int rank) {
    const int nt = ptile % p.n_tiles;
    const int m = 2 * (ptile / p.n_tiles) + rank;
    TileCoord tc;
    if (m >= p.m_total) {
        tc.P = 0; tc.r0 = p.H; tc.j0 = 0; tc.b0 = 0; tc.n0 = nt * BN;
        return tc;
    }
    tc = decode_fwd_tile(p, m * p.n_tiles + nt, BN);
    return tc;
}

// Input box of tap (dc, dr) for an output tile of column class P at (r0, j0) of the stride-s lattice:
// output column C = 2C' + P has its centre at input column sC = 2sC' + sP and row s R + rho_P, where
// rho(C) = floor((sC + parity) / 2) mod s = floor((sP + parity) / 2) mod s depends only on P (A5).
// Tap (dc, dr) then reads input column 2sC' + sP + dc: view Pv = (sP + dc) mod 2, sub-column
// s C' + (sP + dc - Pv) / 2; with the maps traversing rows and view sub-columns with element stride s the
// box starts at sub-column s j0 + (sP + dc - Pv) / 2, row s r0 + rho_P + dr.  s = 1 is the stride-1 case
// (output view P = tensor columns P::2, rho = 0); the centre column's parity, which selects the tap table,
// is (sP + parity) mod 2.
__device__ __forceinline__ void lattice_box(int s, int parity, int P, int r0, int j0, int dc, int dr, int* Pv,
                                            int* row, int* col) {
    if (s == 1) {  // the stride-1 kernels' hot path: no integer division
        *Pv = (P + dc) & 1;
        *col = j0 + (P + dc - *Pv) / 2;
        *row = r0 + dr;
        return;
    }
    const int sp = s * P;
    *Pv = (sp + dc) & 1;
    *col = s * j0 + (sp + dc - *Pv) / 2;
    *row = s * r0 + ((sp + parity) >> 1) % s + dr;
}
__device__ __forceinline__ int lattice_centre_parity(int s, int parity, int P) { return (s * P + parity) & 1; }
__device__ __forceinline__ void tap_box(const TcFwdParams& p, int P, int r0, int j0, int dc, int dr, int* Pv,
                                        int* row, int* col) {
    lattice_box(p.s, p.parity, P, r0, j0, dc, dr, Pv, row, col);
}

// KC = 64-channel chunks per K iteration (one TMA op each for A and B).
template <int BN, int KC = 1>
struct FwdCfg {
    static constexpr int A_CHUNK = TC_BM * 128;
    static constexpr int B_CHUNK = BN * 128;
    static constexpr int A_BYTES = KC * A_CHUNK;
    static constexpr int STAGE = KC * (A_CHUNK + B_CHUNK);
    static constexpr int STAGES = (196608 / STAGE) > 8 ? 8 : (196608 / STAGE);
    static constexpr int OUT_BYTES = TC_BM * 128;  // one 64-channel output chunk, SW128 staging
    static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int SMEM = STAGES * STAGE + 2 * OUT_BYTES + 1024 + 256;
};

// Epilogue shared by the 1-CTA and 2-CTA forward kernels (warps 2..5).
template <int BN, bool PAIR>
__device__ __forceinline__ void fwd_epilogue(const TcFwdParams& p, const CUtensorMap* map_y0,
                                             const CUtensorMap* map_y1, const CUtensorMap* map_m0,
                                             const CUtensorMap* map_m1, uint8_t* obuf, uint64_t* tfull,
                                             uint64_t* tempty, uint64_t* mbar, uint32_t tmem_base, int first,
                                             int step, int rank) {
    using Cfg = FwdCfg<BN>;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    {
        // Epilogue: warps 2..9; warp w owns TMEM lane quadrant w % 4 (tile row m = TMEM lane)
        // and column half h of every 64-channel chunk.  Per chunk: TMEM -> registers ->
        // (bias, ReLU | ReLU-backward mask) -> bf16 -> SW128 staging row m (16-byte chunk i
        // at i ^ (m & 7)) -> one TMA store of the box.
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        const int row = q * 32 + lane;
        const int et = threadIdx.x - 64;  // 0..255
        int acc = 0;
        uint32_t aphase = 0;
        int ob = 0;
        uint32_t mphase0 = 0, mphase1 = 0;
        const int ntiles = PAIR ? p.pair_tiles : p.total_tiles;
        for (int tile = first; tile < ntiles; tile += step) {
            const TileCoord tc = PAIR ? decode_pair_tile(p, tile, BN, rank) : decode_fwd_tile(p, tile, BN);
            const CUtensorMap* my = tc.P ? map_y1 : map_y0;
            const CUtensorMap* mm = tc.P ? map_m1 : map_m0;
            // ReLU-backward mask of the first chunk: fetch before waiting for the accumulator
            if (p.has_mask && et == 0) {
                ptx::bulk_wait_read<1>();  // buffer ob: its last store (2 chunks ago) has been read
                ptx::mbar_arrive_expect_tx(&mbar[ob], Cfg::OUT_BYTES);
                ptx::tma_load_4d(mm, &mbar[ob], obuf + ob * Cfg::OUT_BYTES, tc.n0, tc.r0, tc.j0, tc.b0);
            }
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int ch = 0; ch < BN / 64; ++ch) {
                uint8_t* buf = obuf + ob * Cfg::OUT_BYTES;
                const int c0 = tc.n0 + ch * 64;
                if (p.has_mask) {
                    ptx::mbar_wait(&mbar[ob], ob ? mphase1 : mphase0);
                    if (ob) mphase1 ^= 1; else mphase0 ^= 1;
                } else {
                    if (et == 0) ptx::bulk_wait_read<1>();  // the store issued from this buffer 2 chunks ago
                    ptx::named_bar(1, TC_EPI_THREADS);
                }
                uint32_t v[32];
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + ch * 64 + h * 32;
                ptx::tmem_ld32(taddr, v);
                ptx::tmem_ld_wait();
                uint8_t* rowp = buf + row * 128;
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    const int i = 4 * h + ii;  // 16-byte unit (8 channels) within the 64-channel chunk
                    uint4* slot = reinterpret_cast<uint4*>(rowp + ((i ^ (row & 7)) << 4));
                    float f[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) f[k] = __uint_as_float(v[8 * ii + k]);
                    if (p.bias) {
                        const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + c0 + 8 * i));
                        const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + c0 + 8 * i + 4));
                        f[0] += b0.x; f[1] += b0.y; f[2] += b0.z; f[3] += b0.w;
                        f[4] += b1.x; f[5] += b1.y; f[6] += b1.z; f[7] += b1.w;
                    }
                    if (p.relu) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) f[k] = fmaxf(f[k], 0.f);
                    }
                    if (p.has_mask) {
                        const uint4 m4 = *slot;
                        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const uint32_t bits = (k & 1) ? (mw[k >> 1] & 0xffff0000u) : (mw[k >> 1] << 16);
                            if (!(__uint_as_float(bits) > 0.f)) f[k] = 0.f;
                        }
                    }
                    uint32_t pk[4];
#pragma unroll
                    for (int k = 0; k < 4; ++k) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
                        pk[k] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    *slot = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                ptx::fence_proxy_async();  // generic-proxy smem writes -> visible to the TMA store
                ptx::named_bar(1, TC_EPI_THREADS);
                if (et == 0) {
                    ptx::tma_store_4d(my, buf, c0, tc.r0, tc.j0, tc.b0);
                    ptx::bulk_commit();
                    if (p.has_mask && ch + 1 < BN / 64) {  // prefetch the next chunk's mask
                        ptx::bulk_wait_read<1>();
                        ptx::mbar_arrive_expect_tx(&mbar[ob ^ 1], Cfg::OUT_BYTES);
                        ptx::tma_load_4d(mm, &mbar[ob ^ 1], obuf + (ob ^ 1) * Cfg::OUT_BYTES, c0 + 64, tc.r0, tc.j0,
                                         tc.b0);
                    }
                }
                ob ^= 1;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[acc]), 0));
                else ptx::mbar_arrive(&tempty[acc]);
            }
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
        if (et == 0) ptx::bulk_wait<0>();
    }
}

template <int BN, int KC>
__global__ void __launch_bounds__(TC_FWD_THREADS, 1)
tc_conv_fwd_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                   const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_y0,
                   const __grid_constant__ CUtensorMap map_y1, const __grid_constant__ CUtensorMap map_m0,
                   const __grid_constant__ CUtensorMap map_m1, const __grid_constant__ TcFwdParams p) {
    using Cfg = FwdCfg<BN, KC>;
    constexpr int STAGES = Cfg::STAGES;
    constexpr int STAGE = Cfg::STAGE;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem_base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned, shared space
    uint8_t* smem = smem_base;  // stage ring
    uint8_t* obuf = smem + STAGES * STAGE;
    uint64_t* full = (uint64_t*)(obuf + 2 * Cfg::OUT_BYTES);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* mbar = tempty + 2;  // mask-tile loads into the two staging buffers
    uint32_t* tmem_slot = (uint32_t*)(mbar + 3);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], TC_EPI_THREADS / 32);
            ptx::mbar_init(&mbar[a], 1);
        }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x0);
        ptx::prefetch_tmap(&map_x1);
        ptx::prefetch_tmap(&map_w);
        ptx::prefetch_tmap(&map_y0);
        ptx::prefetch_tmap(&map_y1);
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, Cfg::TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int kgroups = p.kblocks / KC;
    const int k_iters = p.T * kgroups;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
                const TileCoord tc = decode_fwd_tile(p, tile, BN);
                const int pc = lattice_centre_parity(p.s, p.parity, tc.P);  // centre column parity
                for (int t = 0; t < p.T; ++t) {
                    const int dc = p.tap_dc[pc][t], dr = p.tap_dr[pc][t];
                    int Pv, row, col;
                    tap_box(p, tc.P, tc.r0, tc.j0, dc, dr, &Pv, &row, &col);
                    const CUtensorMap* mx = Pv ? &map_x1 : &map_x0;
                    for (int kg = 0; kg < kgroups; ++kg) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * STAGE;
                        ptx::mbar_arrive_expect_tx(&full[stage], STAGE);
                        ptx::tma_load_5d(mx, &full[stage], sa, 0, row, col, tc.b0, kg * KC);
                        ptx::tma_load_4d(&map_w, &full[stage], sa + Cfg::A_BYTES, 0, tc.n0, kg * KC, t);
                        if (++stage == STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(TC_BM, BN, 0, 0);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int tile = blockIdx.x; tile < p.total_tiles; tile += gridDim.x) {
                ptx::mbar_wait(&tempty[acc], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int it = 0; it < k_iters; ++it) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(smem + stage * STAGE);
                    // k iteration it = (tap t, K group kg) with it = t * kgroups + kg
                    const uint32_t b0 = a0 + Cfg::A_BYTES;
#pragma unroll
                    for (int c = 0; c < KC; ++c)
#pragma unroll
                        for (int k = 0; k < TC_BK / 16; ++k) {
                            const uint64_t ad = ptx::smem_desc_sw128(a0 + c * Cfg::A_CHUNK + k * 32, 16, 1024);
                            const uint64_t bd = ptx::smem_desc_sw128(b0 + c * Cfg::B_CHUNK + k * 32, 16, 1024);
                            ptx::mma_bf16(d, ad, bd, idesc, (it | c | k) != 0);
                        }
                    ptx::mma_commit(&empty[stage]);
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                ptx::mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
            }
        }
    } else {
        fwd_epilogue<BN, false>(p, &map_y0, &map_y1, &map_m0, &map_m1, obuf, tfull, tempty, mbar, tmem_base,
                                blockIdx.x, gridDim.x, 0);
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, Cfg::TMEM_COLS);
    }
}


// ------------------------------------------------------------------ 2-CTA (cta_group::2) forward kernel
// A CTA pair computes an M = 256 tile (each CTA its own 128-pixel box) x N = BN:
// each CTA loads its A box and HALF of the weight tile (BN/2 rows), the leader
// issues tcgen05.mma.cta_group::2 (M = 256) reading both CTAs' smem, and each
// CTA's TMEM receives its own 128 rows.  Per SM this halves the weight traffic
// and the B footprint per stage (so the ring is deeper) compared with the
// 1-CTA kernel.
template <int BN, int KC = 1>
struct Fwd2Cfg {
    static constexpr int A_CHUNK = TC_BM * 128;
    static constexpr int B_CHUNK = (BN / 2) * 128;
    static constexpr int A_BYTES = KC * A_CHUNK;
    static constexpr int STAGE = KC * (A_CHUNK + B_CHUNK);
    static constexpr int STAGES = (196608 / STAGE) > 8 ? 8 : (196608 / STAGE);
    static constexpr int TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
    static constexpr int SMEM = STAGES * STAGE + 2 * FwdCfg<BN>::OUT_BYTES + 1024 + 256;
};

template <int BN, int KC>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(TC_FWD_THREADS, 1)
tc_conv_fwd2_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                    const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_y0,
                    const __grid_constant__ CUtensorMap map_y1, const __grid_constant__ CUtensorMap map_m0,
                    const __grid_constant__ CUtensorMap map_m1, const __grid_constant__ TcFwdParams p) {
    using Cfg = Fwd2Cfg<BN, KC>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned, shared space
    uint8_t* obuf = smem + Cfg::STAGES * Cfg::STAGE;
    uint64_t* full = (uint64_t*)(obuf + 2 * FwdCfg<BN>::OUT_BYTES);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* mbar = tempty + 2;
    uint32_t* tmem_slot = (uint32_t*)(mbar + 2);

    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 2 * TC_EPI_THREADS / 32);  // epilogue warps x 2 CTAs (leader's copy)
            ptx::mbar_init(&mbar[a], 1);
        }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x0);
        ptx::prefetch_tmap(&map_x1);
        ptx::prefetch_tmap(&map_w);
        ptx::prefetch_tmap(&map_y0);
        ptx::prefetch_tmap(&map_y1);
    }
    if (warp == 1) ptx::tmem_alloc_2sm(tmem_slot, Cfg::TMEM_COLS);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const int kgroups = p.kblocks / KC;
    const int k_iters = p.T * kgroups;
    const int first = blockIdx.x / 2, step = gridDim.x / 2;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = first; tile < p.pair_tiles; tile += step) {
                const TileCoord tc = decode_pair_tile(p, tile, BN, rank);
                const int pc = lattice_centre_parity(p.s, p.parity, tc.P);  // centre column parity
                for (int t = 0; t < p.T; ++t) {
                    const int dc = p.tap_dc[pc][t], dr = p.tap_dr[pc][t];
                    int Pv, row, col;
                    tap_box(p, tc.P, tc.r0, tc.j0, dc, dr, &Pv, &row, &col);
                    const CUtensorMap* mx = Pv ? &map_x1 : &map_x0;
                    for (int kg = 0; kg < kgroups; ++kg) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = smem + stage * Cfg::STAGE;
                        if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * Cfg::STAGE);
                        ptx::tma_load_5d_2sm(mx, &full[stage], sa, 0, row, col, tc.b0, kg * KC);
                        ptx::tma_load_4d_2sm(&map_w, &full[stage], sa + Cfg::A_BYTES, 0, tc.n0 + (int)rank * (BN / 2),
                                             kg * KC, t);
                        if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            constexpr uint32_t idesc = ptx::idesc_bf16(2 * TC_BM, BN, 0, 0);
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            for (int tile = first; tile < p.pair_tiles; tile += step) {
                ptx::mbar_wait(&tempty[acc], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                for (int it = 0; it < k_iters; ++it) {
                    ptx::mbar_wait(&full[stage], phase);
                    ptx::tc_fence_after();
                    const uint32_t a0 = ptx::smem_u32(smem + stage * Cfg::STAGE);
                    const uint32_t b0 = a0 + Cfg::A_BYTES;
#pragma unroll
                    for (int c = 0; c < KC; ++c)
#pragma unroll
                        for (int k = 0; k < TC_BK / 16; ++k) {
                            const uint64_t ad = ptx::smem_desc_sw128(a0 + c * Cfg::A_CHUNK + k * 32, 16, 1024);
                            const uint64_t bd = ptx::smem_desc_sw128(b0 + c * Cfg::B_CHUNK + k * 32, 16, 1024);
                            ptx::mma_bf16_2sm(d, ad, bd, idesc, (it | c | k) != 0);
                        }
                    ptx::mma_commit_2sm(&empty[stage]);
                    if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
                }
                ptx::mma_commit_2sm(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
            }
        }
    } else {
        fwd_epilogue<BN, true>(p, &map_y0, &map_y1, &map_m0, &map_m1, obuf, tfull, tempty, mbar, tmem_base, first,
                               step, rank);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // the peer's smem / TMEM must outlive the leader's last MMA
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm(tmem_base, Cfg::TMEM_COLS);
    }
}

// ------------------------------------------------------------------ weight packing
__global__ void pack_weights_kernel(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wp, int Cout,
                                    int Cin, int T, int tr) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)T * Cout * Cin;
    if (idx >= total) return;
    if (!tr) {
        // wp[t][co][ci] = w[co][ci][t]
        const int ci = (int)(idx % Cin);
        const int64_t q = idx / Cin;
        const int co = (int)(q % Cout);
        const int t = (int)(q / Cout);
        wp[idx] = w[((int64_t)co * Cin + ci) * T + t];
    } else {
        // wp[t][ci][co] = w[co][ci][T-1-t]
        const int co = (int)(idx % Cout);
        const int64_t q = idx / Cout;
        const int ci = (int)(q % Cin);
        const int t = (int)(q / Cin);
        wp[idx] = w[((int64_t)co * Cin + ci) * T + (T - 1 - t)];
    }
}

// several layers / passes in one launch (hex_conv2d_pack_weights).  One block per ROW: (segment, co) for the
// forward layout, (segment, ci) for the transposed one.  The block stages its contiguous (fwd) or
// T-element-run (bwd) slice of w in shared memory, then writes whole contiguous output runs (coalesced
// both ways); index division by float reciprocal with an exact correction (operands < 2^24).
__device__ __forceinline__ int pk_div(int n, int d, float inv) {
    int q = (int)((float)n * inv);
    const int r = n - q * d;
    if (r < 0) --q;
    else if (r >= d) ++q;
    return q;
}

constexpr int PK_THREADS = 256;

__global__ void __launch_bounds__(PK_THREADS) pack_weights_multi_kernel(const PackSegs segs) {
    extern __shared__ __align__(16) __nv_bfloat16 srow[];  // one row: Cin * T (fwd) or Cout * T (bwd) elements
    int k = 0;
    while (k + 1 < segs.count && (int64_t)blockIdx.x >= segs.seg[k + 1].row0) ++k;
    const PackSeg& sg = segs.seg[k];
    const int row = (int)(blockIdx.x - sg.row0);
    const __nv_bfloat16* w = (const __nv_bfloat16*)sg.w;
    __nv_bfloat16* wp = (__nv_bfloat16*)sg.wpack;
    const int T = sg.T, Cin = sg.Cin, Cout = sg.Cout;
    const float invT = 1.f / (float)T;
    if (!sg.tr) {  // wp[t][co][ci] = w[co][ci][t], row = co
        const int n = Cin * T;
        const __nv_bfloat16* src = w + (int64_t)row * n;
        if ((n & 7) == 0 && ((uintptr_t)src & 15) == 0) {  // 16-byte copies
#pragma unroll 4
            for (int i = threadIdx.x; i < n / 8; i += PK_THREADS)
                reinterpret_cast<uint4*>(srow)[i] = __ldg(reinterpret_cast<const uint4*>(src) + i);
        } else {
#pragma unroll 8
            for (int i = threadIdx.x; i < n; i += PK_THREADS) srow[i] = src[i];
        }
        __syncthreads();
        const float invC = 1.f / (float)Cin;
        for (int i = threadIdx.x; i < n; i += PK_THREADS) {
            const int t = pk_div(i, Cin, invC), ci = i - t * Cin;
            wp[((int64_t)t * Cout + row) * Cin + ci] = srow[ci * T + t];
        }
    } else {  // wp[t][ci][co] = w[co][ci][T-1-t], row = ci
        const int n = Cout * T;
#pragma unroll 8
        for (int i = threadIdx.x; i < n; i += PK_THREADS) {  // runs of T elements, 8 loads in flight
            const int co = pk_div(i, T, invT), t = i - co * T;
            srow[i] = w[((int64_t)co * Cin + row) * T + t];
        }
        __syncthreads();
        const float invC = 1.f / (float)Cout;
        for (int i = threadIdx.x; i < n; i += PK_THREADS) {
            const int t = pk_div(i, Cout, invC), co = i - t * Cout;
            wp[((int64_t)t * Cin + row) * Cout + co] = srow[co * T + (T - 1 - t)];
        }
    }
}

hex_status_t tc_pack_weights_multi(const PackSegs& segs, cudaStream_t st) {
    if (segs.count <= 0) return HEX_OK;
    const PackSeg& last = segs.seg[segs.count - 1];
    const int64_t rows = last.row0 + (last.tr ? last.Cin : last.Cout);
    int64_t smax = 0;
    for (int i = 0; i < segs.count; ++i) {
        const int64_t e = (int64_t)segs.seg[i].T * (segs.seg[i].tr ? segs.seg[i].Cout : segs.seg[i].Cin);
        if (e > smax) smax = e;
    }
    const size_t smem = (size_t)smax * sizeof(__nv_bfloat16);
    if (smem > 200 * 1024) return HEX_ERR_UNSUPPORTED;
    if (smem > 48 * 1024 &&
        cudaFuncSetAttribute(pack_weights_multi_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) !=
            cudaSuccess)
        return HEX_ERR_CUDA;
    pack_weights_multi_kernel<<<(unsigned)rows, PK_THREADS, smem, st>>>(segs);
    count_launch();
    return last_launch_status();
}

hex_status_t tc_pack_weights(const void* w, void* wpack, int Cout, int Cin, int T, int tr, cudaStream_t st) {
    const int64_t total = (int64_t)T * Cout * Cin;
    pack_weights_kernel<<<ceil_div(total, 256), 256, 0, st>>>((const __nv_bfloat16*)w, (__nv_bfloat16*)wpack, Cout,
                                                              Cin, T, tr);
    count_launch();
    return last_launch_status();
}

// ------------------------------------------------------------------ forward host
static int pick_bn(int Cout) {
    if (Cout % 256 == 0) return 256;
    if (Cout % 128 == 0) return 128;
    if (Cout % 64 == 0) return 64;
    return 0;
}

// strides 2 and 3 run the same kernels with element-stride-s input boxes (lattice_box); the strided
// backward passes have their own kernels (lat_dgrad.cu, the lattice weight gradient below)
bool tc_conv_fwd_supported(const Geom& g, int Cin, int Cout) {
    if (g.s == 1) return tc_conv_supported(g, Cin, Cout);
    if ((g.s != 2 && g.s != 3) || g.T > TC_MAXT || sw_on("HEXCONV_NO_TC_STRIDED_FWD")) return false;
    if (Cin % TC_BK != 0 || pick_bn(Cout) == 0 || g.Wo < 2) return false;
    if (sw_on("HEXCONV_DISABLE_TC")) return false;
    return get_encode() != nullptr;
}

bool tc_conv_supported(const Geom& g, int Cin, int Cout) {
    if (g.s != 1 || g.T > TC_MAXT) return false;
    if (Cin % TC_BK != 0 || pick_bn(Cout) == 0) return false;
    if (g.W < 2) return false;
    if (sw_on("HEXCONV_DISABLE_TC")) return false;
    return get_encode() != nullptr;
}

template <int BN, int KC>
static hex_status_t launch_fwd_bn(const CUtensorMap& mx0, const CUtensorMap& mx1, const CUtensorMap& mw,
                                  const CUtensorMap& my0, const CUtensorMap& my1, const CUtensorMap& mm0,
                                  const CUtensorMap& mm1, const TcFwdParams& p, cudaStream_t st) {
    using Cfg = FwdCfg<BN, KC>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(tc_conv_fwd_kernel<BN, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::SMEM) != cudaSuccess)
            return HEX_ERR_CUDA;
        attr_set = true;
    }
    const int grid = p.total_tiles < num_sms() ? p.total_tiles : num_sms();
    tc_conv_fwd_kernel<BN, KC><<<grid, TC_FWD_THREADS, Cfg::SMEM, st>>>(mx0, mx1, mw, my0, my1, mm0, mm1, p);
    count_launch();
    return last_launch_status();
}

template <int BN, int KC>
static hex_status_t launch_fwd2_bn(const CUtensorMap& mx0, const CUtensorMap& mx1, const CUtensorMap& mw,
                                   const CUtensorMap& my0, const CUtensorMap& my1, const CUtensorMap& mm0,
                                   const CUtensorMap& mm1, const TcFwdParams& p, cudaStream_t st) {
    using Cfg = Fwd2Cfg<BN, KC>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(tc_conv_fwd2_kernel<BN, KC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 Cfg::SMEM) != cudaSuccess)
            return HEX_ERR_CUDA;
        attr_set = true;
    }
    const int pairs = p.pair_tiles < num_sms() / 2 ? p.pair_tiles : num_sms() / 2;
    tc_conv_fwd2_kernel<BN, KC><<<2 * pairs, TC_FWD_THREADS, Cfg::SMEM, st>>>(mx0, mx1, mw, my0, my1, mm0, mm1, p);
    count_launch();
    return last_launch_status();
}

// Kernel choice (round-1 measurements).  Each TMA op costs
// ~150 ns of issue time per SM almost independently of its size, so a K
// iteration should carry >= ~512 MMA cycles per (A op, B op) pair: K iterations
// span KC = 2 channel chunks whenever Cin allows, and BN = 256 tiles run as
// CTA pairs (cta_group::2, M = 256) so each SM loads only half the weight tile.
// HEXCONV_FORCE_2SM / HEXCONV_NO_2SM / HEXCONV_KC override for experiments.
static bool use_2sm(int BN) {
    if (sw_on("HEXCONV_NO_2SM")) return false;
    if (sw_on("HEXCONV_FORCE_2SM")) return BN >= 128;
    return BN == 256;
}

hex_status_t tc_conv_fwd(const TcConvArgs& a, cudaStream_t st) {
    if (tc_fwd_tr_supported(a.g, a.Cin, a.Cout)) return tc_fwd_tr(a, st);  // tap-reuse kernel (tc_fwd_tr.cu)
    const Geom& g = a.g;
    TcFwdParams p{};
    p.B = g.B; p.H = g.H; p.W = g.W; p.Cin = a.Cin; p.Cout = a.Cout; p.T = g.T; p.parity = g.parity;
    p.s = g.s;
    const int OH = g.s == 1 ? g.H : g.Ho, OW = g.s == 1 ? g.W : g.Wo;  // output grid (tiles, stores)
    choose_box(g.B, OH, OW, TC_BM, &p.RB, &p.JB, &p.BB, g.s);
    p.rt = ceil_div(OH, p.RB);
    p.bt = ceil_div(g.B, p.BB);
    p.jt0 = ceil_div((OW + 1) / 2, p.JB);
    p.jt1 = ceil_div(OW / 2, p.JB);
    p.tiles0 = p.rt * p.jt0 * p.bt;
    const int BN = pick_bn(a.Cout);
    p.n_tiles = a.Cout / BN;
    p.m_total = p.tiles0 + p.rt * p.jt1 * p.bt;
    const bool pair = use_2sm(BN) && p.m_total >= 2;
    int KC = (a.Cin % 128 == 0 && !(BN == 256 && !pair)) ? 2 : 1;
    if (BN == 256 && !pair) KC = 1;  // a 1-CTA BN = 256 stage with KC = 2 would not fit twice in smem
    p.total_tiles = p.m_total * p.n_tiles;
    p.pair_tiles = ceil_div(p.m_total, 2) * p.n_tiles;
    p.kblocks = a.Cin / TC_BK;
    p.relu = a.relu;
    p.has_mask = a.relu_y != nullptr;
    p.bias = a.bias;
    for (int pc = 0; pc < 2; ++pc)
        for (int t = 0; t < g.T; ++t) {
            int dc, dr;
            tap_offset(g.n, pc, t, &dc, &dr);
            p.tap_dc[pc][t] = (int8_t)dc;
            p.tap_dr[pc][t] = (int8_t)dr;
        }
    CUtensorMap mx0, mx1, mw;
    if (!make_view_map5(&mx0, a.x, g.B, g.H, g.W, a.Cin, 0, p.RB, p.JB, p.BB, KC, g.s)) return HEX_ERR_CUDA;
    if (!make_view_map5(&mx1, a.x, g.B, g.H, g.W, a.Cin, 1, p.RB, p.JB, p.BB, KC, g.s)) return HEX_ERR_CUDA;
    if (!make_weight_map4(&mw, a.wpack, g.T, a.Cout, a.Cin, pair ? BN / 2 : BN, KC)) return HEX_ERR_CUDA;
    CUtensorMap my0, my1, mm0, mm1;
    if (!make_view_map(&my0, a.y, g.B, OH, OW, a.Cout, 0, p.RB, p.JB, p.BB)) return HEX_ERR_CUDA;
    if (!make_view_map(&my1, a.y, g.B, OH, OW, a.Cout, 1, p.RB, p.JB, p.BB)) return HEX_ERR_CUDA;
    if (a.relu_y) {
        if (!make_view_map(&mm0, a.relu_y, g.B, OH, OW, a.Cout, 0, p.RB, p.JB, p.BB)) return HEX_ERR_CUDA;
        if (!make_view_map(&mm1, a.relu_y, g.B, OH, OW, a.Cout, 1, p.RB, p.JB, p.BB)) return HEX_ERR_CUDA;
    } else {
        mm0 = my0;
        mm1 = my1;
    }
#define HEX_FWD_ARGS mx0, mx1, mw, my0, my1, mm0, mm1, p, st
    if (pair) {
        if (BN == 256) return KC == 2 ? launch_fwd2_bn<256, 2>(HEX_FWD_ARGS) : launch_fwd2_bn<256, 1>(HEX_FWD_ARGS);
        return KC == 2 ? launch_fwd2_bn<128, 2>(HEX_FWD_ARGS) : launch_fwd2_bn<128, 1>(HEX_FWD_ARGS);
    }
    switch (BN) {
        case 256: return launch_fwd_bn<256, 1>(HEX_FWD_ARGS);
        case 128: return KC == 2 ? launch_fwd_bn<128, 2>(HEX_FWD_ARGS) : launch_fwd_bn<128, 1>(HEX_FWD_ARGS);
        default: return KC == 2 ? launch_fwd_bn<64, 2>(HEX_FWD_ARGS) : launch_fwd_bn<64, 1>(HEX_FWD_ARGS);
    }
#undef HEX_FWD_ARGS
}

// ------------------------------------------------------------------ weight-gradient kernel
// dW[t][co][ci] = sum_pixels dy[px][co] * x[px + off_t][ci]  (pixels are K).
// The (tap, 64-input-channel chunk) pairs are "atoms"; one unit of work is
// (Cout tile of 128, a group of up to 8 atoms = 512 TMEM columns, a chunk of
// pixel tiles).  Per pixel tile (64 pixels of one parity view, RB x JB x BB):
//   A   = dy box  [64 px rows][64 co] x 2          (MN-major: co contiguous)
//   B_a = x box of atom a, shifted by tap t        (MN-major: ci contiguous)
// Up to four atom boxes sit one LBO (8 KB) apart and form one N = 256 MMA, so
// a full group is two 128x256x16 MMAs per 16 pixels; atom a accumulates in
// TMEM columns [64a, 64a+64).  Partial sums per pixel chunk go to a workspace
// and are reduced in a fixed order (deterministic).
// Pixels per pipeline stage: 32 (5 stages) for Cin = 64, 64 (2 stages) otherwise.
template <int PIX>
struct WgCfg {
    static constexpr int STAGES = PIX == 32 ? 5 : 2;
    static constexpr int BOX = PIX * 128;          // one 64-channel box
    static constexpr int STAGE_BYTES = (2 + 8) * BOX;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 128;
};
constexpr int WG_ATOMS = 8;                        // atoms per unit (512 TMEM columns)

struct TcWgParams {
    int B, H, W, Cin, Cout, T, parity;
    int RB, JB, BB;
    int rt, bt, jt0, jt1, tiles0, ptiles;  // pixel tiles
    int kchunks, cpo, n_atoms, groups, co_tiles, chunks, tiles_per_chunk;  // cpo: chunks per x op
    float* part;     // [chunks][T][Cout][Cin]
    float* db_part;  // [chunks][Cout] or NULL (no bias gradient)
    int dbg;         // development: 1 = skip TMA loads, 2 = skip MMAs (results invalid)
    int8_t tap_dc[2][TC_MAXT];
    int8_t tap_dr[2][TC_MAXT];
    int s;  // 1, 2 or 3: the pixel tiles walk the stride-s lattice (dy), the x maps traverse with element stride s
};

// x box of tap (dc, dr) for the pixel tile (P, r0, j0), and the centre-column parity that selects the tap table:
// the forward's lattice_box.  s = 1: tile of parity view P (tap reuse as the forward); s = 2, 3: tile of lattice
// view P of dy (output columns C = 2C' + P), x maps traversed with element stride s.
__device__ __forceinline__ int wg_centre_parity(const TcWgParams& p, int P) {
    return lattice_centre_parity(p.s, p.parity, P);
}
__device__ __forceinline__ void wg_xbox(const TcWgParams& p, int P, int r0, int j0, int dc, int dr, int* Pv,
                                        int* row, int* col) {
    lattice_box(p.s, p.parity, P, r0, j0, dc, dr, Pv, row, col);
}

__device__ __forceinline__ void decode_ptile(const TcWgParams& p, int m, int* P, int* r0, int* j0, int* b0) {
    int jt;
    if (p.jt0 == p.jt1) { *P = m & 1; m >>= 1; jt = p.jt0; }  // views interleaved (see decode_fwd_tile)
    else if (m < p.tiles0) { *P = 0; jt = p.jt0; }
    else { *P = 1; m -= p.tiles0; jt = p.jt1; }
    const int rti = m % p.rt;
    m /= p.rt;
    const int jti = m % jt;
    const int bti = m / jt;
    *r0 = rti * p.RB;
    *j0 = jti * p.JB;
    *b0 = bti * p.BB;
}

template <int PIX>
__global__ void __launch_bounds__(192, 1)
tc_conv_wgrad_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                     const __grid_constant__ CUtensorMap map_dy0, const __grid_constant__ CUtensorMap map_dy1,
                     const __grid_constant__ TcWgParams p) {
    using Cfg = WgCfg<PIX>;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned, shared space
    uint64_t* full = (uint64_t*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* tfull = empty + Cfg::STAGES;
    uint32_t* tmem_slot = (uint32_t*)(tfull + 1);

    // unit decode
    int u = blockIdx.x;
    const int chunk = u % p.chunks; u /= p.chunks;
    const int grp = u % p.groups;
    const int cot = u / p.groups;
    const int a0 = grp * WG_ATOMS;
    const int na = min(WG_ATOMS, p.n_atoms - a0);
    const int co0 = cot * 128;
    const int pt_begin = chunk * p.tiles_per_chunk;
    const int pt_end = min(p.ptiles, pt_begin + p.tiles_per_chunk);

    // units of atom group 0 also reduce dbias from the dy tiles in shared memory
    const bool do_db = p.db_part != nullptr && grp == 0;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], do_db ? 5 : 1);  // MMA commit (+ 4 epilogue warps reading dy)
        }
        ptx::mbar_init(tfull, 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x0);
        ptx::prefetch_tmap(&map_x1);
        ptx::prefetch_tmap(&map_dy0);
        ptx::prefetch_tmap(&map_dy1);
    }
    if (warp == 1) ptx::tmem_alloc(tmem_slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t stage_bytes = (2 + na) * Cfg::BOX;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = pt_begin; pt < pt_end; ++pt) {
                int P, r0, j0, b0;
                decode_ptile(p, pt, &P, &r0, &j0, &b0);
                const int pc = wg_centre_parity(p, P);
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* s = smem + stage * Cfg::STAGE_BYTES;
                if (HEX_DBG(p.dbg) == 1) {
                    ptx::mbar_arrive(&full[stage]);
                    if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
                    continue;
                }
                ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
                // one op for the two dy channel chunks, one op per tap for all its input-channel chunks
                ptx::tma_load_5d(P ? &map_dy1 : &map_dy0, &full[stage], s, 0, r0, j0, b0, co0 / 64);
                for (int i = 0; i < na; i += p.cpo) {
                    const int t = (a0 + i) / p.kchunks, kc = (a0 + i) - t * p.kchunks;
                    int Pv, row, col;
                    wg_xbox(p, P, r0, j0, p.tap_dc[pc][t], p.tap_dr[pc][t], &Pv, &row, &col);
                    ptx::tma_load_5d(Pv ? &map_x1 : &map_x0, &full[stage], s + (2 + i) * Cfg::BOX, 0, row, col, b0,
                                     kc);
                }
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const int n0 = min(na, 4), n1 = na - n0;
            const uint32_t idesc0 = ptx::idesc_bf16(128, 64 * n0, 1, 1);
            const uint32_t idesc1 = ptx::idesc_bf16(128, 64 * (n1 > 0 ? n1 : 1), 1, 1);
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = pt_begin; pt < pt_end; ++pt) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                const uint32_t s = ptx::smem_u32(smem + stage * Cfg::STAGE_BYTES);
                const uint32_t bx = s + 2 * Cfg::BOX;
#pragma unroll
                for (int k = 0; k < PIX / 16; ++k) {
                    // MN-major SW128: 8-row K groups 1024 B apart, 64-element MN blocks one box (LBO) apart
                    const uint64_t ad = ptx::smem_desc_sw128(s + k * 2048, Cfg::BOX, 1024);
                    const uint32_t acc = (pt != pt_begin) || (k != 0);
                    if (HEX_DBG(p.dbg) == 2) continue;
                    ptx::mma_bf16(tmem_base, ad, ptx::smem_desc_sw128(bx + k * 2048, Cfg::BOX, 1024), idesc0, acc);
                    if (n1 > 0)
                        ptx::mma_bf16(tmem_base + 256, ad,
                                      ptx::smem_desc_sw128(bx + 4 * Cfg::BOX + k * 2048, Cfg::BOX, 1024),
                                      idesc1, acc);
                }
                ptx::mma_commit(&empty[stage]);
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
            ptx::mma_commit(tfull);
        }
    } else {
        const int q = warp & 3;
        const int row = q * 32 + lane;  // co local
        if (do_db) {
            // dbias[co] partial: column sums of the dy tiles (SW128 layout: 16-byte chunk j of
            // pixel row px sits at chunk j ^ (px & 7))
            const int box = row >> 6, e = row & 63, j = e >> 3, sub = e & 7;
            float dsum = 0.f;
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = pt_begin; pt < pt_end; ++pt) {
                ptx::mbar_wait(&full[stage], phase);
                const uint8_t* sdy = smem + stage * Cfg::STAGE_BYTES + box * Cfg::BOX;
#pragma unroll 8
                for (int px = 0; px < PIX; ++px) {
                    const __nv_bfloat16 v =
                        *reinterpret_cast<const __nv_bfloat16*>(sdy + px * 128 + ((j ^ (px & 7)) << 4) + sub * 2);
                    dsum += __bfloat162float(v);
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[stage]);
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
            p.db_part[(int64_t)chunk * p.Cout + co0 + row] = dsum;
        }
        ptx::mbar_wait(tfull, 0);
        ptx::tc_fence_after();
        const int co = co0 + row;
        const bool empty_chunk = pt_end <= pt_begin;
        for (int i = 0; i < na; ++i) {
            const int a = a0 + i;
            const int t = a / p.kchunks, kc = a - t * p.kchunks;
            float* dst = p.part + (((int64_t)chunk * p.T + t) * p.Cout + co) * p.Cin + kc * 64;
#pragma unroll 1
            for (int ch = 0; ch < 2; ++ch) {
                uint32_t v[32];
                ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + i * 64 + ch * 32, v);
                ptx::tmem_ld_wait();
                float4* d4 = reinterpret_cast<float4*>(dst + ch * 32);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    float4 f;
                    f.x = empty_chunk ? 0.f : __uint_as_float(v[4 * j]);
                    f.y = empty_chunk ? 0.f : __uint_as_float(v[4 * j + 1]);
                    f.z = empty_chunk ? 0.f : __uint_as_float(v[4 * j + 2]);
                    f.w = empty_chunk ? 0.f : __uint_as_float(v[4 * j + 3]);
                    d4[j] = f;
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 512);
    }
}


// ------------------------------------------------------------------ 2-CTA weight-gradient kernel
// For Cout % 256 == 0 and Cin % 128 == 0.  A CTA pair owns 256 output channels
// (M = 256, each CTA 128) and a group of up to 8 atoms; per 16 pixels the leader
// issues up to two tcgen05.mma.cta_group::2 (M = 256, N = 64 q, q <= 4 atoms),
// each CTA supplying q/2 atoms of B.  Per CTA and 64-pixel stage: one dy op
// (its 128 channels) + one x op per MMA (2 chunks of one tap) = 48 KB, four
// stages deep.  Atom 4m + j accumulates in TMEM columns 256 m + 64 j.
struct Wg2Cfg {
    static constexpr int PIX = 64;
    static constexpr int BOX = PIX * 128;          // 8 KB per 64-channel box
    static constexpr int STAGE_BYTES = 6 * BOX;    // dy (2 boxes) + x (2 ops x 2 boxes)
    static constexpr int STAGES = 4;
    static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 128;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(192, 1)
tc_conv_wgrad2_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                      const __grid_constant__ CUtensorMap map_dy0, const __grid_constant__ CUtensorMap map_dy1,
                      const __grid_constant__ TcWgParams p) {
    using Cfg = Wg2Cfg;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned, shared space
    uint64_t* full = (uint64_t*)(smem + Cfg::STAGES * Cfg::STAGE_BYTES);
    uint64_t* empty = full + Cfg::STAGES;
    uint64_t* dbr = empty + Cfg::STAGES;  // per stage: MMAs done (multicast) -> dy tile readable for dbias
    uint64_t* tfull = dbr + Cfg::STAGES;
    uint32_t* tmem_slot = (uint32_t*)(tfull + 1);

    const uint32_t rank = ptx::cluster_ctarank();
    const bool leader = rank == 0;
    int u = blockIdx.x / 2;
    const int chunk = u % p.chunks; u /= p.chunks;
    const int grp = u % p.groups;
    const int cop = u / p.groups;
    const int a0 = grp * WG_ATOMS;
    const int na = min(WG_ATOMS, p.n_atoms - a0);  // even
    const int q0 = min(na, 4), q1 = na - q0;       // atoms of MMA 0 / MMA 1
    const int co0 = cop * 256 + 128 * (int)rank;    // this CTA's channels
    const int pt_begin = chunk * p.tiles_per_chunk;
    const int pt_end = min(p.ptiles, pt_begin + p.tiles_per_chunk);
    const bool do_db = p.db_part != nullptr && grp == 0;

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < Cfg::STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], do_db ? 5 : 1);
            ptx::mbar_init(&dbr[s], 1);
        }
        ptx::mbar_init(tfull, 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x0);
        ptx::prefetch_tmap(&map_x1);
        ptx::prefetch_tmap(&map_dy0);
        ptx::prefetch_tmap(&map_dy1);
    }
    if (warp == 1) ptx::tmem_alloc_2sm(tmem_slot, 512);
    ptx::tc_fence_before();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;
    const uint32_t stage_bytes = (2 + (q1 > 0 ? 4 : 2)) * Cfg::BOX;  // per CTA

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = pt_begin; pt < pt_end; ++pt) {
                int P, r0, j0, b0;
                decode_ptile(p, pt, &P, &r0, &j0, &b0);
                const int pc = wg_centre_parity(p, P);
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* s = smem + stage * Cfg::STAGE_BYTES;
                if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * stage_bytes);
                ptx::tma_load_5d_2sm(P ? &map_dy1 : &map_dy0, &full[stage], s, 0, r0, j0, b0, co0 / 64);
                for (int m = 0; m < 2; ++m) {
                    const int q = m ? q1 : q0;
                    if (q == 0) break;
                    const int a = a0 + 4 * m + (int)rank * (q / 2);
                    const int t = a / p.kchunks, kc = a - t * p.kchunks;
                    int Pv, row, col;
                    wg_xbox(p, P, r0, j0, p.tap_dc[pc][t], p.tap_dr[pc][t], &Pv, &row, &col);
                    ptx::tma_load_5d_2sm(Pv ? &map_x1 : &map_x0, &full[stage], s + (2 + 2 * m) * Cfg::BOX, 0, row,
                                         col, b0, kc);
                }
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (leader && lane == 0) {
            const uint32_t idesc0 = ptx::idesc_bf16(256, 64 * q0, 1, 1);
            const uint32_t idesc1 = ptx::idesc_bf16(256, 64 * (q1 > 0 ? q1 : 2), 1, 1);
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = pt_begin; pt < pt_end; ++pt) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                const uint32_t s = ptx::smem_u32(smem + stage * Cfg::STAGE_BYTES);
#pragma unroll
                for (int k = 0; k < Cfg::PIX / 16; ++k) {
                    const uint64_t ad = ptx::smem_desc_sw128(s + k * 2048, Cfg::BOX, 1024);
                    const uint32_t acc = (pt != pt_begin) || (k != 0);
                    ptx::mma_bf16_2sm(tmem_base, ad,
                                      ptx::smem_desc_sw128(s + 2 * Cfg::BOX + k * 2048, Cfg::BOX, 1024), idesc0, acc);
                    if (q1 > 0)
                        ptx::mma_bf16_2sm(tmem_base + 256, ad,
                                          ptx::smem_desc_sw128(s + 4 * Cfg::BOX + k * 2048, Cfg::BOX, 1024), idesc1,
                                          acc);
                }
                ptx::mma_commit_2sm(&empty[stage]);
                if (do_db) ptx::mma_commit_2sm(&dbr[stage]);
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
            ptx::mma_commit_2sm(tfull);
        }
    } else {
        const int q = warp & 3;
        const int row = q * 32 + lane;  // channel within this CTA's 128
        if (do_db) {
            const int box = row >> 6, e = row & 63, j = e >> 3, sub = e & 7;
            float dsum = 0.f;
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = pt_begin; pt < pt_end; ++pt) {
                ptx::mbar_wait(&dbr[stage], phase);  // both CTAs' tiles were consumed by the MMAs
                const uint8_t* sdy = smem + stage * Cfg::STAGE_BYTES + box * Cfg::BOX;
#pragma unroll 8
                for (int px = 0; px < Cfg::PIX; ++px) {
                    const __nv_bfloat16 v =
                        *reinterpret_cast<const __nv_bfloat16*>(sdy + px * 128 + ((j ^ (px & 7)) << 4) + sub * 2);
                    dsum += __bfloat162float(v);
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&empty[stage]);
                if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1; }
            }
            p.db_part[(int64_t)chunk * p.Cout + co0 + row] = dsum;
        }
        ptx::mbar_wait(tfull, 0);
        ptx::tc_fence_after();
        const int co = co0 + row;
        const bool empty_chunk = pt_end <= pt_begin;
        for (int m = 0; m < 2; ++m) {
            const int qm = m ? q1 : q0;
            for (int jj = 0; jj < qm; ++jj) {
                const int a = a0 + 4 * m + jj;
                const int t = a / p.kchunks, kc = a - t * p.kchunks;
                float* dst = p.part + (((int64_t)chunk * p.T + t) * p.Cout + co) * p.Cin + kc * 64;
#pragma unroll 1
                for (int ch = 0; ch < 2; ++ch) {
                    uint32_t v[32];
                    ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + 256 * m + 64 * jj + ch * 32, v);
                    ptx::tmem_ld_wait();
                    float4* d4 = reinterpret_cast<float4*>(dst + ch * 32);
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        float4 f;
                        f.x = empty_chunk ? 0.f : __uint_as_float(v[4 * i]);
                        f.y = empty_chunk ? 0.f : __uint_as_float(v[4 * i + 1]);
                        f.z = empty_chunk ? 0.f : __uint_as_float(v[4 * i + 2]);
                        f.w = empty_chunk ? 0.f : __uint_as_float(v[4 * i + 3]);
                        d4[i] = f;
                    }
                }
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc_2sm(tmem_base, 512);
    }
}

// dw[co][ci][t] (+)= sum_chunk part[chunk][t][co][ci]   (fixed chunk order)
__global__ void wgrad_tc_reduce_kernel(const float* __restrict__ part, int chunks, int T, int Cout, int Cin,
                                       float* __restrict__ dw, const float* __restrict__ db_part,
                                       float* __restrict__ dbias, int accumulate) {
    // threads [0, T*Cout*Cin) reduce dw, the next Cout threads dbias (one launch for both)
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)T * Cout * Cin;
    const bool is_db = idx >= total;
    if (is_db && (dbias == nullptr || idx >= total + Cout)) return;
    const float* src = is_db ? db_part : part;
    const int64_t stride = is_db ? Cout : total;
    const int64_t off = is_db ? idx - total : idx;
    // eight independent partial sums (chunk c -> sum c mod 8) keep eight loads in flight per thread;
    // combined in a fixed tree order: deterministic
    float s8[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    int c = 0;
    for (; c + 8 <= chunks; c += 8)
#pragma unroll
        for (int j = 0; j < 8; ++j) s8[j] += src[(int64_t)(c + j) * stride + off];
#pragma unroll
    for (int j = 0; j < 8; ++j)
        if (c + j < chunks) s8[j] += src[(int64_t)(c + j) * stride + off];
    const float s = ((s8[0] + s8[1]) + (s8[2] + s8[3])) + ((s8[4] + s8[5]) + (s8[6] + s8[7]));
    if (is_db) {
        dbias[off] = accumulate ? dbias[off] + s : s;
        return;
    }
    // idx enumerates (t, co, ci) with ci fastest (coalesced partial reads)
    const int ci = (int)(idx % Cin);
    const int64_t q = idx / Cin;
    const int co = (int)(q % Cout);
    const int t = (int)(q / Cout);
    float* d = dw + ((int64_t)co * Cin + ci) * T + t;
    *d = accumulate ? *d + s : s;
}

// (A variant transposing through shared memory -- block (co, 32 channels) writing dw[co][ci0..ci0+31][t]
// contiguously -- measured slower in the C5 step: 21.5 vs 15.4 us per launch.)
static hex_status_t wgrad_reduce(const float* part, int chunks, int T, int Cout, int Cin, float* dw,
                                 const float* db_part, float* dbias, int accumulate, cudaStream_t st) {
    const int64_t total = (int64_t)T * Cout * Cin;
    wgrad_tc_reduce_kernel<<<ceil_div(total + Cout, 256), 256, 0, st>>>(part, chunks, T, Cout, Cin, dw, db_part, dbias,
                                                                      accumulate);
    count_launch();
    return last_launch_status();
}

struct WgPlan {
    int RB, JB, BB, rt, bt, jt0, jt1, tiles0, ptiles;
    int kchunks, cpo, n_atoms, groups, co_tiles, chunks, tiles_per_chunk;
    bool pair;  // 2-CTA kernel (co_tiles then counts 256-channel pairs)
};

static bool wg_use_pair(int Cin, int Cout) {
    if (sw_on("HEXCONV_NO_2SM")) return false;
    return Cout % 256 == 0 && Cin % 128 == 0;
}

static int wg_pix(int) { return 64; }

static WgPlan wg_plan(const Geom& g, int Cin, int Cout) {
    WgPlan w{};
    choose_box(g.B, g.H, g.W, wg_pix(Cin), &w.RB, &w.JB, &w.BB);
    w.rt = ceil_div(g.H, w.RB);
    w.bt = ceil_div(g.B, w.BB);
    w.jt0 = ceil_div((g.W + 1) / 2, w.JB);
    w.jt1 = ceil_div(g.W / 2, w.JB);
    w.tiles0 = w.rt * w.jt0 * w.bt;
    w.ptiles = w.tiles0 + w.rt * w.jt1 * w.bt;
    w.kchunks = Cin / 64;
    w.cpo = 1;  // largest power of two dividing kchunks and the 8-atom group
    while (w.cpo < 8 && w.kchunks % (2 * w.cpo) == 0) w.cpo *= 2;
    w.n_atoms = g.T * w.kchunks;
    w.groups = ceil_div(w.n_atoms, WG_ATOMS);
    w.pair = wg_use_pair(Cin, Cout);
    w.co_tiles = w.pair ? Cout / 256 : Cout / 128;
    const int base_units = w.co_tiles * w.groups;
    // whole waves: the largest chunk count with base_units * chunks <= 2 x 148 SMs (one CTA per SM, a pair
    // unit takes two) -- one wave of pair units for n = 1, whose 7-tap units are short enough that a second
    // wave's extra partials cost more than its balance gains (C5 layer 6: 124 vs 132 us, A/B in fresh
    // processes on one box; n = 2 keeps two waves: layer 5 270 vs 274 us).  A fixed SM count keeps the split-K summation order identical on every
    // B200.
    int chunks = (w.pair ? (g.n == 1 ? 74 : 148) : 2 * 148) / base_units;
    if (chunks > w.ptiles) chunks = w.ptiles;
    if (chunks < 1) chunks = 1;
    w.tiles_per_chunk = ceil_div(w.ptiles, chunks);
    w.chunks = ceil_div(w.ptiles, w.tiles_per_chunk);
    return w;
}

bool tc_wgrad_supported(const Geom& g, int Cin, int Cout) {
    if (g.s != 1 || g.T > TC_MAXT || g.W < 2) return false;
    if (Cout % 128 != 0 || Cin % 64 != 0) return false;
    if (sw_on("HEXCONV_DISABLE_TC")) return false;
    return get_encode() != nullptr;
}

size_t tc_wgrad_ws_bytes(const Geom& g, int Cin, int Cout) {
    if (tc_wgrad_tr_supported(g, Cin, Cout)) return tc_wgrad_tr_ws_bytes(g, Cin, Cout);
    const WgPlan w = wg_plan(g, Cin, Cout);
    return (size_t)w.chunks * g.T * Cout * Cin * sizeof(float) + (size_t)w.chunks * Cout * sizeof(float) + 256;
}

template <int PIX>
static hex_status_t launch_wgrad_pix(const CUtensorMap& mx0, const CUtensorMap& mx1, const CUtensorMap& md0,
                                     const CUtensorMap& md1, const TcWgParams& p, int units, cudaStream_t st) {
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(tc_conv_wgrad_kernel<PIX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 WgCfg<PIX>::SMEM) != cudaSuccess)
            return HEX_ERR_CUDA;
        attr_set = true;
    }
    tc_conv_wgrad_kernel<PIX><<<units, 192, WgCfg<PIX>::SMEM, st>>>(mx0, mx1, md0, md1, p);
    return HEX_OK;
}

hex_status_t tc_conv3d_wgrad(const TcWgradArgs& a, const TrDepth& dz, void* ws, size_t ws_bytes, cudaStream_t st) {
    int chunks = 0;
    float* db_part = nullptr;
    const hex_status_t s = tc_wgrad_tr(a, ws, ws_bytes, &chunks, &db_part, st, &dz);
    if (s != HEX_OK) return s;
    return wgrad_reduce((const float*)ws, chunks, a.g.T, a.Cout, dz.kd * a.Cin, a.dw, db_part, a.dbias, a.accumulate,
                        st);
}

// strides 2 and 3: the one-box-per-tap weight gradient walks the dy LATTICE directly -- its
// pixel tiles are tiles of the lattice's column-parity views and every tap's x box is read with element stride
// s (wg_xbox) -- instead of the stride-1 kernel on dy scattered onto the full grid (s^2 x the MMAs, mostly zeros)
static Geom lattice_geom(const Geom& g) {
    Geom gl = g;
    gl.H = g.Ho;
    gl.W = g.Wo;
    gl.s = 1;
    return gl;
}

bool tc_wgrad_lat_supported(const Geom& g, int Cin, int Cout) {
    if ((g.s != 2 && g.s != 3) || g.T > TC_MAXT || g.Wo < 2 || Cout % 128 != 0 || Cin % 64 != 0) return false;
    if (sw_on("HEXCONV_DISABLE_TC") || sw_on("HEXCONV_NO_TC_WGRAD_LAT")) return false;
    const WgPlan w = wg_plan(lattice_geom(g), Cin, Cout);
    if (w.RB * g.s > 256 || w.JB * g.s > 256) return false;
    return get_encode() != nullptr;
}

size_t tc_wgrad_lat_ws_bytes(const Geom& g, int Cin, int Cout) {
    const WgPlan w = wg_plan(lattice_geom(g), Cin, Cout);
    return (size_t)w.chunks * g.T * Cout * Cin * sizeof(float) + (size_t)w.chunks * Cout * sizeof(float) + 256;
}

hex_status_t tc_conv_wgrad(const TcWgradArgs& a, void* ws, size_t ws_bytes, cudaStream_t st) {
    const Geom& g = a.g;
    const bool lat = g.s > 1;
    if (!lat && tc_wgrad_tr_supported(g, a.Cin, a.Cout)) {  // tap-reuse kernel (tc_wgrad_tr.cu)
        int chunks = 0;
        float* db_part = nullptr;
        const hex_status_t s = tc_wgrad_tr(a, ws, ws_bytes, &chunks, &db_part, st);
        if (s != HEX_OK) return s;
        return wgrad_reduce((const float*)ws, chunks, g.T, a.Cout, a.Cin, a.dw, db_part, a.dbias, a.accumulate, st);
    }
    const Geom gt = lat ? lattice_geom(g) : g;  // the grid the pixel tiles walk
    const WgPlan w = wg_plan(gt, a.Cin, a.Cout);
    if (ws_bytes < (lat ? tc_wgrad_lat_ws_bytes(g, a.Cin, a.Cout) : tc_wgrad_ws_bytes(g, a.Cin, a.Cout)))
        return HEX_ERR_WORKSPACE;
    TcWgParams p{};
    p.B = g.B; p.H = gt.H; p.W = gt.W; p.Cin = a.Cin; p.Cout = a.Cout; p.T = g.T; p.parity = g.parity;
    p.s = g.s;
    p.RB = w.RB; p.JB = w.JB; p.BB = w.BB; p.rt = w.rt; p.bt = w.bt; p.jt0 = w.jt0; p.jt1 = w.jt1;
    p.tiles0 = w.tiles0; p.ptiles = w.ptiles;
    p.kchunks = w.kchunks; p.cpo = w.cpo; p.n_atoms = w.n_atoms; p.groups = w.groups; p.co_tiles = w.co_tiles;
    p.chunks = w.chunks; p.tiles_per_chunk = w.tiles_per_chunk;
    p.part = (float*)ws;
    p.db_part = a.dbias ? (float*)ws + (size_t)w.chunks * g.T * a.Cout * a.Cin : nullptr;
    p.dbg = debug_mode("HEXCONV_WG_DEBUG");
    for (int pc = 0; pc < 2; ++pc)
        for (int t = 0; t < g.T; ++t) {
            int dc, dr;
            tap_offset(g.n, pc, t, &dc, &dr);
            p.tap_dc[pc][t] = (int8_t)dc;
            p.tap_dr[pc][t] = (int8_t)dr;
        }
    CUtensorMap mx0, mx1, md0, md1;
    const int xbox = w.pair ? 2 : w.cpo;
    const int es = g.s;
    if (!make_view_map5(&mx0, a.x, g.B, g.H, g.W, a.Cin, 0, w.RB, w.JB, w.BB, xbox, es)) return HEX_ERR_CUDA;
    if (!make_view_map5(&mx1, a.x, g.B, g.H, g.W, a.Cin, 1, w.RB, w.JB, w.BB, xbox, es)) return HEX_ERR_CUDA;
    if (!make_view_map5(&md0, a.dy, g.B, gt.H, gt.W, a.Cout, 0, w.RB, w.JB, w.BB, 2)) return HEX_ERR_CUDA;
    if (!make_view_map5(&md1, a.dy, g.B, gt.H, gt.W, a.Cout, 1, w.RB, w.JB, w.BB, 2)) return HEX_ERR_CUDA;
    const int units = w.co_tiles * w.groups * w.chunks;
    if (w.pair) {
        static bool attr2 = false;
        if (!attr2) {
            if (cudaFuncSetAttribute(tc_conv_wgrad2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     Wg2Cfg::SMEM) != cudaSuccess)
                return HEX_ERR_CUDA;
            attr2 = true;
        }
        tc_conv_wgrad2_kernel<<<2 * units, 192, Wg2Cfg::SMEM, st>>>(mx0, mx1, md0, md1, p);
    } else if (wg_pix(a.Cin) == 32) {
        if (launch_wgrad_pix<32>(mx0, mx1, md0, md1, p, units, st) != HEX_OK) return HEX_ERR_CUDA;
    } else {
        if (launch_wgrad_pix<64>(mx0, mx1, md0, md1, p, units, st) != HEX_OK) return HEX_ERR_CUDA;
    }
    count_launch();
    return wgrad_reduce((const float*)ws, w.chunks, g.T, a.Cout, a.Cin, a.dw, p.db_part, a.dbias, a.accumulate, st);
}

}  // namespace hexconv
