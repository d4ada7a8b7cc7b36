// tc_fwd_tr.cu -- tcgen05 hexagonal convolution forward (and stride-1
// backward-data) with TAP REUSE of the A operand (bf16 NHWC, fp32 accumulation
// in tensor memory).
//
//   y[px][co] = bias[co] + sum_t sum_ci x[px + off_t(parity(px))][ci] w[t][co][ci]
// (the sum over the kernel footprint; off-grid taps
// are TMA's zero fill, A4).  Backward-data at stride 1 is the same
// computation on dy with W'[ci][co][t] = W[co][ci][T-1-t] (oracle pin P18).
//
// Output tiles are 16 rows x 8 sub-columns of one parity view of one image in
// row-major order, so M = 128 pixels and one image row is one 1024-byte SW128
// atom of the K-major A operand.  For a tile of view P the taps of kernel
// column dc all read view P' = (P + dc) mod 2 at one sub-column shift and
// differ only by their row: ONE A box of 16 + 2n rows per (column, 64-channel
// chunk) serves every tap of the column, tap k being the 128-row window k atoms
// into the box.  Per tile and chunk that is 2n+1 box loads of (16+2n)/16 tiles
// instead of T = 3n(n+1)+1 tile loads (n = 1: 7 -> 3.4 tiles of traffic).
// Weights are either resident in shared memory for the whole kernel (loaded
// once per CTA when T x Cout x Cin fits) or streamed with each stage.
//
// Persistent, warp specialised: warp 0 TMA producer, warp 1 MMA issuer (all
// shapes compile-time, descriptors advanced by 64-bit adds: see DESIGN.md
// "MMA issue"), warps 2-9 the epilogue (bias, ReLU or the ReLU-backward mask,
// bf16 RNE, SW128 staging, TMA store), two TMEM accumulators.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hexconv {

namespace {

constexpr int FT_RB = 16, FT_JB = 8;  // output tile: 16 rows x 8 sub-columns = 128 pixels
constexpr int FT_EPI = 256;           // epilogue threads (8 warps, two per TMEM lane quadrant)
constexpr int FT_THREADS = 64 + FT_EPI;
constexpr int FT_OUT = 128 * 128;     // one 64-channel output chunk staged (16 KB)
constexpr int FT_SMEM_MAX = 227 * 1024;

struct FtParams {
    int B, H, W, Cin, Cout, T, parity;
    int rt, jt0, jt1, tiles0, mtiles, n_tiles, total_tiles, kchunks, stages;
    int pair_tiles;  // CTA-pair kernel: (n tile, pair of m tiles) work items
    int relu, has_mask;
    int debug;  // HEXCONV_FT_DEBUG: 1 = epilogue skipped, 2 = MMAs skipped (timing experiments)
    // 3-D convolution: tile image index b is an OUTPUT slice b = vol * Do + zo; depth
    // tap kz reads input image vol * D + sd * zo + kz - pd (a fully out-of-bounds box -- zeros -- when
    // that slice is outside the volume), weight taps kz * T + t.  2-D: kd = D = Do = sd = 1, pd = 0.
    int kd, D, Do, sd, pd;
    const float* bias;
};

__device__ __forceinline__ void ft_decode(const FtParams& p, int tile, int BN, int* P, int* r0, int* j0, int* b,
                                          int* n0) {
    const int nt = tile % p.n_tiles;
    int m = tile / p.n_tiles;
    *n0 = nt * BN;
    int jt;
    if (p.jt0 == p.jt1) { *P = m & 1; m >>= 1; jt = p.jt0; }  // views interleaved (L2 reuse across views)
    else if (m < p.tiles0) { *P = 0; jt = p.jt0; }
    else { *P = 1; m -= p.tiles0; jt = p.jt1; }
    const int rti = m % p.rt;
    m /= p.rt;
    const int jti = m % jt;
    *b = m / jt;
    *r0 = rti * FT_RB;
    *j0 = jti * FT_JB;
}

// CTA pairs: work item = (n tile, pair of consecutive m tiles); CTA `rank` takes m tile 2 mp + rank.
// A missing odd tile gets r0 = H: its loads are zero fill and its stores are clipped.
__device__ __forceinline__ void ft_decode_pair(const FtParams& p, int ptile, int BN, int rank, int* P, int* r0,
                                               int* j0, int* b, int* n0) {
    const int nt = ptile % p.n_tiles;
    const int m = 2 * (ptile / p.n_tiles) + rank;
    if (m >= p.mtiles) {
        *P = 0; *r0 = p.H; *j0 = 0; *b = 0; *n0 = nt * BN;
        return;
    }
    ft_decode(p, m * p.n_tiles + nt, BN, P, r0, j0, b, n0);
}

// Stage list of one 64-channel chunk: (kernel column, first tap, tap count), taps of a column split
// into groups of <= TG (streamed weights: each stage also carries its taps' weight tiles).
template <int N, int TG>
struct StageList {
    __host__ __device__ static constexpr int len(int dc) { return 2 * N + 1 - (dc < 0 ? -dc : dc); }
    __host__ __device__ static constexpr int groups(int dc) { return (len(dc) + TG - 1) / TG; }
    __host__ __device__ static constexpr int count() {
        int c = 0;
        for (int dc = -N; dc <= N; ++dc) c += groups(dc);
        return c;
    }
    // stage s -> dc, g0 (first tap within the column), cnt, tb (canonical index of the column's tap 0)
    __host__ __device__ static constexpr int dc_of(int s) {
        for (int dc = -N; dc <= N; ++dc) {
            if (s < groups(dc)) return dc;
            s -= groups(dc);
        }
        return 0;
    }
    __host__ __device__ static constexpr int g0_of(int s) {
        for (int dc = -N; dc <= N; ++dc) {
            if (s < groups(dc)) return s * TG;
            s -= groups(dc);
        }
        return 0;
    }
    __host__ __device__ static constexpr int cnt_of(int s) {
        const int dc = dc_of(s), g0 = g0_of(s);
        return len(dc) - g0 < TG ? len(dc) - g0 : TG;
    }
    __host__ __device__ static constexpr int tb_of(int s) {
        const int dc = dc_of(s);
        int t = 0;
        for (int c = -N; c < dc; ++c) t += len(c);
        return t;
    }
};

// MMAs of one stage: taps g0 .. g0+CNT-1 of the column, 4 K-steps of 16 channels each.
template <int BN, int CNT, bool RES>
__device__ __forceinline__ void issue_stage(uint32_t d, uint64_t a_desc, uint64_t b_desc, int b_tap_stride16,
                                            uint32_t first) {
    constexpr uint32_t idesc = ptx::idesc_bf16(128, BN, 0, 0);
#pragma unroll
    for (int i = 0; i < CNT; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k)
            ptx::mma_bf16(d, a_desc + (uint64_t)(i * 64 + k * 2), b_desc + (uint64_t)(i * b_tap_stride16 + k * 2),
                          idesc, (i | k) ? 1u : first);
}

// the same for a CTA pair (M = 256, issued by the leader)
template <int BN, int CNT>
__device__ __forceinline__ void issue_stage_pair(uint32_t d, uint64_t a_desc, uint64_t b_desc, int b_tap_stride16,
                                                 uint32_t first) {
    constexpr uint32_t idesc = ptx::idesc_bf16(256, BN, 0, 0);
#pragma unroll
    for (int i = 0; i < CNT; ++i)
#pragma unroll
        for (int k = 0; k < 4; ++k)
            ptx::mma_bf16_2sm(d, a_desc + (uint64_t)(i * 64 + k * 2), b_desc + (uint64_t)(i * b_tap_stride16 + k * 2),
                              idesc, (i | k) ? 1u : first);
}

template <int BN, int N, int TG, bool RES, bool PAIR, int S>
__device__ __forceinline__ void issue_stages_from(uint32_t d, uint64_t a_ring, uint64_t b_ring, uint64_t res_desc,
                                                  uint64_t* full, uint64_t* empty, int& stage, uint32_t& phase,
                                                  int nstages, uint32_t stage16, uint32_t a_bytes16, int kc,
                                                  int kchunks, uint32_t first) {
    using SL = StageList<N, TG>;
    if constexpr (S < SL::count()) {
        constexpr int g0 = SL::g0_of(S), cnt = SL::cnt_of(S), tb = SL::tb_of(S);
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t soff = (uint64_t)stage * stage16;
        const uint64_t ad = a_ring + soff + (uint64_t)(g0 * 64);  // tap g0 = g0 rows (1024 B) into the box
        uint64_t bd;
        int bstride;
        constexpr int BROWS = PAIR ? BN / 2 : BN;  // weight rows held per CTA
        if (RES) {  // resident weights: tile (t, kc) at ((t * kchunks + kc) * BROWS * 128) bytes
            bd = res_desc + (uint64_t)(((tb + g0) * kchunks + kc) * (BROWS * 8));
            bstride = kchunks * BROWS * 8;
        } else {
            bd = b_ring + soff + a_bytes16;
            bstride = BROWS * 8;
        }
        if constexpr (PAIR) {
            issue_stage_pair<BN, cnt>(d, ad, bd, bstride, S == 0 ? first : 1u);
            ptx::mma_commit_2sm(&empty[stage]);
        } else {
            issue_stage<BN, cnt, RES>(d, ad, bd, bstride, S == 0 ? first : 1u);
            ptx::mma_commit(&empty[stage]);
        }
        if (++stage == nstages) { stage = 0; phase ^= 1; }
        issue_stages_from<BN, N, TG, RES, PAIR, S + 1>(d, a_ring, b_ring, res_desc, full, empty, stage, phase, nstages,
                                                  stage16, a_bytes16, kc, kchunks, 1u);
    }
}

}  // namespace

template <int BN, int N, int TG, bool RES, bool PAIR>
__global__ void __launch_bounds__(FT_THREADS, 1)
tc_fwd_tr_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                 const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_y0,
                 const __grid_constant__ CUtensorMap map_y1, const __grid_constant__ CUtensorMap map_m0,
                 const __grid_constant__ CUtensorMap map_m1, const __grid_constant__ FtParams p) {
    using SL = StageList<N, TG>;
    constexpr int A_BYTES = (FT_RB + 2 * N) * FT_JB * 128;   // one A box
    constexpr int W_TILE = (PAIR ? BN / 2 : BN) * 128;         // one (tap, chunk) weight tile (this CTA's rows)
    constexpr int STAGE = RES ? A_BYTES : A_BYTES + TG * W_TILE;
    constexpr int TMEM_COLS = 2 * BN;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned
    const int res_bytes = RES ? p.T * p.kchunks * W_TILE : 0;
    uint8_t* resw = base;
    uint8_t* ring = base + res_bytes;
    uint8_t* obuf = ring + p.stages * STAGE;
    uint64_t* full = (uint64_t*)(obuf + 2 * FT_OUT);
    uint64_t* empty = full + p.stages;
    uint64_t* tfull = empty + p.stages;
    uint64_t* tempty = tfull + 2;
    uint64_t* mbar = tempty + 2;
    uint64_t* bres = mbar + 2;
    uint32_t* tmem_slot = (uint32_t*)(bres + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], (PAIR ? 2 : 1) * FT_EPI / 32);  // pairs: both CTAs' epilogue warps
            ptx::mbar_init(&mbar[a], 1);
        }
        ptx::mbar_init(bres, 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x0);
        ptx::prefetch_tmap(&map_x1);
        ptx::prefetch_tmap(&map_w);
        ptx::prefetch_tmap(&map_y0);
        ptx::prefetch_tmap(&map_y1);
    }
    if (warp == 1) {
        if constexpr (PAIR) ptx::tmem_alloc_2sm(tmem_slot, TMEM_COLS);
        else ptx::tmem_alloc(tmem_slot, TMEM_COLS);
    }
    ptx::tc_fence_before();
    if constexpr (PAIR) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            if constexpr (RES) {
                if constexpr (PAIR) {  // each CTA holds its half of every tile; bytes land on the leader
                    if (leader) ptx::mbar_arrive_expect_tx(bres, (uint32_t)(2 * res_bytes));
                    for (int t = 0; t < p.T; ++t)
                        for (int kc = 0; kc < p.kchunks; ++kc)
                            ptx::tma_load_4d_2sm(&map_w, bres, resw + (t * p.kchunks + kc) * W_TILE, 0,
                                                 (int)rank * (BN / 2), kc, t);
                } else {
                    ptx::mbar_arrive_expect_tx(bres, (uint32_t)res_bytes);
                    for (int t = 0; t < p.T; ++t)
                        for (int kc = 0; kc < p.kchunks; ++kc)
                            ptx::tma_load_4d(&map_w, bres, resw + (t * p.kchunks + kc) * W_TILE, 0, 0, kc, t);
                }
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = PAIR ? blockIdx.x / 2 : blockIdx.x; tile < (PAIR ? p.pair_tiles : p.total_tiles);
             tile += PAIR ? gridDim.x / 2 : gridDim.x) {
                int P, r0, j0, b, n0;
                if (PAIR) ft_decode_pair(p, tile, BN, (int)rank, &P, &r0, &j0, &b, &n0);
                else ft_decode(p, tile, BN, &P, &r0, &j0, &b, &n0);
                const int pc = (P + p.parity) & 1;  // centre column parity
                const int vol = b / p.Do, zo = b - vol * p.Do;
                for (int kz = 0; kz < p.kd; ++kz)
                for (int kc = 0; kc < p.kchunks; ++kc) {
                    const int z = p.sd * zo + kz - p.pd;
                    const bool zin = z >= 0 && z < p.D;
                    const int img = vol * p.D + (zin ? z : 0);
                    const int roff = zin ? 0 : p.H + 64;  // outside the volume: the box is all zero fill
#pragma unroll 1
                    for (int s = 0; s < SL::count(); ++s) {
                        const int dc = SL::dc_of(s), g0 = SL::g0_of(s), cnt = SL::cnt_of(s), tb = SL::tb_of(s);
                        const int Pv = (P + dc) & 1;
                        const int jsh = (P + dc - Pv) / 2;
                        const int top = -N + (((dc < 0 ? -dc : dc) + pc) >> 1);
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = ring + stage * STAGE;
                        const uint32_t bytes = RES ? A_BYTES : A_BYTES + cnt * W_TILE;
                        if constexpr (PAIR) {  // both CTAs' bytes land on the leader's barrier
                            if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * bytes);
                            ptx::tma_load_5d_2sm(Pv ? &map_x1 : &map_x0, &full[stage], sa, 0, j0 + jsh,
                                                 r0 + top + roff, img, kc);
                            if constexpr (!RES)
                                for (int i = 0; i < cnt; ++i)
                                    ptx::tma_load_4d_2sm(&map_w, &full[stage], sa + A_BYTES + i * W_TILE, 0,
                                                         n0 + (int)rank * (BN / 2), kc, kz * p.T + tb + g0 + i);
                        } else {
                            ptx::mbar_arrive_expect_tx(&full[stage], bytes);
                            ptx::tma_load_5d(Pv ? &map_x1 : &map_x0, &full[stage], sa, 0, j0 + jsh, r0 + top + roff,
                                             img, kc);
                            if constexpr (!RES)
                                for (int i = 0; i < cnt; ++i)
                                    ptx::tma_load_4d(&map_w, &full[stage], sa + A_BYTES + i * W_TILE, 0, n0, kc,
                                                     kz * p.T + tb + g0 + i);
                        }
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && (!PAIR || leader)) {
            const uint64_t a_ring = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
            const uint64_t b_ring = a_ring;  // streamed weight tiles sit A_BYTES into the stage
            const uint64_t res_desc = ptx::smem_desc_sw128(ptx::smem_u32(resw), 16, 1024);
            const uint32_t stage16 = STAGE >> 4, a_bytes16 = A_BYTES >> 4;
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t aphase = 0;
            if constexpr (RES) ptx::mbar_wait(bres, 0);
            for (int tile = PAIR ? blockIdx.x / 2 : blockIdx.x; tile < (PAIR ? p.pair_tiles : p.total_tiles);
                 tile += PAIR ? gridDim.x / 2 : gridDim.x) {
                ptx::mbar_wait(&tempty[acc], aphase ^ 1);
                ptx::tc_fence_after();
                const uint32_t d = tmem_base + acc * BN;
                if (HEX_DBG(p.debug) == 2) {
                    for (int u = 0; u < p.kd * p.kchunks * SL::count(); ++u) {
                        ptx::mbar_wait(&full[stage], phase);
                        ptx::mbar_arrive(&empty[stage]);
                        if (PAIR) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&empty[stage]), 1));
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                    ptx::mbar_arrive(&tfull[acc]);
                    if (PAIR) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tfull[acc]), 1));
                    acc ^= 1;
                    if (acc == 0) aphase ^= 1;
                    continue;
                }
                for (int kz = 0; kz < p.kd; ++kz)
                    for (int kc = 0; kc < p.kchunks; ++kc)
                        issue_stages_from<BN, N, TG, RES, PAIR, 0>(d, a_ring, b_ring, res_desc, full, empty, stage,
                                                                   phase, p.stages, stage16, a_bytes16, kc,
                                                                   p.kchunks, (kz | kc) == 0 ? 0u : 1u);
                if constexpr (PAIR) ptx::mma_commit_2sm(&tfull[acc]);
                else ptx::mma_commit(&tfull[acc]);
                acc ^= 1;
                if (acc == 0) aphase ^= 1;
            }
        }
    } else {
        // Epilogue: warps 2..9; warp w owns TMEM lane quadrant w % 4 (tile row m = TMEM lane) and
        // column half h of every 64-channel chunk.  Per chunk: TMEM -> registers -> (bias, ReLU |
        // ReLU-backward mask) -> bf16 -> SW128 staging row m -> one TMA store of the 16 x 8 box.
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        const int row = q * 32 + lane;
        const int et = threadIdx.x - 64;
        int acc = 0;
        uint32_t aphase = 0;
        int ob = 0;
        uint32_t mphase0 = 0, mphase1 = 0;
        // ReLU-backward mask tiles are TMA-loaded one chunk ahead -- across tile boundaries too, so
        // the next tile's first mask chunk is in flight while the current tile's last chunk drains
        if (p.has_mask && et == 0 && HEX_DBG(p.debug) != 1) {
            const int t0 = PAIR ? blockIdx.x / 2 : blockIdx.x;
            if (t0 < (PAIR ? p.pair_tiles : p.total_tiles)) {
                int P, r0, j0, b, n0;
                if (PAIR) ft_decode_pair(p, t0, BN, (int)rank, &P, &r0, &j0, &b, &n0);
                else ft_decode(p, t0, BN, &P, &r0, &j0, &b, &n0);
                ptx::mbar_arrive_expect_tx(&mbar[0], FT_OUT);
                ptx::tma_load_4d(P ? &map_m1 : &map_m0, &mbar[0], obuf, n0, j0, r0, b);
            }
        }
        for (int tile = PAIR ? blockIdx.x / 2 : blockIdx.x; tile < (PAIR ? p.pair_tiles : p.total_tiles);
             tile += PAIR ? gridDim.x / 2 : gridDim.x) {
            int P, r0, j0, b, n0;
            if (PAIR) ft_decode_pair(p, tile, BN, (int)rank, &P, &r0, &j0, &b, &n0);
            else ft_decode(p, tile, BN, &P, &r0, &j0, &b, &n0);
            const CUtensorMap* my = P ? &map_y1 : &map_y0;
            const CUtensorMap* mm = P ? &map_m1 : &map_m0;
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int ch = 0; ch < (HEX_DBG(p.debug) == 1 ? 0 : BN / 64); ++ch) {
                uint8_t* buf = obuf + ob * FT_OUT;
                const int c0 = n0 + ch * 64;
                if (p.has_mask) {
                    ptx::mbar_wait(&mbar[ob], ob ? mphase1 : mphase0);
                    if (ob) mphase1 ^= 1; else mphase0 ^= 1;
                } else {
                    if (et == 0) ptx::bulk_wait_read<1>();
                    ptx::named_bar(1, FT_EPI);
                }
                uint32_t v[32];
                ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + ch * 64 + h * 32, v);
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
                    if (p.relu && !p.has_mask) {  // ReLU inside the conversion (bit-identical to fmaxf + cvt)
                        *slot = make_uint4(ptx::pack_bf16x2_relu(f[0], f[1]), ptx::pack_bf16x2_relu(f[2], f[3]),
                                           ptx::pack_bf16x2_relu(f[4], f[5]), ptx::pack_bf16x2_relu(f[6], f[7]));
                        continue;
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
                        __nv_bfloat162 hv = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
                        pk[k] = *reinterpret_cast<uint32_t*>(&hv);
                    }
                    *slot = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                ptx::fence_proxy_async();
                ptx::named_bar(1, FT_EPI);
                if (et == 0) {
                    ptx::tma_store_4d(my, buf, c0, j0, r0, b);
                    ptx::bulk_commit();
                    if (p.has_mask) {
                        if (ch + 1 < BN / 64) {
                            ptx::bulk_wait_read<1>();
                            ptx::mbar_arrive_expect_tx(&mbar[ob ^ 1], FT_OUT);
                            ptx::tma_load_4d(mm, &mbar[ob ^ 1], obuf + (ob ^ 1) * FT_OUT, c0 + 64, j0, r0, b);
                        } else {
                            const int nt = tile + (PAIR ? gridDim.x / 2 : gridDim.x);
                            if (nt < (PAIR ? p.pair_tiles : p.total_tiles)) {
                                int P2, r2, j2, b2, n2;
                                if (PAIR) ft_decode_pair(p, nt, BN, (int)rank, &P2, &r2, &j2, &b2, &n2);
                                else ft_decode(p, nt, BN, &P2, &r2, &j2, &b2, &n2);
                                ptx::bulk_wait_read<1>();
                                ptx::mbar_arrive_expect_tx(&mbar[ob ^ 1], FT_OUT);
                                ptx::tma_load_4d(P2 ? &map_m1 : &map_m0, &mbar[ob ^ 1], obuf + (ob ^ 1) * FT_OUT, n2,
                                                 j2, r2, b2);
                            }
                        }
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
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) ptx::cluster_sync();  // the peer's smem / TMEM must outlive the leader's last MMA
    if (warp == 1) {
        ptx::tc_fence_after();
        if constexpr (PAIR) ptx::tmem_dealloc_2sm(tmem_base, TMEM_COLS);
        else ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ------------------------------------------------------------------ fused conv -> ReLU -> max pool
// maxpool_{n=1,s=2}(relu(conv(x) + bias)) without writing the conv output.
// Column geometry: window centre column 2C is view-0 sub-column C; its side columns 2C -+ 1 are view-1
// sub-columns C-1 and C.  A column STRIP k computes view-0 sub-columns [7k, 7k+8) and view-1 sub-columns
// [7k-1, 7k+7) (two 16 x 8 tap-reuse tiles, two TMEM accumulators) and owns window columns [7k, 7k+7).
// Rows: a strip walks down the image in tiles of 16 conv rows (r0 = 16 t) and carries the last two rows
// of each tile (bf16) in shared memory, so tile t owns the windows with centre row cr in [r0-1, r0+14]
// (+ r0+15 on the last tile) and no row is computed twice.  Strips are dealt round-robin to the
// persistent CTAs in whole rounds; the strips left over after the last whole round are cut into
// independent REGIONS (r0 = 14 i - 1, centre rows [14 i, 14 i + 14), halo rows recomputed) so the tail
// spreads over all CTAs.
// Epilogue, warp-specialised per 32-channel chunk: 8 CONVERTER warps (one per TMEM lane quadrant and
// view) drain the accumulators (bias, ReLU, bf16; pixels outside the image become -inf) into one of two
// region buffers (rows r0-2 .. r0+16), 8 WINDOW warps reduce the owned windows from the other buffer:
// first maximum in canonical tap order (A9), value = the bf16 conv output of that tap --
// bit-identical to the unfused conv + pool.  Named barriers FULL/EMPTY per buffer.  The conv output
// never reaches HBM.
constexpr int FP_ROWS = FT_RB + 3;               // region rows: 2 carried + 16 tile + 1 (-inf)
constexpr int FP_PIX = 64;                       // bytes per pixel per chunk (32 channels bf16)
constexpr int FP_VIEW = FP_ROWS * FT_JB * FP_PIX;  // one view of one chunk (9.5 KB)
constexpr int FP_BUF = 2 * FP_VIEW;                // both views
constexpr int FP_CARRY = 2 * 2 * FT_JB * FP_PIX;   // carried rows of one chunk: 2 views x 2 rows (2 KB)
constexpr int FP_EPI = 512;                      // 8 converter + 8 window warps
constexpr int FP_THREADS = 64 + FP_EPI;
constexpr int FP_BAR_FULL = 2, FP_BAR_EMPTY = 6;  // named barrier ids (+ buffer index, up to 4 buffers)

// byte offset of 16-byte channel group i (0..3) of pixel (region row r, sub-column sc): conflict-free
// for 8 consecutive pixels of one group and for 2 adjacent sub-columns x 4 groups
__device__ __forceinline__ int fp_off(int r, int sc, int i) {
    return r * (FT_JB * FP_PIX) + sc * FP_PIX + ((i ^ ((sc >> 1) & 3)) << 4);
}

struct FpParams {
    int B, H, W, Cin, Cout, T, parity, Ho, Wo;
    int nr, nc, kchunks, stages, relu;
    int ntr;           // tiles per strip = ceil(H / 16)
    int full_rounds;   // strips per CTA in strip mode
    int left_regions;  // regions cut from the strips after full_rounds * gridDim.x
    int debug;         // HEXCONV_FP_DEBUG: 1 = no epilogue work, 2 = no MMAs, 3 = window warps idle, 4 = no
                       // converter stores (timing experiments; -DHEXCONV_TIMING_DEBUG=1 builds only)
    int nreg;          // region buffers, 2 or 4 (4: the converters drain a whole tile ahead of the windows)
    const float* bias;
    uint16_t* y;   // pooled bf16 NHWC [B][Ho][Wo][Cout]
    uint8_t* am;   // argmax tap [B][Ho][Wo][Cout]
};

struct FpTile {
    int b, k, r0;
    bool strip, first, last;
    bool valid;  // false: a CTA-pair tail slot with no region (loads zero fill, nothing is stored)
};

// the seq-th tile of this CTA; false past the end.  CTA pairs (PAIR): the two CTAs of a cluster walk
// strips 2u and 2u+1 (regions likewise) in lockstep; both CTAs end together.
template <bool PAIR>
__device__ __forceinline__ bool fp_tile(const FpParams& p, int seq, FpTile& tl) {
    const int cid = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
    const int ncl = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
    const int rank = PAIR ? (int)(blockIdx.x & 1) : 0;
    const int per = PAIR ? 2 : 1;
    const int ns = p.full_rounds * p.ntr;
    tl.valid = true;
    if (seq < ns) {
        const int j = seq / p.ntr, t = seq - j * p.ntr;
        const int strip = (cid + j * ncl) * per + rank;
        tl.b = strip / p.nc;
        tl.k = strip - tl.b * p.nc;
        tl.r0 = FT_RB * t;
        tl.strip = true;
        tl.first = t == 0;
        tl.last = t == p.ntr - 1;
        return true;
    }
    const int rgu = cid + (seq - ns) * ncl;
    if (rgu * per >= p.left_regions) return false;
    int rg = rgu * per + rank;
    if (rg >= p.left_regions) {  // pair tail: a slot without a region
        tl.valid = false;
        rg = p.left_regions - 1;
    }
    const int strip = p.full_rounds * ncl * per + rg / p.nr;
    const int i = rg % p.nr;
    tl.b = strip / p.nc;
    tl.k = strip - tl.b * p.nc;
    tl.r0 = tl.valid ? 14 * i - 1 : p.H + 64;
    tl.strip = tl.first = tl.last = false;
    return true;
}

// one tap group of the view-pair MMA sequences: cta_group::1, or ::2 (M = 256 over a CTA pair)
template <int BN, int CNT, bool PAIR>
__device__ __forceinline__ void fv_group(uint32_t d, uint64_t ad, uint64_t bd, int bs, uint32_t first) {
    if constexpr (PAIR) issue_stage_pair<BN, CNT>(d, ad, bd, bs, first);
    else issue_stage<BN, CNT, true>(d, ad, bd, bs, first);
}

// n = 1 MMA sequence of one tile pair (view-0 tile -> accumulator d0, view-1 tile -> d1) from four
// 19-row boxes (top row r0 - 1) that each serve every column group reading them, in an order that keeps
// both accumulators in the canonical column order dc = -1, 0, +1 (same fp32 summation as the unfused
// forward):
//   box 0 = view 0 at sub-column 7k-1: view-1 dc = -1 (taps 0,1)
//   box 1 = view 1 at 7k-1:            view-0 dc = -1 (taps 0,1) and view-1 dc = 0 (taps 2..4)
//   box 2 = view 0 at 7k:              view-0 dc =  0 (taps 2..4) and view-1 dc = +1 (taps 5,6)
//   box 3 = view 1 at 7k:              view-0 dc = +1 (taps 5,6)
// A side column of view P starts pc_P = (P + parity) mod 2 rows below the box top.
template <int BN, bool PAIR>
__device__ __forceinline__ void fp_issue_n1(uint32_t d0, uint32_t d1, uint64_t a_ring, uint64_t res_desc,
                                            uint64_t* full, uint64_t* empty, int& stage, uint32_t& phase,
                                            int nstages, uint32_t stage16, int kc, int kchunks, uint32_t first,
                                            uint32_t pc0) {
    constexpr int BROWS = PAIR ? BN / 2 : BN;  // weight rows held per CTA
    const uint64_t o0 = (uint64_t)(pc0 * 64), o1 = (uint64_t)((pc0 ^ 1u) * 64);  // 1024-byte rows
    const int bs = kchunks * BROWS * 8;
    const uint64_t w0 = res_desc + (uint64_t)(kc * (BROWS * 8));  // tap t at w0 + t * bs
#pragma unroll
    for (int bx = 0; bx < 4; ++bx) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t ad = a_ring + (uint64_t)stage * stage16;
        if (bx == 0) {
            fv_group<BN, 2, PAIR>(d1, ad + o1, w0, bs, first);
        } else if (bx == 1) {
            fv_group<BN, 2, PAIR>(d0, ad + o0, w0, bs, first);
            fv_group<BN, 3, PAIR>(d1, ad, w0 + (uint64_t)(2 * bs), bs, 1u);
        } else if (bx == 2) {
            fv_group<BN, 3, PAIR>(d0, ad, w0 + (uint64_t)(2 * bs), bs, 1u);
            fv_group<BN, 2, PAIR>(d1, ad + o1, w0 + (uint64_t)(5 * bs), bs, 1u);
        } else {
            fv_group<BN, 2, PAIR>(d0, ad + o0, w0 + (uint64_t)(5 * bs), bs, 1u);
        }
        if constexpr (PAIR) ptx::mma_commit_2sm(&empty[stage]);
        else ptx::mma_commit(&empty[stage]);
        if (++stage == nstages) { stage = 0; phase ^= 1; }
    }
}

template <int BN, int N, bool PAIR, bool AVG>
__global__ void __launch_bounds__(FP_THREADS, 1)
tc_conv_maxpool_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                       const __grid_constant__ CUtensorMap map_w, const __grid_constant__ FpParams p) {
    constexpr int TG = 2 * N + 1;
    using SL = StageList<N, TG>;
    constexpr int A_BYTES = (FT_RB + 2 * N + (N == 1 ? 1 : 0)) * FT_JB * 128;  // n = 1: shared 19-row boxes
    constexpr int W_TILE = BN * 128;
    constexpr int TMEM_COLS = 4 * BN;  // 2 slots x 2 views
    constexpr int NCH = BN / 32;       // 32-channel chunks per tile
    constexpr uint32_t NEG_INF2 = 0xFF80FF80u;
    static_assert(!PAIR || N == 1, "CTA pairs: n = 1 only");
    constexpr int W_CTA = PAIR ? W_TILE / 2 : W_TILE;  // this CTA's rows of one (tap, chunk) weight tile
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned
    const int res_bytes = p.T * p.kchunks * W_CTA;
    uint8_t* resw = base;
    uint8_t* ring = base + res_bytes;
    uint8_t* region = ring + p.stages * A_BYTES;  // [buffer][view][row][sub-column][64 B]
    uint8_t* carry = region + p.nreg * FP_BUF;    // [chunk][view][2 rows][sub-column][64 B]
    float* sbias = (float*)(carry + NCH * FP_CARRY);  // [BN]
    uint64_t* full = (uint64_t*)(sbias + BN);
    uint64_t* empty = full + p.stages;
    uint64_t* tfull = empty + p.stages;
    uint64_t* tempty = tfull + 2;
    uint64_t* bres = tempty + 2;
    uint32_t* tmem_slot = (uint32_t*)(bres + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], PAIR ? 16 : 8);  // the converter warps (of both CTAs of a pair)
        }
        ptx::mbar_init(bres, 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x0);
        ptx::prefetch_tmap(&map_x1);
        ptx::prefetch_tmap(&map_w);
    }
    if (warp == 1) {
        if constexpr (PAIR) ptx::tmem_alloc_2sm(tmem_slot, TMEM_COLS);
        else ptx::tmem_alloc(tmem_slot, TMEM_COLS);
    }
    if (threadIdx.x >= 64) {  // region row 18 (r0 + 16) is only read on a strip's last tile: below the image
        const int e = threadIdx.x - 64;
        if (p.bias && e < BN) sbias[e] = p.bias[e];
        if (e < p.nreg * 2 * FT_JB * 4) {
            const int bf = e >> 6, v = (e >> 5) & 1, sc = (e >> 2) & 7, c16 = e & 3;
            *reinterpret_cast<uint4*>(region + bf * FP_BUF + v * FP_VIEW + fp_off(18, sc, c16)) =
                make_uint4(NEG_INF2, NEG_INF2, NEG_INF2, NEG_INF2);
        }
    }
    ptx::tc_fence_before();
    if constexpr (PAIR) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            if constexpr (PAIR) {  // each CTA holds its half of every weight tile; bytes land on the leader
                if (leader) ptx::mbar_arrive_expect_tx(bres, (uint32_t)(2 * res_bytes));
                for (int t = 0; t < p.T; ++t)
                    for (int kc = 0; kc < p.kchunks; ++kc)
                        ptx::tma_load_4d_2sm(&map_w, bres, resw + (t * p.kchunks + kc) * W_CTA, 0,
                                             (int)rank * (BN / 2), kc, t);
            } else {
                ptx::mbar_arrive_expect_tx(bres, (uint32_t)res_bytes);
                for (int t = 0; t < p.T; ++t)
                    for (int kc = 0; kc < p.kchunks; ++kc)
                        ptx::tma_load_4d(&map_w, bres, resw + (t * p.kchunks + kc) * W_TILE, 0, 0, kc, t);
            }
            int stage = 0;
            uint32_t phase = 0;
            FpTile tl;
            for (int seq = 0; fp_tile<PAIR>(p, seq, tl); ++seq) {
                if constexpr (N == 1) {
                    for (int kc = 0; kc < p.kchunks; ++kc)
#pragma unroll
                        for (int bx = 0; bx < 4; ++bx) {
                            ptx::mbar_wait(&empty[stage], phase ^ 1);
                            uint8_t* sa = ring + stage * A_BYTES;
                            const CUtensorMap* mx = (bx & 1) ? &map_x1 : &map_x0;
                            const int jj = 7 * tl.k - (bx < 2 ? 1 : 0);
                            if constexpr (PAIR) {
                                if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * A_BYTES);
                                ptx::tma_load_5d_2sm(mx, &full[stage], sa, 0, jj, tl.r0 - 1, tl.b, kc);
                            } else {
                                ptx::mbar_arrive_expect_tx(&full[stage], A_BYTES);
                                ptx::tma_load_5d(mx, &full[stage], sa, 0, jj, tl.r0 - 1, tl.b, kc);
                            }
                            if (++stage == p.stages) { stage = 0; phase ^= 1; }
                        }
                    continue;
                }
                for (int v = 0; v < 2; ++v) {
                    const int P = v, j0 = 7 * tl.k - v;
                    const int pc = (P + p.parity) & 1;
                    for (int kc = 0; kc < p.kchunks; ++kc) {
#pragma unroll 1
                        for (int s = 0; s < SL::count(); ++s) {
                            const int dc = SL::dc_of(s);
                            const int Pv = (P + dc) & 1;
                            const int jsh = (P + dc - Pv) / 2;
                            const int top = -N + (((dc < 0 ? -dc : dc) + pc) >> 1);
                            ptx::mbar_wait(&empty[stage], phase ^ 1);
                            uint8_t* sa = ring + stage * A_BYTES;
                            ptx::mbar_arrive_expect_tx(&full[stage], A_BYTES);
                            ptx::tma_load_5d(Pv ? &map_x1 : &map_x0, &full[stage], sa, 0, j0 + jsh, tl.r0 + top,
                                             tl.b, kc);
                            if (++stage == p.stages) { stage = 0; phase ^= 1; }
                        }
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && (!PAIR || leader)) {
            const uint64_t a_ring = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
            const uint64_t res_desc = ptx::smem_desc_sw128(ptx::smem_u32(resw), 16, 1024);
            int stage = 0;
            uint32_t phase = 0;
            int slot = 0;
            uint32_t sphase = 0;
            ptx::mbar_wait(bres, 0);
            FpTile tl;
            for (int seq = 0; fp_tile<PAIR>(p, seq, tl); ++seq) {
                ptx::mbar_wait(&tempty[slot], sphase ^ 1);
                ptx::tc_fence_after();
                if (!PAIR && HEX_DBG(p.debug) == 2) {
                    for (int u = 0; u < (N == 1 ? 4 : 2 * SL::count()) * p.kchunks; ++u) {
                        ptx::mbar_wait(&full[stage], phase);
                        ptx::mbar_arrive(&empty[stage]);
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
                    ptx::mbar_arrive(&tfull[slot]);
                    slot ^= 1;
                    if (slot == 0) sphase ^= 1;
                    continue;
                }
                if constexpr (N == 1) {
                    for (int kc = 0; kc < p.kchunks; ++kc)
                        fp_issue_n1<BN, PAIR>(tmem_base + (slot * 2) * BN, tmem_base + (slot * 2 + 1) * BN, a_ring,
                                              res_desc, full, empty, stage, phase, p.stages, A_BYTES >> 4, kc,
                                              p.kchunks, kc == 0 ? 0u : 1u, (uint32_t)(p.parity & 1));
                } else {
                    for (int v = 0; v < 2; ++v) {
                        const uint32_t d = tmem_base + (slot * 2 + v) * BN;
                        for (int kc = 0; kc < p.kchunks; ++kc)
                            issue_stages_from<BN, N, TG, true, false, 0>(d, a_ring, a_ring, res_desc, full, empty,
                                                                         stage, phase, p.stages, A_BYTES >> 4,
                                                                         A_BYTES >> 4, kc, p.kchunks,
                                                                         kc == 0 ? 0u : 1u);
                    }
                }
                if constexpr (PAIR) ptx::mma_commit_2sm(&tfull[slot]);
                else ptx::mma_commit(&tfull[slot]);
                slot ^= 1;
                if (slot == 0) sphase ^= 1;
            }
        }
    } else if (warp < 10) {
        // ---- converter warps: TMEM lane quadrant q (pixels 32 q .. 32 q + 31), view cv
        const int q = warp & 3;
        const int cv = (warp - 2) >> 2;
        const int row = q * 32 + lane;  // tile pixel m = 8 * (tile row) + sub-column
        const int et = threadIdx.x - 64;  // 0..255
        // carried 16-byte group of this thread (et < 128): view kv, carried row kr, sub-column ks, group ki
        const int kv = (et >> 6) & 1, kr = (et >> 5) & 1, ks = (et >> 2) & 7, ki = et & 3;
        const int koff = kv * FP_VIEW + fp_off(kr, ks, ki);
        const int kcar = kv * 1024 + kr * 512 + ks * FP_PIX + ki * 16;
        int soff[4];  // this pixel's 16-byte groups in a region buffer (region rows 2..17)
#pragma unroll
        for (int ii = 0; ii < 4; ++ii) soff[ii] = cv * FP_VIEW + fp_off(2 + (row >> 3), row & 7, ii);
        int slot = 0;
        uint32_t sphase = 0;
        int g = 0;  // chunk counter (buffer g % nreg)
        FpTile tl;
        for (int seq = 0; fp_tile<PAIR>(p, seq, tl); ++seq) {
            const int img_r = tl.r0 + (row >> 3);
            const int jv = 7 * tl.k - cv + (row & 7);  // sub-column of this pixel in view cv
            const bool outside = img_r < 0 || img_r >= p.H || jv < 0 || 2 * jv + cv >= p.W;
            ptx::mbar_wait(&tfull[slot], sphase);
            ptx::tc_fence_after();
            if (!PAIR && HEX_DBG(p.debug) == 1) {
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(&tempty[slot]);
                slot ^= 1;
                if (slot == 0) sphase ^= 1;
                continue;
            }
#pragma unroll 1
            for (int c = 0; c < NCH; ++c, ++g) {
                const int bf = g & (p.nreg - 1);
                if (g >= p.nreg) ptx::named_bar(FP_BAR_EMPTY + bf, 512);  // window warps are done with it
                uint8_t* rb = region + bf * FP_BUF;
                uint32_t vals[32];
                ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (slot * 2 + cv) * BN + c * 32, vals);
                ptx::tmem_ld_wait();
                if (HEX_DBG(p.debug) == 4) {  // timing experiment: converters skip their shared-memory stores
                } else if (outside) {
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii)
                        *reinterpret_cast<uint4*>(rb + soff[ii]) = make_uint4(NEG_INF2, NEG_INF2, NEG_INF2, NEG_INF2);
                } else {
#pragma unroll
                    for (int ii = 0; ii < 4; ++ii) {
                        float f[8];
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) f[kk] = __uint_as_float(vals[8 * ii + kk]);
                        if (p.bias) {  // bias staged in shared memory (broadcast reads)
                            const float4 b0 = *reinterpret_cast<const float4*>(sbias + c * 32 + 8 * ii);
                            const float4 b1 = *reinterpret_cast<const float4*>(sbias + c * 32 + 8 * ii + 4);
                            f[0] += b0.x; f[1] += b0.y; f[2] += b0.z; f[3] += b0.w;
                            f[4] += b1.x; f[5] += b1.y; f[6] += b1.z; f[7] += b1.w;
                        }
                        uint32_t pk[4];
                        if (p.relu) {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) pk[kk] = ptx::pack_bf16x2_relu(f[2 * kk], f[2 * kk + 1]);
                        } else {
#pragma unroll
                            for (int kk = 0; kk < 4; ++kk) {
                                __nv_bfloat162 hv = __floats2bfloat162_rn(f[2 * kk], f[2 * kk + 1]);
                                pk[kk] = *reinterpret_cast<uint32_t*>(&hv);
                            }
                        }
                        *reinterpret_cast<uint4*>(rb + soff[ii]) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                    }
                }
                // rows r0-2, r0-1: carried from the previous tile of the strip (above the image: -inf)
                if (tl.strip && et < 128)
                    *reinterpret_cast<uint4*>(rb + koff) =
                        tl.first ? make_uint4(NEG_INF2, NEG_INF2, NEG_INF2, NEG_INF2)
                                 : *reinterpret_cast<const uint4*>(carry + c * FP_CARRY + kcar);
                if (c + 1 == NCH) {  // TMEM slot fully read: the MMA may refill it
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                        if constexpr (PAIR) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[slot]), 0));
                        else ptx::mbar_arrive(&tempty[slot]);
                    }
                }
                ptx::named_bar_arrive(FP_BAR_FULL + bf, 512);
            }
            slot ^= 1;
            if (slot == 0) sphase ^= 1;
        }
        for (int r = g < p.nreg ? 0 : g - p.nreg; r < g; ++r)  // drain
            ptx::named_bar(FP_BAR_EMPTY + (r & (p.nreg - 1)), 512);
    } else {
        // ---- window warps: one (window, 8-channel group) item per thread and chunk
        const int et = threadIdx.x - 64 - 256;  // 0..255
        const bool relu = p.relu != 0;
        const int pcen = p.parity & 1;  // centre column parity of every window (centres in even columns)
        const int top1 = -1 + ((1 + pcen) >> 1);  // first row offset of the dc = +-1 taps
        const int cg = et & 3, wi = et >> 2;
        const int wc = wi % 7, ws = wi / 7;
        const int kv = (et >> 6) & 1, kr = (et >> 5) & 1, ks = (et >> 2) & 7, ki = et & 3;
        const int soff = kv * FP_VIEW + fp_off(16 + kr, ks, ki);
        const int kcar = kv * 1024 + kr * 512 + ks * FP_PIX + ki * 16;
        int g = 0;
        FpTile tl;
        for (int seq = 0; (PAIR || HEX_DBG(p.debug) != 1) && fp_tile<PAIR>(p, seq, tl); ++seq) {
            const int C = 7 * tl.k + wc;
            const int rho = C & 1;  // centre row of window (R, C): cr = 2R + rho
            // owned centre rows [lo, hi]
            const int lo = tl.strip ? tl.r0 - 1 : tl.r0 + 1;
            const int hi = tl.strip ? (tl.r0 + FT_RB >= p.H ? tl.r0 + 15 : tl.r0 + 14) : tl.r0 + 14;
            const int R = (lo - rho + 3) / 2 - 1 + ws;  // ceil((lo - rho) / 2) + ws, lo - rho >= -2
            const int cr = 2 * R + rho;
            const bool valid = ws < (tl.strip ? 9 : 7) && C < p.Wo && R >= 0 && R < p.Ho && cr <= hi;
            const int lr = cr - tl.r0 + 2;  // region row of the centre
            // canonical taps: 0,1 column 2C-1 (view 1, local sub-column wc); 2,3,4 column 2C (view 0, wc);
            // 5,6 column 2C+1 (view 1, wc + 1)
            const int ol0 = FP_VIEW + fp_off(lr + top1, wc, cg), ol1 = FP_VIEW + fp_off(lr + top1 + 1, wc, cg);
            const int oc0 = fp_off(lr - 1, wc, cg), oc1 = fp_off(lr, wc, cg), oc2 = fp_off(lr + 1, wc, cg);
            const int or0 = FP_VIEW + fp_off(lr + top1, wc + 1, cg);
            const int or1 = FP_VIEW + fp_off(lr + top1 + 1, wc + 1, cg);
            const int64_t obase = (((int64_t)tl.b * p.Ho + R) * p.Wo + C) * p.Cout + cg * 8;
#pragma unroll 1
            for (int c = 0; c < NCH; ++c, ++g) {
                const int bf = g & (p.nreg - 1);
                ptx::named_bar(FP_BAR_FULL + bf, 512);
                const uint8_t* rb = region + bf * FP_BUF;
                if (tl.strip && !tl.last && et < 128)  // rows r0+14, r0+15 carry into the next tile
                    *reinterpret_cast<uint4*>(carry + c * FP_CARRY + kcar) =
                        *reinterpret_cast<const uint4*>(rb + soff);
                if (HEX_DBG(p.debug) == 3) {  // timing experiment: window warps skip their reads / math
                } else if (valid && AVG) {
                    // average over the in-grid taps (A8): fp32 sum in canonical tap order from 0, times
                    // 1/count, RNE -- the operations of the unfused NHWC average pool on the bf16 conv output
                    const int c2 = 2 * C;
                    const bool cl = c2 >= 1, cm = true, crt = c2 + 1 < p.W;
                    const int rs0 = cr + top1, rs1 = cr + top1 + 1;
                    const bool ok[7] = {cl && rs0 >= 0 && rs0 < p.H, cl && rs1 >= 0 && rs1 < p.H,
                                        cm && cr - 1 >= 0, cm, cm && cr + 1 < p.H,
                                        crt && rs0 >= 0 && rs0 < p.H, crt && rs1 >= 0 && rs1 < p.H};
                    const int offs[7] = {ol0, ol1, oc0, oc1, oc2, or0, or1};
                    float sum[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                    int cnt = 0;
#pragma unroll
                    for (int t = 0; t < 7; ++t) {
                        if (!ok[t]) continue;
                        const uint4 q = *reinterpret_cast<const uint4*>(rb + offs[t]);
                        const uint32_t w4[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
                        for (int kk = 0; kk < 4; ++kk) {
                            sum[2 * kk] += __uint_as_float(w4[kk] << 16);
                            sum[2 * kk + 1] += __uint_as_float(w4[kk] & 0xffff0000u);
                        }
                        ++cnt;
                    }
                    const float inv = 1.f / (float)cnt;
                    uint32_t pk[4];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        __nv_bfloat162 h = __floats2bfloat162_rn(sum[2 * kk] * inv, sum[2 * kk + 1] * inv);
                        pk[kk] = *reinterpret_cast<uint32_t*>(&h);
                    }
                    *reinterpret_cast<uint4*>(p.y + obase + c * 32) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                } else if (valid) {
                    uint4 tv[7];
                    tv[0] = *reinterpret_cast<const uint4*>(rb + ol0);
                    tv[1] = *reinterpret_cast<const uint4*>(rb + ol1);
                    tv[2] = *reinterpret_cast<const uint4*>(rb + oc0);
                    tv[3] = *reinterpret_cast<const uint4*>(rb + oc1);
                    tv[4] = *reinterpret_cast<const uint4*>(rb + oc2);
                    tv[5] = *reinterpret_cast<const uint4*>(rb + or0);
                    tv[6] = *reinterpret_cast<const uint4*>(rb + or1);
                    uint32_t best[4], ix[4];
#pragma unroll
                    for (int kk = 0; kk < 4; ++kk) {
                        __nv_bfloat162 mx = *reinterpret_cast<const __nv_bfloat162*>(
                            reinterpret_cast<const uint32_t*>(&tv[0]) + kk);
#pragma unroll
                        for (int t = 1; t < 7; ++t)
                            mx = __hmax2(mx, *reinterpret_cast<const __nv_bfloat162*>(
                                                 reinterpret_cast<const uint32_t*>(&tv[t]) + kk));
                        // first tap equal to the maximum == first strict maximum in canonical order; with
                        // ReLU no value is -0 (cvt.relu gives +0), so the maximum's bits are that tap's bits
                        best[kk] = relu ? *reinterpret_cast<const uint32_t*>(&mx)
                                        : reinterpret_cast<const uint32_t*>(&tv[6])[kk];
                        ix[kk] = 6u * 0x00010001u;
#pragma unroll
                        for (int t = 5; t >= 0; --t) {
                            const uint32_t wv = reinterpret_cast<const uint32_t*>(&tv[t])[kk];
                            const uint32_t mk = __heq2_mask(*reinterpret_cast<const __nv_bfloat162*>(&wv), mx);
                            if (!relu) best[kk] = (wv & mk) | (best[kk] & ~mk);
                            ix[kk] = ((uint32_t)t * 0x00010001u & mk) | (ix[kk] & ~mk);
                        }
                    }
                    const int64_t o = obase + c * 32;
                    *reinterpret_cast<uint4*>(p.y + o) = make_uint4(best[0], best[1], best[2], best[3]);
                    *reinterpret_cast<uint2*>(p.am + o) =
                        make_uint2(__byte_perm(ix[0], ix[1], 0x6420), __byte_perm(ix[2], ix[3], 0x6420));
                }
                ptx::named_bar_arrive(FP_BAR_EMPTY + bf, 512);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) ptx::cluster_sync();  // the peer's smem / TMEM must outlive the leader's last MMA
    if (warp == 1) {
        ptx::tc_fence_after();
        if constexpr (PAIR) ptx::tmem_dealloc_2sm(tmem_base, TMEM_COLS);
        else ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ------------------------------------------------------------------ n = 1 view-pair forward / bwd-data
// The tap-reuse forward above computes one 16 x 8 tile of ONE parity view per work item, reading three
// 18-row boxes (one per kernel column), two of which come from the other view at overlapping
// sub-columns.  Here a work item is the PAIR of tiles (view 0 and view 1) at the same sub-columns
// [j0, j0+8) and rows [r0, r0+16); four 19-row boxes (top row r0 - 1) serve both tiles:
//   box 0 = view 1 at j0-1: view-0 dc = -1 (taps 0,1)
//   box 1 = view 0 at j0:   view-0 dc =  0 (taps 2..4), view-1 dc = -1 (taps 0,1)
//   box 2 = view 1 at j0:   view-0 dc = +1 (taps 5,6),  view-1 dc =  0 (taps 2..4)
//   box 3 = view 0 at j0+1: view-1 dc = +1 (taps 5,6)
// (4 boxes / 76 KB per 2 tiles instead of 6 / 108 KB), each accumulator still summed in the canonical
// column order.  Resident weights, n = 1, Cout = 64 or 128 (C5 layer-2 bwd-data).
struct FvParams {
    int B, H, W, Cin, Cout, parity;
    int rt, jt, pairs, kchunks, stages, relu, has_mask, debug, prefetch;
    const float* bias;
};

template <int BN, bool PAIR>
__device__ __forceinline__ void fv_issue(uint32_t d0, uint32_t d1, uint64_t a_ring, uint64_t res_desc, uint64_t* full,
                                         uint64_t* empty, int& stage, uint32_t& phase, int nstages, uint32_t stage16,
                                         int kc, int kchunks, uint32_t first, uint32_t pc0) {
    constexpr int BROWS = PAIR ? BN / 2 : BN;  // weight rows held per CTA
    const uint64_t o0 = (uint64_t)(pc0 * 64), o1 = (uint64_t)((pc0 ^ 1u) * 64);  // 1024-byte rows
    const int bs = kchunks * BROWS * 8;
    const uint64_t w0 = res_desc + (uint64_t)(kc * (BROWS * 8));  // tap t at w0 + t * bs
#pragma unroll
    for (int bx = 0; bx < 4; ++bx) {
        ptx::mbar_wait(&full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t ad = a_ring + (uint64_t)stage * stage16;
        if (bx == 0) {
            fv_group<BN, 2, PAIR>(d0, ad + o0, w0, bs, first);
        } else if (bx == 1) {
            fv_group<BN, 3, PAIR>(d0, ad, w0 + (uint64_t)(2 * bs), bs, 1u);
            fv_group<BN, 2, PAIR>(d1, ad + o1, w0, bs, first);
        } else if (bx == 2) {
            fv_group<BN, 2, PAIR>(d0, ad + o0, w0 + (uint64_t)(5 * bs), bs, 1u);
            fv_group<BN, 3, PAIR>(d1, ad, w0 + (uint64_t)(2 * bs), bs, 1u);
        } else {
            fv_group<BN, 2, PAIR>(d1, ad + o1, w0 + (uint64_t)(5 * bs), bs, 1u);
        }
        if constexpr (PAIR) ptx::mma_commit_2sm(&empty[stage]);
        else ptx::mma_commit(&empty[stage]);
        if (++stage == nstages) { stage = 0; phase ^= 1; }
    }
}

__device__ __forceinline__ void fv_decode(const FvParams& p, int pr, int* r0, int* j0, int* b) {
    if (pr >= p.pairs) {  // CTA-pair tail: a missing unit loads zero fill and stores nothing (rows >= H)
        *r0 = p.H; *j0 = 0; *b = 0;
        return;
    }
    const int ji = pr % p.jt;
    const int t = pr / p.jt;
    *r0 = (t % p.rt) * FT_RB;
    *j0 = ji * FT_JB;
    *b = t / p.rt;
}

template <int BN, bool PAIR>
__global__ void __launch_bounds__(FT_THREADS, 1)
tc_fwd_vpair_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                    const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_y0,
                    const __grid_constant__ CUtensorMap map_y1, const __grid_constant__ CUtensorMap map_m0,
                    const __grid_constant__ CUtensorMap map_m1, const __grid_constant__ FvParams p) {
    constexpr int A_BYTES = (FT_RB + 3) * FT_JB * 128;  // 19-row box
    constexpr int W_TILE = (PAIR ? BN / 2 : BN) * 128;  // one (tap, chunk) weight tile (this CTA's rows)
    constexpr int TMEM_COLS = 4 * BN;  // 2 slots x 2 views
    constexpr int UNITS = 2 * (BN / 64);  // (view, 64-channel chunk) epilogue units per pair
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const int res_bytes = 7 * p.kchunks * W_TILE;
    uint8_t* resw = base;
    uint8_t* ring = base + res_bytes;
    uint8_t* obuf = ring + p.stages * A_BYTES;
    uint64_t* full = (uint64_t*)(obuf + 2 * FT_OUT);
    uint64_t* empty = full + p.stages;
    uint64_t* tfull = empty + p.stages;
    uint64_t* tempty = tfull + 2;
    uint64_t* mbar = tempty + 2;
    uint64_t* bres = mbar + 2;
    uint32_t* tmem_slot = (uint32_t*)(bres + 1);

    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    const uint32_t rank = PAIR ? ptx::cluster_ctarank() : 0u;
    const bool leader = rank == 0;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) { ptx::mbar_init(&full[s], 1); ptx::mbar_init(&empty[s], 1); }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], (PAIR ? 2 : 1) * FT_EPI / 32);
            ptx::mbar_init(&mbar[a], 1);
        }
        ptx::mbar_init(bres, 1);
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_x0);
        ptx::prefetch_tmap(&map_x1);
        ptx::prefetch_tmap(&map_w);
        ptx::prefetch_tmap(&map_y0);
        ptx::prefetch_tmap(&map_y1);
    }
    if (warp == 1) {
        if constexpr (PAIR) ptx::tmem_alloc_2sm(tmem_slot, TMEM_COLS);
        else ptx::tmem_alloc(tmem_slot, TMEM_COLS);
    }
    ptx::tc_fence_before();
    if constexpr (PAIR) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            if constexpr (PAIR) {  // each CTA holds its half of every weight tile; bytes land on the leader
                if (leader) ptx::mbar_arrive_expect_tx(bres, (uint32_t)(2 * res_bytes));
                for (int t = 0; t < 7; ++t)
                    for (int kc = 0; kc < p.kchunks; ++kc)
                        ptx::tma_load_4d_2sm(&map_w, bres, resw + (t * p.kchunks + kc) * W_TILE, 0,
                                             (int)rank * (BN / 2), kc, t);
            } else {
                ptx::mbar_arrive_expect_tx(bres, (uint32_t)res_bytes);
                for (int t = 0; t < 7; ++t)
                    for (int kc = 0; kc < p.kchunks; ++kc)
                        ptx::tma_load_4d(&map_w, bres, resw + (t * p.kchunks + kc) * W_TILE, 0, 0, kc, t);
            }
            int stage = 0;
            uint32_t phase = 0;
            for (int u = PAIR ? blockIdx.x / 2 : blockIdx.x; u < (PAIR ? (p.pairs + 1) / 2 : p.pairs);
                 u += PAIR ? gridDim.x / 2 : gridDim.x) {
                const int pr = PAIR ? 2 * u + (int)rank : u;
                int r0, j0, b;
                fv_decode(p, pr, &r0, &j0, &b);
                for (int kc = 0; kc < p.kchunks; ++kc)
#pragma unroll
                    for (int bx = 0; bx < 4; ++bx) {
                        ptx::mbar_wait(&empty[stage], phase ^ 1);
                        uint8_t* sa = ring + stage * A_BYTES;
                        const int jj = j0 + (bx == 0 ? -1 : (bx == 3 ? 1 : 0));
                        if constexpr (PAIR) {
                            if (leader) ptx::mbar_arrive_expect_tx(&full[stage], 2 * A_BYTES);
                            ptx::tma_load_5d_2sm((bx & 1) ? &map_x0 : &map_x1, &full[stage], sa, 0, jj, r0 - 1, b, kc);
                        } else {
                            ptx::mbar_arrive_expect_tx(&full[stage], A_BYTES);
                            ptx::tma_load_5d((bx & 1) ? &map_x0 : &map_x1, &full[stage], sa, 0, jj, r0 - 1, b, kc);
                        }
                        if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    }
            }
        }
    } else if (warp == 1) {
        if (lane == 0 && (!PAIR || leader)) {
            const uint64_t a_ring = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
            const uint64_t res_desc = ptx::smem_desc_sw128(ptx::smem_u32(resw), 16, 1024);
            int stage = 0;
            uint32_t phase = 0;
            int slot = 0;
            uint32_t sphase = 0;
            ptx::mbar_wait(bres, 0);
            for (int u = PAIR ? blockIdx.x / 2 : blockIdx.x; u < (PAIR ? (p.pairs + 1) / 2 : p.pairs);
                 u += PAIR ? gridDim.x / 2 : gridDim.x) {
                ptx::mbar_wait(&tempty[slot], sphase ^ 1);
                ptx::tc_fence_after();
                for (int kc = 0; kc < p.kchunks; ++kc)
                    fv_issue<BN, PAIR>(tmem_base + (slot * 2) * BN, tmem_base + (slot * 2 + 1) * BN, a_ring, res_desc,
                                       full, empty, stage, phase, p.stages, A_BYTES >> 4, kc, p.kchunks,
                                       kc == 0 ? 0u : 1u, (uint32_t)(p.parity & 1));
                if constexpr (PAIR) ptx::mma_commit_2sm(&tfull[slot]);
                else ptx::mma_commit(&tfull[slot]);
                slot ^= 1;
                if (slot == 0) sphase ^= 1;
            }
        }
    } else {
        // Epilogue (as in tc_fwd_tr_kernel): warps 2..9, TMEM lane quadrant warp % 4, channel half h.
        // Units (view v, 64-channel chunk ch) of a pair in order; ReLU-backward mask tiles are
        // TMA-loaded one unit ahead, across pairs too.
        const int q = warp & 3;
        const int h = (warp - 2) >> 2;
        const int row = q * 32 + lane;
        const int et = threadIdx.x - 64;
        int slot = 0;
        uint32_t sphase = 0;
        int ob = 0;
        uint32_t mphase0 = 0, mphase1 = 0;
        if (p.has_mask && et == 0 && HEX_DBG(p.debug) != 1 && (int)(PAIR ? blockIdx.x / 2 : blockIdx.x) < (PAIR ? (p.pairs + 1) / 2 : p.pairs)) {
            int r0, j0, b;
            fv_decode(p, PAIR ? (int)(blockIdx.x / 2) * 2 + (int)rank : (int)blockIdx.x, &r0, &j0, &b);
            ptx::mbar_arrive_expect_tx(&mbar[0], FT_OUT);
            ptx::tma_load_4d(&map_m0, &mbar[0], obuf, 0, j0, r0, b);
        }
        for (int wu = PAIR ? blockIdx.x / 2 : blockIdx.x; wu < (PAIR ? (p.pairs + 1) / 2 : p.pairs);
             wu += PAIR ? gridDim.x / 2 : gridDim.x) {
            const int pr = PAIR ? 2 * wu + (int)rank : wu;
            int r0, j0, b;
            fv_decode(p, pr, &r0, &j0, &b);
            ptx::mbar_wait(&tfull[slot], sphase);
            ptx::tc_fence_after();
#pragma unroll 1
            for (int u = 0; u < (HEX_DBG(p.debug) == 1 ? 0 : UNITS); ++u) {
                const int v = u / (BN / 64), ch = u % (BN / 64);
                uint8_t* buf = obuf + ob * FT_OUT;
                const int c0 = ch * 64;
                if (p.has_mask) {
                    ptx::mbar_wait(&mbar[ob], ob ? mphase1 : mphase0);
                    if (ob) mphase1 ^= 1; else mphase0 ^= 1;
                } else {
                    if (et == 0) ptx::bulk_wait_read<1>();
                    ptx::named_bar(1, FT_EPI);
                }
                uint32_t vals[32];
                ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (slot * 2 + v) * BN + c0 + h * 32, vals);
                ptx::tmem_ld_wait();
                uint8_t* rowp = buf + row * 128;
#pragma unroll
                for (int ii = 0; ii < 4; ++ii) {
                    const int i = 4 * h + ii;  // 16-byte unit (8 channels) within the 64-channel chunk
                    uint4* sl = reinterpret_cast<uint4*>(rowp + ((i ^ (row & 7)) << 4));
                    float f[8];
#pragma unroll
                    for (int k = 0; k < 8; ++k) f[k] = __uint_as_float(vals[8 * ii + k]);
                    if (p.bias) {
                        const float4 b0 = __ldg(reinterpret_cast<const float4*>(p.bias + c0 + 8 * i));
                        const float4 b1 = __ldg(reinterpret_cast<const float4*>(p.bias + c0 + 8 * i + 4));
                        f[0] += b0.x; f[1] += b0.y; f[2] += b0.z; f[3] += b0.w;
                        f[4] += b1.x; f[5] += b1.y; f[6] += b1.z; f[7] += b1.w;
                    }
                    if (p.relu && !p.has_mask) {
                        *sl = make_uint4(ptx::pack_bf16x2_relu(f[0], f[1]), ptx::pack_bf16x2_relu(f[2], f[3]),
                                         ptx::pack_bf16x2_relu(f[4], f[5]), ptx::pack_bf16x2_relu(f[6], f[7]));
                        continue;
                    }
                    if (p.relu) {
#pragma unroll
                        for (int k = 0; k < 8; ++k) f[k] = fmaxf(f[k], 0.f);
                    }
                    if (p.has_mask) {
                        const uint4 m4 = *sl;
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
                        __nv_bfloat162 hv = __floats2bfloat162_rn(f[2 * k], f[2 * k + 1]);
                        pk[k] = *reinterpret_cast<uint32_t*>(&hv);
                    }
                    *sl = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
                ptx::fence_proxy_async();
                ptx::named_bar(1, FT_EPI);
                if (et == 0) {
                    ptx::tma_store_4d(v ? &map_y1 : &map_y0, buf, c0, j0, r0, b);
                    ptx::bulk_commit();
                    if (p.has_mask) {  // the next unit's mask tile
                        int nr = r0, nj = j0, nb = b, nu = u + 1;
                        bool more = true;
                        if (nu == UNITS) {
                            nu = 0;
                            const int nw = wu + (PAIR ? gridDim.x / 2 : gridDim.x);
                            more = nw < (PAIR ? (p.pairs + 1) / 2 : p.pairs);
                            if (more) fv_decode(p, PAIR ? 2 * nw + (int)rank : nw, &nr, &nj, &nb);
                        }
                        if (more) {
                            const int nv = nu / (BN / 64), nch = nu % (BN / 64);
                            ptx::bulk_wait_read<1>();
                            ptx::mbar_arrive_expect_tx(&mbar[ob ^ 1], FT_OUT);
                            ptx::tma_load_4d(nv ? &map_m1 : &map_m0, &mbar[ob ^ 1], obuf + (ob ^ 1) * FT_OUT, nch * 64,
                                             nj, nr, nb);
                        }
                    }
                }
                ob ^= 1;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (PAIR) ptx::mbar_arrive_cluster(ptx::mapa(ptx::smem_u32(&tempty[slot]), 0));
                else ptx::mbar_arrive(&tempty[slot]);
            }
            slot ^= 1;
            if (slot == 0) sphase ^= 1;
        }
        if (et == 0) ptx::bulk_wait<0>();
    }
    ptx::tc_fence_before();
    __syncthreads();
    if constexpr (PAIR) ptx::cluster_sync();  // the peer's smem / TMEM must outlive the leader's last MMA
    if (warp == 1) {
        ptx::tc_fence_after();
        if constexpr (PAIR) ptx::tmem_dealloc_2sm(tmem_base, TMEM_COLS);
        else ptx::tmem_dealloc(tmem_base, TMEM_COLS);
    }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 ft_encode() {
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

// parity view P, sub-columns before rows: dims {64, Wp, H, B, C/64}, box {64, 8, rows, 1, 1}
static bool ft_view5(CUtensorMap* m, const void* base, int B, int H, int W, int C, int P, int rows) {
    auto enc = ft_encode();
    const int Wp = (W - P + 1) / 2;
    if (!enc || Wp < 1 || C % 64) return false;
    cuuint64_t dims[5] = {64, (cuuint64_t)Wp, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)(C / 64)};
    cuuint64_t strides[4] = {(cuuint64_t)2 * C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, 128};
    cuuint32_t box[5] = {64, (cuuint32_t)FT_JB, (cuuint32_t)rows, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, (void*)((const char*)base + (size_t)P * C * 2), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// output / mask tiles: dims {C, Wp, H, B}, box {64, 8, 16, 1}
static bool ft_view4(CUtensorMap* m, const void* base, int B, int H, int W, int C, int P) {
    auto enc = ft_encode();
    const int Wp = (W - P + 1) / 2;
    if (!enc || Wp < 1) return false;
    cuuint64_t dims[4] = {(cuuint64_t)C, (cuuint64_t)Wp, (cuuint64_t)H, (cuuint64_t)B};
    cuuint64_t strides[3] = {(cuuint64_t)2 * C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)FT_JB, (cuuint32_t)FT_RB, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)((const char*)base + (size_t)P * C * 2), dims, strides,
               box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// packed weights [T][Cout][Cin]: dims {64, Cout, Cin/64, T}, box {64, BN, 1, 1}
static bool ft_wmap(CUtensorMap* m, const void* base, int T, int Cout, int Cin, int BN) {
    auto enc = ft_encode();
    if (!enc) return false;
    cuuint64_t dims[4] = {64, (cuuint64_t)Cout, (cuuint64_t)(Cin / 64), (cuuint64_t)T};
    cuuint64_t strides[3] = {(cuuint64_t)Cin * 2, 128, (cuuint64_t)Cout * Cin * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)BN, 1, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, (void*)base, dims, strides, box, es,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

namespace {
struct FtPlan {
    int BN, res, pair, tg, stages, smem;
    bool ok;
};

// taps per stage: the whole column with resident weights; with streamed weight halves (CTA pairs) as
// many as keep >= 3 stages in shared memory
constexpr int ft_tg(bool res, int n, int BN) { return res ? 2 * n + 1 : (BN == 256 ? 2 : (n == 1 ? 3 : 5)); }

FtPlan ft_plan(const Geom& g, int Cin, int Cout, bool allow_res = true) {
    FtPlan pl{};
    if (Cin % 64) return pl;
    const int A = (FT_RB + 2 * g.n) * FT_JB * 128;
    const int fixed = 2 * FT_OUT + 1024 + 512;
    // 1) resident weights: one Cout tile (Cout = 64 or 128), one CTA per tile.  (A CTA-pair variant holding
    //    half of the weights per CTA measured slower on C5 layer 2, fwd 382 vs 230 us, and was removed.)
    if (allow_res && (Cout == 64 || Cout == 128) && !sw_on("HEXCONV_FWD_TR_NORES")) {
        const int res_bytes = g.T * (Cin / 64) * Cout * 128;
        if (res_bytes + fixed + 4 * A <= FT_SMEM_MAX) {
            pl.BN = Cout;
            pl.res = 1;
            pl.tg = ft_tg(true, g.n, Cout);
            pl.stages = (FT_SMEM_MAX - fixed - res_bytes) / A;
            if (pl.stages > 8) pl.stages = 8;
            pl.smem = res_bytes + pl.stages * A + fixed;
            pl.ok = true;
            return pl;
        }
    }
    // 2) CTA pairs (M = 256) with streamed weights, each CTA loading half of every weight tile
    pl.BN = Cout % 256 == 0 ? 256 : (Cout % 128 == 0 ? 128 : (Cout % 64 == 0 ? 64 : 0));
    if (!pl.BN || sw_on("HEXCONV_NO_FWD_TR_PAIR")) return pl;
    pl.pair = 1;
    pl.tg = ft_tg(false, g.n, pl.BN);
    const int st = A + pl.tg * (pl.BN / 2) * 128;
    pl.stages = (FT_SMEM_MAX - fixed) / st;
    if (pl.stages > 6) pl.stages = 6;
    if (pl.stages < 2) return pl;
    pl.smem = pl.stages * st + fixed;
    pl.ok = true;
    return pl;
}
}  // namespace

// Taken for stride-1 bf16 NHWC layers whose 16 x 8 tiles fill >= 85% of both views (n = 1, 2), with
// resident weights or as CTA pairs; HEXCONV_NO_FWD_TR disables it.
bool tc_fwd_tr_supported(const Geom& g, int Cin, int Cout) {
    if (sw_on("HEXCONV_NO_FWD_TR")) return false;
    if (g.s != 1 || (g.n != 1 && g.n != 2) || g.W < 2 || g.B > 65535) return false;
    const double fill_c = (double)((g.W + 1) / 2) / (ceil_div((g.W + 1) / 2, FT_JB) * FT_JB);
    const double fill_r = (double)g.H / (ceil_div(g.H, FT_RB) * FT_RB);
    if (fill_c * fill_r < 0.85) return false;
    const FtPlan pl = ft_plan(g, Cin, Cout);
    if (!pl.ok) return false;
    return ft_encode() != nullptr;
}

template <int BN, int N, bool RES, bool PAIR>
static hex_status_t launch_ft(const CUtensorMap* maps, const FtParams& p, int smem, cudaStream_t st) {
    constexpr int TG = ft_tg(RES, N, BN);
    auto kern = tc_fwd_tr_kernel<BN, N, TG, RES, PAIR>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return HEX_ERR_CUDA;
    if constexpr (PAIR) {
        const int pairs = p.pair_tiles < num_sms() / 2 ? p.pair_tiles : num_sms() / 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * pairs);
        cfg.blockDim = dim3(FT_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], p) !=
            cudaSuccess)
            return HEX_ERR_CUDA;
    } else {
        const int grid = p.total_tiles < num_sms() ? p.total_tiles : num_sms();
        kern<<<grid, FT_THREADS, smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], p);
    }
    count_launch();
    return last_launch_status();
}

// view-pair plan: n = 1, resident weights, Cout 64 / 128; returns stages (0 = not eligible).  *pair is
// always false: the CTA-pair variant (M = 256 per MMA) measured no faster (291 vs 289 us) and is not built.
static int fv_stages(const Geom& g, int Cin, int Cout, int* smem, bool* pair) {
    if (g.n != 1 || g.s != 1 || Cin % 64 || (Cout != 64 && Cout != 128) || sw_on("HEXCONV_NO_FWD_VPAIR")) return 0;
    *pair = false;
    const int A = (FT_RB + 3) * FT_JB * 128;
    const int res_bytes = 7 * (Cin / 64) * (*pair ? Cout / 2 : Cout) * 128;
    const int fixed = 2 * FT_OUT + 1024 + 512;
    int stages = (FT_SMEM_MAX - fixed - res_bytes) / A;
    if (stages > 8) stages = 8;
    if (stages < 3) return 0;
    *smem = res_bytes + stages * A + fixed;
    return stages;
}

template <int BN, bool PAIR>
static hex_status_t launch_fv(const CUtensorMap* maps, const FvParams& p, int smem, cudaStream_t st) {
    auto kern = tc_fwd_vpair_kernel<BN, PAIR>;
    if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
        return HEX_ERR_CUDA;
    if constexpr (PAIR) {
        const int units = (p.pairs + 1) / 2;
        const int clusters = units < num_sms() / 2 ? units : num_sms() / 2;
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(2 * clusters);
        cfg.blockDim = dim3(FT_THREADS);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeClusterDimension;
        attr[0].val.clusterDim.x = 2;
        attr[0].val.clusterDim.y = 1;
        attr[0].val.clusterDim.z = 1;
        cfg.attrs = attr;
        cfg.numAttrs = 1;
        if (cudaLaunchKernelEx(&cfg, kern, maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], p) !=
            cudaSuccess)
            return HEX_ERR_CUDA;
    } else {
        const int grid = p.pairs < num_sms() ? p.pairs : num_sms();
        kern<<<grid, FT_THREADS, smem, st>>>(maps[0], maps[1], maps[2], maps[3], maps[4], maps[5], maps[6], p);
    }
    count_launch();
    return last_launch_status();
}

static hex_status_t tc_fwd_vpair(const TcConvArgs& a, int stages, int smem, bool pair, cudaStream_t st) {
    const Geom& g = a.g;
    FvParams p{};
    p.B = g.B; p.H = g.H; p.W = g.W; p.Cin = a.Cin; p.Cout = a.Cout; p.parity = g.parity;
    p.rt = ceil_div(g.H, FT_RB);
    p.jt = ceil_div((g.W + 1) / 2, FT_JB);  // view 0 has the most sub-columns
    p.pairs = p.rt * p.jt * g.B;
    p.kchunks = a.Cin / 64;
    p.stages = stages;
    p.relu = a.relu;
    p.has_mask = a.relu_y != nullptr;
    p.debug = 0;
    p.prefetch = 0;
    p.bias = a.bias;
    CUtensorMap maps[7];
    if (!ft_view5(&maps[0], a.x, g.B, g.H, g.W, a.Cin, 0, FT_RB + 3)) return HEX_ERR_CUDA;
    if (!ft_view5(&maps[1], a.x, g.B, g.H, g.W, a.Cin, 1, FT_RB + 3)) return HEX_ERR_CUDA;
    if (!ft_wmap(&maps[2], a.wpack, g.T, a.Cout, a.Cin, pair ? a.Cout / 2 : a.Cout)) return HEX_ERR_CUDA;
    if (!ft_view4(&maps[3], a.y, g.B, g.H, g.W, a.Cout, 0)) return HEX_ERR_CUDA;
    if (!ft_view4(&maps[4], a.y, g.B, g.H, g.W, a.Cout, 1)) return HEX_ERR_CUDA;
    if (a.relu_y) {
        if (!ft_view4(&maps[5], a.relu_y, g.B, g.H, g.W, a.Cout, 0)) return HEX_ERR_CUDA;
        if (!ft_view4(&maps[6], a.relu_y, g.B, g.H, g.W, a.Cout, 1)) return HEX_ERR_CUDA;
    } else {
        maps[5] = maps[3];
        maps[6] = maps[4];
    }
    return a.Cout == 128 ? launch_fv<128, false>(maps, p, smem, st) : launch_fv<64, false>(maps, p, smem, st);
}

hex_status_t tc_fwd_tr(const TcConvArgs& a, cudaStream_t st) {
    const Geom& g = a.g;
    {
        int smem = 0;
        bool pair = false;
        const int stages = fv_stages(g, a.Cin, a.Cout, &smem, &pair);
        if (stages) return tc_fwd_vpair(a, stages, smem, pair, st);
    }
    const FtPlan pl = ft_plan(g, a.Cin, a.Cout);
    if (!pl.ok) return HEX_ERR_UNSUPPORTED;
    FtParams p{};
    p.B = g.B; p.H = g.H; p.W = g.W; p.Cin = a.Cin; p.Cout = a.Cout; p.T = g.T; p.parity = g.parity;
    p.rt = ceil_div(g.H, FT_RB);
    p.jt0 = ceil_div((g.W + 1) / 2, FT_JB);
    p.jt1 = ceil_div(g.W / 2, FT_JB);
    p.tiles0 = p.rt * p.jt0 * g.B;
    p.mtiles = p.tiles0 + p.rt * p.jt1 * g.B;
    p.n_tiles = a.Cout / pl.BN;
    p.total_tiles = p.mtiles * p.n_tiles;
    p.pair_tiles = ceil_div(p.mtiles, 2) * p.n_tiles;
    p.kchunks = a.Cin / 64;
    p.stages = pl.stages;
    p.relu = a.relu;
    p.has_mask = a.relu_y != nullptr;
    p.debug = debug_mode("HEXCONV_FT_DEBUG");
    p.kd = p.D = p.Do = p.sd = 1;
    p.pd = 0;
    p.bias = a.bias;
    CUtensorMap maps[7];
    if (!ft_view5(&maps[0], a.x, g.B, g.H, g.W, a.Cin, 0, FT_RB + 2 * g.n)) return HEX_ERR_CUDA;
    if (!ft_view5(&maps[1], a.x, g.B, g.H, g.W, a.Cin, 1, FT_RB + 2 * g.n)) return HEX_ERR_CUDA;
    if (!ft_wmap(&maps[2], a.wpack, g.T, a.Cout, a.Cin, pl.pair ? pl.BN / 2 : pl.BN)) return HEX_ERR_CUDA;
    if (!ft_view4(&maps[3], a.y, g.B, g.H, g.W, a.Cout, 0)) return HEX_ERR_CUDA;
    if (!ft_view4(&maps[4], a.y, g.B, g.H, g.W, a.Cout, 1)) return HEX_ERR_CUDA;
    if (a.relu_y) {
        if (!ft_view4(&maps[5], a.relu_y, g.B, g.H, g.W, a.Cout, 0)) return HEX_ERR_CUDA;
        if (!ft_view4(&maps[6], a.relu_y, g.B, g.H, g.W, a.Cout, 1)) return HEX_ERR_CUDA;
    } else {
        maps[5] = maps[3];
        maps[6] = maps[4];
    }
    if (pl.res) {
        if (pl.BN == 128) return g.n == 1 ? launch_ft<128, 1, true, false>(maps, p, pl.smem, st)
                                          : launch_ft<128, 2, true, false>(maps, p, pl.smem, st);
        return g.n == 1 ? launch_ft<64, 1, true, false>(maps, p, pl.smem, st)
                        : launch_ft<64, 2, true, false>(maps, p, pl.smem, st);
    }
    if (pl.BN == 256) return g.n == 1 ? launch_ft<256, 1, false, true>(maps, p, pl.smem, st)
                                      : launch_ft<256, 2, false, true>(maps, p, pl.smem, st);
    if (pl.BN == 128) return g.n == 1 ? launch_ft<128, 1, false, true>(maps, p, pl.smem, st)
                                      : launch_ft<128, 2, false, true>(maps, p, pl.smem, st);
    return g.n == 1 ? launch_ft<64, 1, false, true>(maps, p, pl.smem, st)
                    : launch_ft<64, 2, false, true>(maps, p, pl.smem, st);
}

// ------------------------------------------------------------------ 3-D convolution
// a.g: per-slice 2-D geometry with g.B = number of VOLUMES; x bf16 NDHWC [B][D][H][W][Cin], y NDHWC
// [B][Do][Ho][Wo][Cout] (s = 1), a.wpack bf16 [kd*T][Cout][Cin] (depth-major taps).  The depth taps run
// inside the K loop of the streamed CTA-pair tap-reuse kernel (no unfold copy).
bool tc_conv3d_supported(const Geom& g, int Cin, int Cout, int Do) {
    if (sw_on("HEXCONV_NO_CONV3D_TC")) return false;
    Geom go = g;
    go.B = g.B * Do;
    if (go.B > 65535 || !tc_fwd_tr_supported(go, Cin, Cout)) return false;
    return ft_plan(go, Cin, Cout, false).ok;
}

hex_status_t tc_conv3d_fwd(const TcConvArgs& a, int D, int Do, int sd, int kd, cudaStream_t st) {
    Geom go = a.g;
    go.B = a.g.B * Do;  // output images
    const FtPlan pl = ft_plan(go, a.Cin, a.Cout, false);
    if (!pl.ok || !pl.pair || pl.res) return HEX_ERR_UNSUPPORTED;
    FtParams p{};
    p.B = go.B; p.H = go.H; p.W = go.W; p.Cin = a.Cin; p.Cout = a.Cout; p.T = go.T; p.parity = go.parity;
    p.rt = ceil_div(go.H, FT_RB);
    p.jt0 = ceil_div((go.W + 1) / 2, FT_JB);
    p.jt1 = ceil_div(go.W / 2, FT_JB);
    p.tiles0 = p.rt * p.jt0 * go.B;
    p.mtiles = p.tiles0 + p.rt * p.jt1 * go.B;
    p.n_tiles = a.Cout / pl.BN;
    p.total_tiles = p.mtiles * p.n_tiles;
    p.pair_tiles = ceil_div(p.mtiles, 2) * p.n_tiles;
    p.kchunks = a.Cin / 64;
    p.stages = pl.stages;
    p.relu = a.relu;
    p.has_mask = a.relu_y != nullptr;
    p.debug = 0;
    p.kd = kd; p.D = D; p.Do = Do; p.sd = sd; p.pd = (kd - 1) / 2;
    p.bias = a.bias;
    const int Bin = a.g.B * D;  // input images
    CUtensorMap maps[7];
    if (!ft_view5(&maps[0], a.x, Bin, go.H, go.W, a.Cin, 0, FT_RB + 2 * go.n)) return HEX_ERR_CUDA;
    if (!ft_view5(&maps[1], a.x, Bin, go.H, go.W, a.Cin, 1, FT_RB + 2 * go.n)) return HEX_ERR_CUDA;
    if (!ft_wmap(&maps[2], a.wpack, kd * go.T, a.Cout, a.Cin, pl.BN / 2)) return HEX_ERR_CUDA;
    if (!ft_view4(&maps[3], a.y, go.B, go.H, go.W, a.Cout, 0)) return HEX_ERR_CUDA;
    if (!ft_view4(&maps[4], a.y, go.B, go.H, go.W, a.Cout, 1)) return HEX_ERR_CUDA;
    if (a.relu_y) {
        if (!ft_view4(&maps[5], a.relu_y, go.B, go.H, go.W, a.Cout, 0)) return HEX_ERR_CUDA;
        if (!ft_view4(&maps[6], a.relu_y, go.B, go.H, go.W, a.Cout, 1)) return HEX_ERR_CUDA;
    } else {
        maps[5] = maps[3];
        maps[6] = maps[4];
    }
    if (pl.BN == 256) return go.n == 1 ? launch_ft<256, 1, false, true>(maps, p, pl.smem, st)
                                       : launch_ft<256, 2, false, true>(maps, p, pl.smem, st);
    if (pl.BN == 128) return go.n == 1 ? launch_ft<128, 1, false, true>(maps, p, pl.smem, st)
                                       : launch_ft<128, 2, false, true>(maps, p, pl.smem, st);
    return go.n == 1 ? launch_ft<64, 1, false, true>(maps, p, pl.smem, st)
                     : launch_ft<64, 2, false, true>(maps, p, pl.smem, st);
}

// ------------------------------------------------------------------ fused conv + max pool host side
namespace {
struct FpPlan {
    int stages, smem, nr, nc, Ho, Wo, nreg;
    bool ok, pair;
};
// pair is always false: the CTA-pair variant (M = 256 MMAs) measured no faster (265.6 vs 263.6 us) and is
// not built
FpPlan fp_plan(const Geom& g, int Cin, int Cout) {
    FpPlan pl{};
    pl.pair = false;
    if (g.s != 1 || (g.n != 1 && g.n != 2) || Cin % 64 || (Cout != 64 && Cout != 128) || g.W < 2) return pl;
    int po;
    if (!out_shape(g.H, g.W, 2, g.parity, &pl.Ho, &pl.Wo, &po)) return pl;
    const int A = (FT_RB + 2 * g.n + (g.n == 1 ? 1 : 0)) * FT_JB * 128;
    const int res_bytes = g.T * (Cin / 64) * (pl.pair ? Cout / 2 : Cout) * 128;
    // 4 region buffers when 3 ring stages still fit next to them (HEXCONV_FP_NREG=2 forces 2)
    for (pl.nreg = sw_int("HEXCONV_FP_NREG", 4) == 2 ? 2 : 4; pl.nreg >= 2; pl.nreg /= 2) {
        const int fixed = pl.nreg * FP_BUF + (Cout / 32) * FP_CARRY + Cout * 4 + 1024 + 512;
        pl.stages = (FT_SMEM_MAX - fixed - res_bytes) / A;
        if (pl.stages >= 3) break;
    }
    if (pl.stages > 8) pl.stages = 8;
    if (pl.nreg < 2 || pl.stages < 3) return pl;
    const int fixed = pl.nreg * FP_BUF + (Cout / 32) * FP_CARRY + Cout * 4 + 1024 + 512;
    pl.smem = res_bytes + pl.stages * A + fixed;
    const int cr_max = 2 * (pl.Ho - 1) + 1;
    pl.nr = (cr_max + 1 + 13) / 14;
    pl.nc = (pl.Wo + 6) / 7;
    pl.ok = true;
    return pl;
}
}  // namespace

bool tc_conv_pool_supported(const Geom& g, int Cin, int Cout, int mode) {
    if (sw_on("HEXCONV_NO_FUSED_POOL") || !ft_encode()) return false;
    if (mode != HEX_POOL_MAX && mode != HEX_POOL_AVG) return false;
    return fp_plan(g, Cin, Cout).ok;
}

hex_status_t tc_conv_pool(const TcConvArgs& a, int mode, void* y_pool, uint8_t* argmax, cudaStream_t st) {
    const Geom& g = a.g;
    const FpPlan pl = fp_plan(g, a.Cin, a.Cout);
    if (!pl.ok || (mode != HEX_POOL_MAX && mode != HEX_POOL_AVG)) return HEX_ERR_UNSUPPORTED;
    FpParams p{};
    p.B = g.B; p.H = g.H; p.W = g.W; p.Cin = a.Cin; p.Cout = a.Cout; p.T = g.T; p.parity = g.parity;
    p.Ho = pl.Ho; p.Wo = pl.Wo; p.nr = pl.nr; p.nc = pl.nc;
    p.kchunks = a.Cin / 64; p.stages = pl.stages; p.relu = a.relu; p.bias = a.bias; p.nreg = pl.nreg;
    p.y = (uint16_t*)y_pool; p.am = argmax;
    // whole rounds of strips (one per CTA per round), the remaining strips as independent regions
    const int strips = g.B * pl.nc;
    p.ntr = (g.H + FT_RB - 1) / FT_RB;
    const int sms = num_sms();
    const bool strip_mode = !sw_on("HEXCONV_FUSED_POOL_REGIONS");
    p.debug = debug_mode("HEXCONV_FP_DEBUG");
    int grid = pl.pair ? sms & ~1 : sms;
    p.full_rounds = strip_mode ? strips / grid : 0;
    p.left_regions = (strips - p.full_rounds * grid) * pl.nr;
    if (p.full_rounds == 0 && p.left_regions < grid) grid = pl.pair ? (p.left_regions + 1) & ~1 : p.left_regions;
    CUtensorMap mx0, mx1, mw;
    const int box_rows = FT_RB + 2 * g.n + (g.n == 1 ? 1 : 0);  // n = 1: 19-row boxes shared by both views
    if (!ft_view5(&mx0, a.x, g.B, g.H, g.W, a.Cin, 0, box_rows)) return HEX_ERR_CUDA;
    if (!ft_view5(&mx1, a.x, g.B, g.H, g.W, a.Cin, 1, box_rows)) return HEX_ERR_CUDA;
    if (!ft_wmap(&mw, a.wpack, g.T, a.Cout, a.Cin, pl.pair ? a.Cout / 2 : a.Cout)) return HEX_ERR_CUDA;
#define HEX_FP(BN_, N_, PAIR_)                                                                                \
    {                                                                                                         \
        auto kern = mode == HEX_POOL_AVG ? tc_conv_maxpool_kernel<BN_, N_, PAIR_, true>                      \
                                         : tc_conv_maxpool_kernel<BN_, N_, PAIR_, false>;                     \
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, pl.smem) != cudaSuccess) \
            return HEX_ERR_CUDA;                                                                              \
        if (PAIR_) {                                                                                          \
            cudaLaunchConfig_t cfg{};                                                                         \
            cfg.gridDim = dim3(grid);                                                                         \
            cfg.blockDim = dim3(FP_THREADS);                                                                  \
            cfg.dynamicSmemBytes = pl.smem;                                                                   \
            cfg.stream = st;                                                                                  \
            cudaLaunchAttribute attr[1];                                                                      \
            attr[0].id = cudaLaunchAttributeClusterDimension;                                                 \
            attr[0].val.clusterDim.x = 2;                                                                     \
            attr[0].val.clusterDim.y = 1;                                                                     \
            attr[0].val.clusterDim.z = 1;                                                                     \
            cfg.attrs = attr;                                                                                 \
            cfg.numAttrs = 1;                                                                                 \
            if (cudaLaunchKernelEx(&cfg, kern, mx0, mx1, mw, p) != cudaSuccess) return HEX_ERR_CUDA;          \
        } else {                                                                                              \
            kern<<<grid, FP_THREADS, pl.smem, st>>>(mx0, mx1, mw, p);                                         \
        }                                                                                                     \
    }
    if (a.Cout == 128) {
        if (g.n == 1) {
            HEX_FP(128, 1, false)
        } else HEX_FP(128, 2, false)
    } else {
        if (g.n == 1) {
            HEX_FP(64, 1, false)
        } else HEX_FP(64, 2, false)
    }
#undef HEX_FP
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
