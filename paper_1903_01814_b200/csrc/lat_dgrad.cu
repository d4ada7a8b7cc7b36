// lat_dgrad.cu -- strided (s > 1) hexagonal convolution backward-data on the tcgen05 tensor cores, bf16 NHWC,
// by PHASE CLASSES ("TC path for s > 1 (phase GEMMs)"): no upsampled copy of dy and only the
// taps that reach a lattice centre are multiplied.
//
//   dx[b][p][ci] = sum_{t, co} W[co][ci][T-1-t] * dy[b][lattice(q)][co]   over the taps t whose neighbour
//                  q = p + off_t(p) is a centre of the stride-s lattice   (the
//                  adjoint of the strided forward: the stride-1 adjoint (pin P18) of dy scattered onto the
//                  full grid (pin P10), where every non-centre neighbour contributes 0)
//
// Output pixels p = (r, c) fall into 2 s^2 classes (r mod s, c mod 2s); within a class the set of taps whose
// neighbour is a lattice centre is the same for every pixel (the centre test depends on q's column mod s, on
// rho(C) -- period 2 in C -- and on q's row mod s), so each class is a dense GEMM over its own K list:
//   M = 128 output pixels of one class (flattened b, i, j of the class grid), N = an input-channel tile
//   (64 or 128), K = (lattice tap, 16-channel chunk of dy).  s^2 times fewer MMAs than the upsampled route.
//   * A is built in TENSOR MEMORY by builder warps (one thread per output pixel = per TMEM lane): per K-step
//     the 16 dy channels of the pixel's lattice neighbour are 32 contiguous bytes (NHWC: two 16-byte loads),
//     written with tcgen05.st; the MMA reads A from TMEM ([a_tmem] operand).  An off-grid neighbour (an
//     edge pixel) reads zeros.
//   * B (the K-step's weight block: N-tile rows x 16 K values, K-major SWIZZLE_32B, packed once per call by
//     lat_pack_kernel in the K-step order of the full (tap, chunk) list) is streamed into a shared-memory
//     ring by a producer warp with bulk copies (the whole weight set would not stay resident).
//   * Warp roles: 4 epilogue warps (one per TMEM lane quadrant: TMEM -> registers -> ReLU-backward mask ->
//     bf16 -> 16-byte NHWC stores), 16 builder warps in 4
//     groups taking 4-K-step stages round-robin (with Cout % 64 == 0 a stage is one 128-byte dy line per
//     pixel, loaded cooperatively), 1 MMA-issuing warp, 1 B producer warp; two TMEM accumulators (the
//     epilogue of tile i overlaps the MMAs of tile i+1).
// Deterministic: every output element is one MMA chain in fixed K order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hexconv {
namespace {

constexpr int LD_KPS = 4;       // K-steps per stage
constexpr int LD_STAGES = 8;    // A stages (TMEM) = B stages (smem), a multiple of the builder groups
constexpr int LD_GROUPS = 4;
constexpr int LD_EPI_WARPS = 4;
constexpr int LD_BLD_WARPS = 4 * LD_GROUPS;
constexpr int LD_MMA_WARP = LD_EPI_WARPS + LD_BLD_WARPS;
constexpr int LD_BW_WARP = LD_MMA_WARP + 1;  // B producer
constexpr int LD_THREADS = (LD_BW_WARP + 1) * 32;
constexpr int LD_MAXT = 37;      // n <= 3
constexpr int LD_MAXCLS = 18;    // 2 s^2, s <= 3
constexpr int LD_MAXKL = 4096;   // K-step list entries over all classes
constexpr int LD_SMEM_MAX = 220 * 1024;

struct LdClass {
    int cr, ccl;        // r mod s, c mod 2s
    int nr, nc;         // class rows / columns per image
    int tile0, k0, kn;  // first tile (per N tile), first K-list entry, K-steps
};

struct LdParams {
    const uint16_t* dy;      // [B][Ho][Wo][Cout] bf16 (the lattice grid)
    const uint16_t* relu_y;  // [B][H][W][Cin] mask source or null
    uint16_t* dx;            // [B][H][W][Cin]
    const uint8_t* wpack;    // [n tile][K-step (t, c16)][NT rows x 32 B] SW32 blocks
    int B, H, W, Ho, Wo, Cin, Cout, s, parity, T, kc16, ksteps_all, ntiles, mtiles, tiles;
    int8_t dc[LD_MAXT], dr0[LD_MAXT], dr1[LD_MAXT];
    int ncls;
    LdClass cls[LD_MAXCLS];
    uint16_t klist[LD_MAXKL];  // per class: tap | chunk << 8
};

__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__device__ __forceinline__ void mma_bf16_ts_elect(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            ptx::smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t* v) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ptx::smem_u32(dst)),
                 "l"((uint64_t)src), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}

template <int NT>
__global__ void __launch_bounds__(LD_THREADS, 1) lat_dgrad_kernel(const __grid_constant__ LdParams p) {
    constexpr int ACC_COLS = 2 * NT;
    constexpr int STAGE_COLS = 8 * LD_KPS;  // 16 bf16 K values = 8 columns per K-step
    constexpr int TMEM_COLS = (ACC_COLS + LD_STAGES * STAGE_COLS) <= 256 ? 256 : 512;
    constexpr uint32_t KBLK = NT * 32;      // one K-step's weight block
    constexpr uint32_t BSTAGE = LD_KPS * KBLK;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* bring = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // B ring
    // [B ring][builder staging tiles: 16 warps x 32 rows x 128 B][barriers][tables]
    uint64_t* full = reinterpret_cast<uint64_t*>(bring + LD_STAGES * BSTAGE + LD_BLD_WARPS * 4096);
    uint64_t* empty = full + LD_STAGES;                                          // A + B stage consumed
    uint64_t* bfull = empty + LD_STAGES;                                         // B stage landed
    uint64_t* tfull = bfull + LD_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    uint32_t* ktab = tslot + 4;  // per K-list entry: dc | dr0 << 8 | dr1 << 16 | chunk << 24
    const int nkl = p.cls[p.ncls - 1].k0 + p.cls[p.ncls - 1].kn;
    uint16_t* wtab = reinterpret_cast<uint16_t*>(ktab + nkl);  // its weight block t * kc16 + chunk
    for (int i = threadIdx.x; i < nkl; i += blockDim.x) {
        const int t = p.klist[i] & 0xFF, c16 = p.klist[i] >> 8;
        ktab[i] = (uint32_t)(uint8_t)p.dc[t] | ((uint32_t)(uint8_t)p.dr0[t] << 8) |
                  ((uint32_t)(uint8_t)p.dr1[t] << 16) | ((uint32_t)c16 << 24);
        wtab[i] = (uint16_t)(t * p.kc16 + c16);
    }
    // tile = (n tile, class tile): n tile major so the class tiles of one n tile share its weights in L2
    auto tile_class = [&](int mt) {
        int c = 0;
        while (c + 1 < p.ncls && mt >= p.cls[c + 1].tile0) ++c;
        return c;
    };
    auto tile_stages = [&](int tile) {
        const LdClass& cl = p.cls[tile_class(tile % p.mtiles)];
        return (cl.kn + LD_KPS - 1) / LD_KPS;
    };
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == LD_MMA_WARP && lane == 0) {
        for (int s = 0; s < LD_STAGES; ++s) {
            ptx::mbar_init(&full[s], 4);
            ptx::mbar_init(&empty[s], 1);
            ptx::mbar_init(&bfull[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], LD_EPI_WARPS);
        }
        ptx::fence_barrier_init();
    }
    if (warp == LD_MMA_WARP) ptx::tmem_alloc(tslot, TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = *tslot;

    if (warp == LD_BW_WARP) {
        // B producer: the stage sequence of the MMA warp; each stage = the weight blocks of its K-steps
        if (lane == 0) {
            int sglob = 0;
            for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
                const int nt = tile / p.mtiles;
                const LdClass& cl = p.cls[tile_class(tile % p.mtiles)];
                const int tst = (cl.kn + LD_KPS - 1) / LD_KPS;
                const uint8_t* wn = p.wpack + (size_t)nt * p.ksteps_all * KBLK;
                for (int js = 0; js < tst; ++js, ++sglob) {
                    const int st = sglob & (LD_STAGES - 1);
                    ptx::mbar_wait(&empty[st], ((sglob / LD_STAGES) & 1) ^ 1);
                    ptx::mbar_arrive_expect_tx(&bfull[st], BSTAGE);
                    for (int kk = 0; kk < LD_KPS; ++kk) {
                        const int ks = js * LD_KPS + kk;
                        // padded tail K-steps load block 0 (finite weights times zero A columns)
                        const int blk = ks < cl.kn ? wtab[cl.k0 + ks] : 0;
                        bulk_g2s(bring + st * BSTAGE + kk * KBLK, wn + (size_t)blk * KBLK, KBLK, &bfull[st]);
                    }
                }
            }
        }
    } else if (warp == LD_MMA_WARP) {
        // the whole warp runs the issue loop (warp-uniform values); an elected lane issues
        constexpr uint32_t idesc = ptx::idesc_bf16(128, NT, 0, 0);
        const uint64_t bdesc0 = desc_sw32(ptx::smem_u32(bring));
        int sglob = 0, acc = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tempty[acc], aphase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tm + acc * NT;
            const int tst = tile_stages(tile);
            for (int js = 0; js < tst; ++js, ++sglob) {
                const int st = sglob & (LD_STAGES - 1);
                const uint32_t ph = (sglob / LD_STAGES) & 1;
                ptx::mbar_wait(&full[st], ph);
                ptx::mbar_wait(&bfull[st], ph);
                ptx::tc_fence_after();
                const uint32_t a0 = tm + ACC_COLS + st * STAGE_COLS;
                const uint64_t b0 = bdesc0 + (uint64_t)((st * BSTAGE) >> 4);
#pragma unroll
                for (int kk = 0; kk < LD_KPS; ++kk)
                    mma_bf16_ts_elect(d, a0 + 8 * kk, b0 + (uint64_t)((kk * KBLK) >> 4), idesc, (js | kk) ? 1u : 0u);
                commit_elect(&empty[st]);
            }
            commit_elect(&tfull[acc]);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    } else if (warp >= LD_EPI_WARPS) {
        // builders: group g fills the stages sglob = g (mod LD_GROUPS) (every use of a stage by one group)
        const int g = (warp - LD_EPI_WARPS) >> 2, q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        int sglob = g, js = g, tile = blockIdx.x;
        auto advance = [&](int& t, int& j) {
            while (t < p.tiles) {
                const int n = tile_stages(t);
                if (j < n) break;
                j -= n;
                t += gridDim.x;
            }
        };
        advance(tile, js);
        // this lane's pixel in a tile and the dy neighbour of K-list entry ks of it
        struct Px {
            int rc, cc, pc, k0, kn;
            bool valid;
            const uint16_t* dyb;
        };
        auto pixel = [&](int t) {
            Px x;
            const LdClass& cl = p.cls[tile_class(t % p.mtiles)];
            const int idx = (t % p.mtiles - cl.tile0) * 128 + q * 32 + lane, per = cl.nr * cl.nc;
            x.valid = idx < p.B * per;
            const int b = x.valid ? idx / per : 0;
            const int r2 = idx - b * per, i = r2 / cl.nc, j = r2 - i * cl.nc;
            x.rc = cl.cr + p.s * i;
            x.cc = cl.ccl + 2 * p.s * j;
            x.pc = (x.cc + p.parity) & 1;
            x.dyb = p.dy + (size_t)b * p.Ho * p.Wo * p.Cout;
            x.k0 = cl.k0;
            x.kn = cl.kn;
            return x;
        };
        auto neighbour = [&](const Px& x, int ks, bool* ok) -> const uint16_t* {
            const bool in_k = ks < x.kn;
            const uint32_t e = ktab[x.k0 + (in_k ? ks : 0)];
            const int dc = (int8_t)(e & 0xFF), dr = (int8_t)((x.pc ? e >> 16 : e >> 8) & 0xFF);
            const int c0 = (int)(e >> 24) * 16;
            const int qr = x.rc + dr, qc = x.cc + dc;
            // the neighbour must be in the grid and a centre of the stride-s lattice (the class guarantees the
            // latter away from the borders; tested per pixel like the grid edges)
            const int Cq = qc / p.s;
            const int rr = qr - hex_rho(Cq, p.s, p.parity);
            const int Rq = rr / p.s;
            *ok = in_k && x.valid && (unsigned)qr < (unsigned)p.H && (unsigned)qc < (unsigned)p.W && qc == Cq * p.s &&
                  rr >= 0 && rr == Rq * p.s && Rq < p.Ho && Cq < p.Wo;
            return x.dyb + ((size_t)(*ok ? Rq * p.Wo + Cq : 0)) * p.Cout + c0;
        };
        auto finish_stage = [&](int st) {
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&full[st]);
        };
        if (p.kc16 % LD_KPS == 0) {
            // A stage's K-steps are 4 consecutive 16-channel chunks of ONE tap: every pixel needs one 128-byte
            // line of dy.  The warp loads its 32 lines cooperatively -- 8 lanes per line, 4 lines per request
            // instead of 32 -- into registers one stage AHEAD, parks them in its staging tile (16-byte chunks
            // XOR-swizzled by the row: conflict-free both ways) and each lane reads back its own row.
            uint8_t* stg = bring + LD_STAGES * BSTAGE + (warp - LD_EPI_WARPS) * 4096;
            uint4 pre[8];
            int pre_nvalid = 0;
            auto prefetch = [&](int t, int j) {
                const Px x = pixel(t);
                bool ok;
                const unsigned long long my = (unsigned long long)neighbour(x, j * LD_KPS, &ok);
                pre_nvalid = x.kn - j * LD_KPS;  // < 4 only for a padded (neighbour-less) class
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int m = 4 * i + (lane >> 3), c = lane & 7;
                    const unsigned long long a = __shfl_sync(0xffffffffu, my, m);
                    const int okm = __shfl_sync(0xffffffffu, ok ? 1 : 0, m);
                    pre[i] = okm ? __ldg(reinterpret_cast<const uint4*>(a) + c) : make_uint4(0u, 0u, 0u, 0u);
                }
            };
            if (tile < p.tiles) prefetch(tile, js);
            for (; tile < p.tiles; sglob += LD_GROUPS) {
                __syncwarp();  // the previous stage's reads of the staging tile are done
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                    const int m = 4 * i + (lane >> 3), c = lane & 7;
                    *reinterpret_cast<uint4*>(stg + m * 128 + ((c ^ (m & 7)) << 4)) = pre[i];
                }
                __syncwarp();
                const int nvalid = pre_nvalid;
                int nt = tile, nj = js + LD_GROUPS;
                advance(nt, nj);
                if (nt < p.tiles) prefetch(nt, nj);  // next stage's lines in flight during this stage's stores
                const int st = sglob & (LD_STAGES - 1);
                ptx::mbar_wait(&empty[st], ((sglob / LD_STAGES) & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t ta = tm + lane_base + ACC_COLS + st * STAGE_COLS;
#pragma unroll
                for (int kk = 0; kk < LD_KPS; ++kk) {
                    const uint4 z = make_uint4(0u, 0u, 0u, 0u);
                    uint4 a0 = *reinterpret_cast<const uint4*>(stg + lane * 128 + (((2 * kk) ^ (lane & 7)) << 4));
                    uint4 a1 = *reinterpret_cast<const uint4*>(stg + lane * 128 + (((2 * kk + 1) ^ (lane & 7)) << 4));
                    if (kk >= nvalid) { a0 = z; a1 = z; }
                    const uint32_t w8[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
                    tmem_st8(ta + 8 * kk, w8);
                }
                finish_stage(st);
                tile = nt;
                js = nj;
            }
        } else {
            // general Cout: per K-step one 256-bit load of the 16 channels (32 contiguous bytes) per lane
            int cur = -1;
            Px x{};
            for (; tile < p.tiles; sglob += LD_GROUPS) {
                if (tile != cur) {
                    cur = tile;
                    x = pixel(tile);
                }
                uint4 v[LD_KPS][2];
#pragma unroll
                for (int kk = 0; kk < LD_KPS; ++kk) {
                    bool ok;
                    const uint16_t* src = neighbour(x, js * LD_KPS + kk, &ok);
                    uint32_t r8[8];
                    asm volatile("ld.global.nc.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                                 : "=r"(r8[0]), "=r"(r8[1]), "=r"(r8[2]), "=r"(r8[3]), "=r"(r8[4]), "=r"(r8[5]),
                                   "=r"(r8[6]), "=r"(r8[7])
                                 : "l"(src));
                    v[kk][0] = ok ? make_uint4(r8[0], r8[1], r8[2], r8[3]) : make_uint4(0u, 0u, 0u, 0u);
                    v[kk][1] = ok ? make_uint4(r8[4], r8[5], r8[6], r8[7]) : make_uint4(0u, 0u, 0u, 0u);
                }
                const int st = sglob & (LD_STAGES - 1);
                ptx::mbar_wait(&empty[st], ((sglob / LD_STAGES) & 1) ^ 1);
                ptx::tc_fence_after();
                const uint32_t ta = tm + lane_base + ACC_COLS + st * STAGE_COLS;
#pragma unroll
                for (int kk = 0; kk < LD_KPS; ++kk) {
                    const uint32_t w8[8] = {v[kk][0].x, v[kk][0].y, v[kk][0].z, v[kk][0].w,
                                            v[kk][1].x, v[kk][1].y, v[kk][1].z, v[kk][1].w};
                    tmem_st8(ta + 8 * kk, w8);
                }
                finish_stage(st);
                js += LD_GROUPS;
                advance(tile, js);
            }
        }
    } else {
        // epilogue: warp w drains TMEM lanes 32q .. 32q+31 (q = w % 4: its 32 pixels), channel part w / 4
        constexpr int PARTS = LD_EPI_WARPS / 4, PCOLS = NT / PARTS;
        const int q = warp & 3, half = warp >> 2;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        int acc = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const int nt = tile / p.mtiles;
            const LdClass& cl = p.cls[tile_class(tile % p.mtiles)];
            const int idx = (tile % p.mtiles - cl.tile0) * 128 + q * 32 + lane, per = cl.nr * cl.nc;
            const bool vpix = idx < p.B * per;
            const int b = vpix ? idx / per : 0;
            const int r2 = idx - b * per, i = r2 / cl.nc, j = r2 - i * cl.nc;
            const int r = cl.cr + p.s * i, c = cl.ccl + 2 * p.s * j;
            const size_t pix = ((size_t)b * p.H + r) * p.W + c;
            uint16_t* out = p.dx + pix * p.Cin + nt * NT;
            const uint16_t* msk = p.relu_y ? p.relu_y + pix * p.Cin + nt * NT : nullptr;
            const uint32_t dbase = tm + lane_base + acc * NT;
#pragma unroll 1
            for (int c0 = half * PCOLS; c0 < (half + 1) * PCOLS; c0 += 32) {
                uint32_t u[32];
                ptx::tmem_ld32(dbase + c0, u);
                ptx::tmem_ld_wait();
                if (c0 + 32 >= (half + 1) * PCOLS) {  // this warp's part is drained: hand it back
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
                }
                if (!vpix) continue;
#pragma unroll
                for (int h = 0; h < 4; ++h) {  // 8 channels per 16-byte store
                    uint32_t mk[4] = {0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu, 0xFFFFFFFFu};
                    if (msk) {
                        const uint4 m4 = __ldg(reinterpret_cast<const uint4*>(msk + c0 + 8 * h));
                        const uint32_t mw[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
                        for (int e = 0; e < 4; ++e) {  // keep where the bf16 mask value is > 0
                            const float lo = __uint_as_float(mw[e] << 16), hi = __uint_as_float(mw[e] & 0xFFFF0000u);
                            mk[e] = (lo > 0.f ? 0x0000FFFFu : 0u) | (hi > 0.f ? 0xFFFF0000u : 0u);
                        }
                    }
                    uint32_t pk[4];
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        __nv_bfloat162 hv = __floats2bfloat162_rn(__uint_as_float(u[8 * h + 2 * e]),
                                                                  __uint_as_float(u[8 * h + 2 * e + 1]));
                        pk[e] = *reinterpret_cast<uint32_t*>(&hv) & mk[e];
                    }
                    *reinterpret_cast<uint4*>(out + c0 + 8 * h) = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                }
            }
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == LD_MMA_WARP) ptx::tmem_dealloc(tm, TMEM_COLS);
}

// wp[nt][ks = t * kc16 + c16][row n][16 k] (SW32: 16-byte chunk (k / 8) ^ ((n >> 2) & 1)) =
//   W'[ci = nt * NT + n][co = 16 c16 + k][t] = W[co][ci][T-1-t]     (bwd-data weights, pin P18)
__global__ void lat_pack_kernel(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wp, int Cout,
                                int Cin, int T, int NT, int kc16) {
    const int64_t total = (int64_t)(Cin / NT) * T * kc16 * NT * 16;
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= total) return;
    const int k = (int)(i % 16);
    int64_t r = i / 16;
    const int n = (int)(r % NT);
    r /= NT;
    const int ks = (int)(r % (T * kc16));
    const int nt = (int)(r / (T * kc16));
    const int t = ks / kc16, c16 = ks - t * kc16;
    const int ci = nt * NT + n, co = 16 * c16 + k;
    const __nv_bfloat16 v = w[((int64_t)co * Cin + ci) * T + (T - 1 - t)];
    const int64_t blk = ((int64_t)nt * T * kc16 + ks) * NT * 16;
    wp[blk + n * 16 + (((k >> 3) ^ ((n >> 2) & 1)) << 3) + (k & 7)] = v;
}

int lat_nt(int Cin) { return Cin % 128 == 0 ? 128 : 64; }

}  // namespace

bool lat_dgrad_supported(const Geom& g, int Cin, int Cout) {
    if (sw_on("HEXCONV_NO_LAT_DGRAD")) return false;
    if (g.s < 2 || g.s > 3 || g.T > LD_MAXT || Cin % 64 || Cout % 16 || Cout > 16 * 255) return false;
    if (g.B * (int64_t)g.H * g.W > INT32_MAX / 2) return false;
    return true;
}

size_t lat_dgrad_ws_bytes(const Geom& g, int Cin, int Cout) {
    return (size_t)g.T * (Cout / 16) * Cin * 32 + 1024;
}

hex_status_t lat_dgrad(const Geom& g, int Cin, int Cout, const void* dy, const void* w, const void* relu_y, void* dx,
                       void* ws, size_t ws_bytes, cudaStream_t st) {
    if (!lat_dgrad_supported(g, Cin, Cout)) return HEX_ERR_UNSUPPORTED;
    if (ws_bytes < lat_dgrad_ws_bytes(g, Cin, Cout)) return HEX_ERR_WORKSPACE;
    const int NT = lat_nt(Cin);
    const int kc16 = Cout / 16;
    uint8_t* wp = reinterpret_cast<uint8_t*>(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    LdParams p{};
    p.dy = (const uint16_t*)dy;
    p.relu_y = (const uint16_t*)relu_y;
    p.dx = (uint16_t*)dx;
    p.wpack = wp;
    p.B = g.B; p.H = g.H; p.W = g.W; p.Ho = g.Ho; p.Wo = g.Wo; p.Cin = Cin; p.Cout = Cout;
    p.s = g.s; p.parity = g.parity; p.T = g.T; p.kc16 = kc16; p.ksteps_all = g.T * kc16;
    p.ntiles = Cin / NT;
    for (int t = 0; t < g.T; ++t) {
        int dc, dr0, dr1;
        tap_offset(g.n, 0, t, &dc, &dr0);
        tap_offset(g.n, 1, t, &dc, &dr1);
        p.dc[t] = (int8_t)dc;
        p.dr0[t] = (int8_t)dr0;
        p.dr1[t] = (int8_t)dr1;
    }
    // phase classes (r mod s, c mod 2s), their lattice taps decided on a representative interior pixel
    const int s = g.s;
    int nk = 0, tile0 = 0;
    for (int cr = 0; cr < s; ++cr)
        for (int ccl = 0; ccl < 2 * s; ++ccl) {
            const int nr = cr < g.H ? (g.H - cr + s - 1) / s : 0, nc = ccl < g.W ? (g.W - ccl + 2 * s - 1) / (2 * s) : 0;
            if (nr * nc == 0) continue;
            LdClass& cl = p.cls[p.ncls++];
            cl.cr = cr; cl.ccl = ccl; cl.nr = nr; cl.nc = nc; cl.tile0 = tile0; cl.k0 = nk;
            const int r_rep = cr + 8 * s, c_rep = ccl + 16 * s, pc = (c_rep + g.parity) & 1;
            for (int t = 0; t < g.T; ++t) {
                const int qc = c_rep + p.dc[t], qr = r_rep + (pc ? p.dr1[t] : p.dr0[t]);
                if (qc % s) continue;
                if ((qr - hex_rho(qc / s, s, g.parity)) % s) continue;
                for (int c16 = 0; c16 < kc16; ++c16) {
                    if (nk >= LD_MAXKL) return HEX_ERR_UNSUPPORTED;
                    p.klist[nk++] = (uint16_t)(t | (c16 << 8));
                }
            }
            cl.kn = nk - cl.k0;
            if (cl.kn == 0) {  // no lattice tap: the class's dx is zero but its tiles still need writing
                p.klist[nk++] = (uint16_t)0;
                cl.kn = 1;
            }
            tile0 += ceil_div((int64_t)g.B * nr * nc, 128);
        }
    p.mtiles = tile0;
    p.tiles = tile0 * p.ntiles;
    const int smem = 1024 + LD_STAGES * LD_KPS * NT * 32 + LD_BLD_WARPS * 4096 + 3 * LD_STAGES * 8 + 32 + 16 + 6 * nk + 16;
    if (smem > LD_SMEM_MAX) return HEX_ERR_UNSUPPORTED;
    {  // weights packed only once the plan fits (UNSUPPORTED above launches nothing)
        const int64_t total = (int64_t)(Cin / NT) * g.T * kc16 * NT * 16;
        lat_pack_kernel<<<ceil_div(total, 256), 256, 0, st>>>((const __nv_bfloat16*)w, (__nv_bfloat16*)wp, Cout, Cin,
                                                               g.T, NT, kc16);
        count_launch();
        if (last_launch_status() != HEX_OK) return HEX_ERR_CUDA;
    }
    const int grid = p.tiles < num_sms() ? p.tiles : num_sms();
    if (NT == 128) {
        static bool attr = false;
        if (!attr) {
            if (cudaFuncSetAttribute(lat_dgrad_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, LD_SMEM_MAX) !=
                cudaSuccess)
                return HEX_ERR_CUDA;
            attr = true;
        }
        lat_dgrad_kernel<128><<<grid, LD_THREADS, smem, st>>>(p);
    } else {
        static bool attr = false;
        if (!attr) {
            if (cudaFuncSetAttribute(lat_dgrad_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, LD_SMEM_MAX) !=
                cudaSuccess)
                return HEX_ERR_CUDA;
            attr = true;
        }
        lat_dgrad_kernel<64><<<grid, LD_THREADS, smem, st>>>(p);
    }
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
