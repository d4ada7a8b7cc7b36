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
//   * A tile = 16 class rows x 8 class columns.  For a class and a lattice tap the dy neighbours of those 128
//     pixels are a RECTANGLE of dy: rows Rq = i + a, lattice columns Cq = 2 j + b (s = 2; in general the
//     class column period 2s is two lattice columns), i.e. one box of a parity view of dy (the lattice
//     columns of one parity) -- so A is ONE TMA box per (tap, 64-channel chunk), SWIZZLE_128B K-major, and
//     the MMA reads it from shared memory.  Out-of-grid neighbours are the box's zero fill.
//   * B (the chunk's four K16 weight blocks: N-tile rows x 16 K values, K-major SWIZZLE_32B, packed once per
//     call by lat_pack_kernel in (tap, chunk) order) arrives with the A box in the same pipeline stage (one
//     bulk copy).
//   * Warp roles: warp 0 produces (TMA box + bulk copy per K-list entry, 6-stage ring), warp 1 issues the
//     kind::f16 MMAs (warp-uniform loop, elect.sync), warps 2..5 drain TMEM (ReLU-backward mask, bf16,
//     16-byte NHWC stores); two TMEM accumulators (the epilogue of tile i overlaps the MMAs of tile i+1).
// Deterministic: every output element is one MMA chain in fixed K order.
#include <cuda.h>
#include <cudaTypedefs.h>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hexconv {
namespace {

constexpr int LD_STAGES = 6;
constexpr int LD_THREADS = 192;   // warp 0 producer, warp 1 MMA, warps 2..5 epilogue
constexpr int LD_MAXT = 37;       // n <= 3
constexpr int LD_MAXCLS = 18;     // 2 s^2, s <= 3
constexpr int LD_MAXKL = 1024;    // K-list entries (lattice tap, 64-channel chunk) over all classes
constexpr int LD_TR = 16, LD_TC = 8;  // class rows x class columns per tile (M = 128, m = 16 jj + ii)
constexpr int LD_SMEM_MAX = 220 * 1024;

struct LdClass {
    int cr, ccl;        // r mod s, c mod 2s
    int nr, nc;         // class rows / columns per image
    int ti, tj;         // tiles along class rows / columns per image
    int tile0, k0, kn;  // first tile (per N tile), first K-list entry, entries
};

struct LdParams {
    const uint16_t* relu_y;  // [B][H][W][Cin] mask source or null
    uint16_t* dx;            // [B][H][W][Cin]
    const uint8_t* wpack;    // [n tile][K-step (t, c16)][NT rows x 32 B] SW32 blocks
    int B, H, W, Cin, Cout, s, kc16, ksteps_all, ntiles, mtiles, tiles;
    int ncls;
    LdClass cls[LD_MAXCLS];
    // per K-list entry: dy parity view | 64-channel chunk << 1, box row offset, box sub-column offset, and the
    // entry's first weight block (t * kc16 + 4 * chunk; the chunk's 4 blocks are consecutive)
    uint8_t kview[LD_MAXKL];
    int8_t krow[LD_MAXKL], kcol[LD_MAXKL];
    uint16_t kblk[LD_MAXKL];
};

__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__device__ __forceinline__ void mma_ss_elect(uint32_t d, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                             uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void commit_elect(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n\t}" ::"r"(
            ptx::smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ptx::smem_u32(dst)),
                 "l"((uint64_t)src), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}

struct LdTile {
    int nt, cls, b, i0, j0;
};
__device__ __forceinline__ LdTile ld_tile(const LdParams& p, int tile) {
    LdTile t;
    t.nt = tile / p.mtiles;
    const int m = tile - t.nt * p.mtiles;
    int c = 0;
    while (c + 1 < p.ncls && m >= p.cls[c + 1].tile0) ++c;
    t.cls = c;
    const LdClass& cl = p.cls[c];
    int r = m - cl.tile0;
    const int jt = r % cl.tj;
    r /= cl.tj;
    const int it = r % cl.ti;
    t.b = r / cl.ti;
    t.i0 = it * LD_TR;
    t.j0 = jt * LD_TC;
    return t;
}

template <int NT>
__global__ void __launch_bounds__(LD_THREADS, 1)
lat_dgrad_kernel(const __grid_constant__ CUtensorMap map_v0, const __grid_constant__ CUtensorMap map_v1,
                 const __grid_constant__ LdParams p) {
    constexpr uint32_t A_BYTES = LD_TR * LD_TC * 128;  // one 64-channel dy box (16 KB)
    constexpr uint32_t KBLK = NT * 32;                 // one K16 weight block
    constexpr uint32_t B_BYTES = 4 * KBLK;             // the chunk's 4 blocks
    constexpr uint32_t STAGE = A_BYTES + B_BYTES;
    constexpr int TMEM_COLS = 2 * NT <= 256 ? 256 : 512;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* ring = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint64_t* full = reinterpret_cast<uint64_t*>(ring + LD_STAGES * STAGE);
    uint64_t* empty = full + LD_STAGES;
    uint64_t* tfull = empty + LD_STAGES;
    uint64_t* tempty = tfull + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < LD_STAGES; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], 1);
            ptx::mbar_init(&tempty[a], 4);
        }
        ptx::fence_barrier_init();
        ptx::prefetch_tmap(&map_v0);
        ptx::prefetch_tmap(&map_v1);
    }
    if (warp == 1) ptx::tmem_alloc(tslot, TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = *tslot;

    if (warp == 0) {
        // producer: per K-list entry of the tile's class, the dy box and the chunk's 4 weight blocks
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
                const LdTile t = ld_tile(p, tile);
                const LdClass& cl = p.cls[t.cls];
                const uint8_t* wn = p.wpack + (size_t)t.nt * p.ksteps_all * KBLK;
                for (int e = cl.k0; e < cl.k0 + cl.kn; ++e) {
                    ptx::mbar_wait(&empty[stage], phase ^ 1);
                    uint8_t* sa = ring + stage * STAGE;
                    ptx::mbar_arrive_expect_tx(&full[stage], STAGE);
                    const int kv = p.kview[e];
                    ptx::tma_load_5d((kv & 1) ? &map_v1 : &map_v0, &full[stage], sa, 0, t.i0 + p.krow[e],
                                     t.j0 + p.kcol[e], t.b, kv >> 1);
                    bulk_g2s(sa + A_BYTES, wn + (size_t)p.kblk[e] * KBLK, B_BYTES, &full[stage]);
                    if (++stage == LD_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // MMA issue: the whole warp runs the loop (warp-uniform values), an elected lane issues
        constexpr uint32_t idesc = ptx::idesc_bf16(128, NT, 0, 0);
        const uint64_t adesc0 = ptx::smem_desc_sw128(ptx::smem_u32(ring), 16, 1024);
        const uint64_t bdesc0 = desc_sw32(ptx::smem_u32(ring) + A_BYTES);
        int stage = 0, acc = 0;
        uint32_t phase = 0, aphase = 0;
        for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            const LdTile t = ld_tile(p, tile);
            const int kn = p.cls[t.cls].kn;
            ptx::mbar_wait(&tempty[acc], aphase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tm + acc * NT;
            for (int e = 0; e < kn; ++e) {
                ptx::mbar_wait(&full[stage], phase);
                ptx::tc_fence_after();
                const uint64_t ad = adesc0 + (uint64_t)((stage * STAGE) >> 4);
                const uint64_t bd = bdesc0 + (uint64_t)((stage * STAGE) >> 4);
#pragma unroll
                for (int k = 0; k < 4; ++k)  // 16 channels each: A advances 32 bytes, B one block
                    mma_ss_elect(d, ad + (uint64_t)(2 * k), bd + (uint64_t)((k * KBLK) >> 4), idesc,
                                 (e | k) ? 1u : 0u);
                commit_elect(&empty[stage]);
                if (++stage == LD_STAGES) { stage = 0; phase ^= 1; }
            }
            commit_elect(&tfull[acc]);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    } else {
        // epilogue: warp w drains TMEM lanes 32q .. 32q+31 (q = w % 4): tile pixel m = 16 jj + ii
        const int q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const int m = q * 32 + lane, ii = m & (LD_TR - 1), jj = m / LD_TR;
        int acc = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            const LdTile t = ld_tile(p, tile);
            const LdClass& cl = p.cls[t.cls];
            ptx::mbar_wait(&tfull[acc], aphase);
            ptx::tc_fence_after();
            const int i = t.i0 + ii, j = t.j0 + jj;
            const bool vpix = i < cl.nr && j < cl.nc;
            const int r = cl.cr + p.s * i, c = cl.ccl + 2 * p.s * j;
            const size_t pix = ((size_t)t.b * p.H + r) * p.W + c;
            uint16_t* out = p.dx + pix * p.Cin + t.nt * NT;
            const uint16_t* msk = p.relu_y ? p.relu_y + pix * p.Cin + t.nt * NT : nullptr;
            const uint32_t dbase = tm + lane_base + acc * NT;
#pragma unroll 1
            for (int c0 = 0; c0 < NT; c0 += 32) {
                uint32_t u[32];
                ptx::tmem_ld32(dbase + c0, u);
                ptx::tmem_ld_wait();
                if (c0 + 32 >= NT) {  // the accumulator is drained: hand it back to the MMA warp
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
    if (warp == 1) ptx::tmem_dealloc(tm, TMEM_COLS);
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

// parity view v of the dy lattice grid (lattice columns v, v+2, ...), NHWC bf16, channels split into 64-channel
// chunks as the outer dimension: dims {64, Ho, ceil((Wo-v)/2), B, C/64}, box {64, 16 rows, 8 sub-columns, 1, 1}
bool lat_view_map(CUtensorMap* m, const void* base, int B, int Ho, int Wo, int C, int v) {
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            enc = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    if (!enc) return false;
    const int Wv = (Wo - v + 1) / 2;
    if (Wv < 1) return false;
    cuuint64_t dims[5] = {64, (cuuint64_t)Ho, (cuuint64_t)Wv, (cuuint64_t)B, (cuuint64_t)(C / 64)};
    cuuint64_t strides[4] = {(cuuint64_t)Wo * C * 2, (cuuint64_t)2 * C * 2, (cuuint64_t)Ho * Wo * C * 2, 128};
    cuuint32_t box[5] = {64, (cuuint32_t)LD_TR, (cuuint32_t)LD_TC, 1, 1};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    void* addr = (void*)((const char*)base + (size_t)v * C * 2);
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, addr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }

}  // namespace

bool lat_dgrad_supported(const Geom& g, int Cin, int Cout) {
    if (sw_on("HEXCONV_NO_LAT_DGRAD")) return false;
    if (g.s < 2 || g.s > 3 || g.T > LD_MAXT || Cin % 64 || Cout % 64 || g.Wo < 2) return false;
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
    const int NT = Cin % 128 == 0 ? 128 : 64;
    const int kc16 = Cout / 16, kc64 = Cout / 64;
    uint8_t* wp = reinterpret_cast<uint8_t*>(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    LdParams p{};
    p.relu_y = (const uint16_t*)relu_y;
    p.dx = (uint16_t*)dx;
    p.wpack = wp;
    p.B = g.B; p.H = g.H; p.W = g.W; p.Cin = Cin; p.Cout = Cout;
    p.s = g.s; p.kc16 = kc16; p.ksteps_all = g.T * kc16;
    p.ntiles = Cin / NT;
    int dc[LD_MAXT], dr0[LD_MAXT], dr1[LD_MAXT];
    for (int t = 0; t < g.T; ++t) {
        tap_offset(g.n, 0, t, &dc[t], &dr0[t]);
        tap_offset(g.n, 1, t, &dc[t], &dr1[t]);
    }
    // phase classes (r mod s, c mod 2s).  For class pixel (i, j) at (cr + s i, ccl + 2s j) and tap t the
    // neighbour q = (cr + s i + dr, ccl + 2s j + dc) is a lattice centre (decided on a representative pixel)
    // at lattice column Cq = (ccl + dc) / s + 2j and row Rq = (cr + dr - rho(Cq)) / s + i: view Cq mod 2,
    // sub-column ((ccl + dc) / s) div 2 + j, row offset (cr + dr - rho) / s.
    const int s = g.s;
    int nk = 0, tile0 = 0;
    for (int cr = 0; cr < s; ++cr)
        for (int ccl = 0; ccl < 2 * s; ++ccl) {
            const int nr = cr < g.H ? (g.H - cr + s - 1) / s : 0, nc = ccl < g.W ? (g.W - ccl + 2 * s - 1) / (2 * s) : 0;
            if (nr * nc == 0) continue;
            LdClass& cl = p.cls[p.ncls++];
            cl.cr = cr; cl.ccl = ccl; cl.nr = nr; cl.nc = nc;
            cl.ti = ceil_div(nr, LD_TR);
            cl.tj = ceil_div(nc, LD_TC);
            cl.tile0 = tile0;
            cl.k0 = nk;
            const int pc = (ccl + g.parity) & 1;  // centre column parity of every pixel of the class
            for (int t = 0; t < g.T; ++t) {
                const int ddr = pc ? dr1[t] : dr0[t];
                const int qc0 = ccl + dc[t];          // the neighbour column of class column j = 0
                if (((qc0 % s) + s) % s) continue;    // not a lattice column
                const int Cq0 = floor_div(qc0, s);   // lattice column of j = 0 (Cq = Cq0 + 2j)
                const int rho = hex_rho(((Cq0 % 2) + 2) % 2, s, g.parity);  // rho has period 2 in C
                const int rr0 = cr + ddr - rho;        // neighbour row minus rho for i = 0 (Rq = rr0 / s + i)
                if (((rr0 % s) + s) % s) continue;    // not a lattice row
                const int Rq0 = floor_div(rr0, s);
                const int v = ((Cq0 % 2) + 2) % 2;
                const int sub0 = floor_div(Cq0 - v, 2);  // sub-column of view v for j = 0
                if (Rq0 < -128 || Rq0 > 127 || sub0 < -128 || sub0 > 127) return HEX_ERR_UNSUPPORTED;
                for (int c64 = 0; c64 < kc64; ++c64) {
                    if (nk >= LD_MAXKL) return HEX_ERR_UNSUPPORTED;
                    p.kview[nk] = (uint8_t)(v | (c64 << 1));
                    p.krow[nk] = (int8_t)Rq0;
                    p.kcol[nk] = (int8_t)sub0;
                    p.kblk[nk] = (uint16_t)(t * kc16 + 4 * c64);
                    ++nk;
                }
            }
            cl.kn = nk - cl.k0;
            if (cl.kn == 0) {  // no lattice tap: the class's dx is zero, written by one all-zero-fill entry
                if (nk >= LD_MAXKL) return HEX_ERR_UNSUPPORTED;
                p.kview[nk] = 0;
                p.krow[nk] = -64;  // a box entirely above the grid: zero fill
                p.kcol[nk] = 0;
                p.kblk[nk] = 0;
                ++nk;
                cl.kn = 1;
            }
            tile0 += g.B * cl.ti * cl.tj;
        }
    p.mtiles = tile0;
    p.tiles = tile0 * p.ntiles;
    const int stage = LD_TR * LD_TC * 128 + 4 * NT * 32;
    const int smem = 1024 + LD_STAGES * stage + 2 * LD_STAGES * 8 + 4 * 8 + 16;
    if (smem > LD_SMEM_MAX || (int64_t)g.T * kc16 > 65535) return HEX_ERR_UNSUPPORTED;
    CUtensorMap mv0, mv1;
    if (!lat_view_map(&mv0, dy, g.B, g.Ho, g.Wo, Cout, 0) || !lat_view_map(&mv1, dy, g.B, g.Ho, g.Wo, Cout, 1))
        return HEX_ERR_UNSUPPORTED;
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
        lat_dgrad_kernel<128><<<grid, LD_THREADS, smem, st>>>(mv0, mv1, p);
    } else {
        static bool attr = false;
        if (!attr) {
            if (cudaFuncSetAttribute(lat_dgrad_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, LD_SMEM_MAX) !=
                cudaSuccess)
                return HEX_ERR_CUDA;
            attr = true;
        }
        lat_dgrad_kernel<64><<<grid, LD_THREADS, smem, st>>>(mv0, mv1, p);
    }
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
