// tf32_conv.cu -- fp32 hexagonal convolution on the tcgen05 tensor cores in 3xTF32.
//
// The fp32 layers of configs 2 and 3 (16 -> 32, 32 -> 64 channels) are dense contractions too small for the
// 64-channel bf16 tiles, and on CUDA cores they are FFMA-bound (arithmetic intensity 50-100 FLOP/B).
// Here each one is an implicit GEMM on the tensor cores with fp32 accuracy:
//
//   * M = 128 output pixels (consecutive in the flattened (b, R, C) order of the output grid, so a tile may
//     span images and no pixel of a ragged image is wasted), N = output channels (padded to 16, <= 64),
//     K = (tap, 8-channel chunk) -- (tap, ci) packed into K, so 16 input channels x 19 taps is K = 304
//     with no 64-channel padding.
//   * 3xTF32 split (reading A13): every operand value v = hi + lo with hi = cvt.rna.tf32(v) and
//     lo = v - hi (exact in fp32); D += A_hi.B_hi + A_hi.B_lo + A_lo.B_hi.  The dropped A_lo.B_lo term and
//     the tf32 rounding of lo are ~2^-22 of |a.b|: normwise error ~5e-7 against fp64 (tools/tf32_probe.cu),
//     inside the fp32 bar of 1e-5 (A14).
//   * A (the hexagonal gather) is built directly in TENSOR MEMORY: builder warps -- one thread per output
//     pixel, i.e. per TMEM lane -- gather the 8 channels of one tap for their pixel (offset-column geometry,
//     PAPER.md:144-151; off-grid neighbours read 0, A4), split them and write hi / lo with tcgen05.st; the
//     MMA reads A from TMEM ([a_tmem] operand), so the gather costs no shared-memory bandwidth.
//   * B (weights, pre-split hi / lo, K-major SWIZZLE_32B: one 32-byte row = the 8 K values of one output
//     channel) is resident in shared memory for the whole persistent kernel (one bulk copy).
//   * Warp roles: 4 epilogue warps (TMEM -> registers -> bias / ReLU / ReLU-backward mask -> NCHW stores,
//     coalesced across the 32 pixels of a warp), 16 builder warps in 4 groups taking 4-K-step stages
//     round-robin (all 32 loads of a stage issued before any is used; the hi / lo split as two integer ops),
//     and 1 or 2 MMA-issuing warps (2 where the accumulators fit, N <= 32: the tcgen05.mma front end is
//     per issuing thread) running a warp-uniform loop with elect.sync issue.  A ring of 4 TMEM A stages
//     (4 K-steps x 16 columns: hi, lo) and two accumulator slots (the epilogue of tile i overlaps the MMAs
//     of tile i+1).
//
// Modes (one kernel):
//   forward       output pixel (R, C) of the stride-s lattice has its centre at (rho(C) + sR, sC)
//                 (PAPER.md:152-154, 172-175); taps read x on the full grid.
//   bwd-data      the adjoint: dx = forward of dy with reversed taps and transposed channels (pin P18) on the
//                 full grid; for s > 1 dy is read through the lattice -- a neighbour that is not a lattice
//                 centre contributes 0 (the stride-1 adjoint of dy scattered onto the full grid, P10) -- so
//                 no upsampled copy of dy is written.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

// Development timing probe (tools/tf32_prof.cu builds this file with -DTF_PROF=1): clock64 accumulators of
// where the MMA, builder and epilogue threads of CTA 0 spend their cycles.  Compiled out of the library.
#ifndef TF_PROF
#define TF_PROF 0
#endif
#if TF_PROF
__device__ long long g_tf_prof[32];
#define PROF_T0() long long _pt0 = clock64()
#define PROF_ACC(slot) \
    do { if (blockIdx.x == 0) g_tf_prof_acc[slot] += clock64() - _pt0; _pt0 = clock64(); } while (0)
#else
#define PROF_T0() \
    do {          \
    } while (0)
#define PROF_ACC(slot) \
    do {               \
    } while (0)
#endif

namespace hexconv {
namespace {

constexpr int TF_KPS = 4;                          // K-steps per A stage (one barrier handshake each)
constexpr int TF_STAGES = 4;                       // A stages in TMEM (power of two, = TF_GROUPS)
constexpr int TF_GROUPS = 4;                       // builder groups (K-steps round-robin)
constexpr int TF_EPI_WARPS = 4;
constexpr int TF_BLD_WARPS = 4 * TF_GROUPS;
constexpr int TF_MMA_WARP = TF_EPI_WARPS + TF_BLD_WARPS;
constexpr int tf_threads(int iss) { return (TF_MMA_WARP + iss) * 32; }  // iss MMA-issuing warps
constexpr int TF_MAXT = 37;                        // n <= 3
constexpr int TF_MAX_NT = 64;
constexpr int TF_SMEM_MAX = 220 * 1024;

constexpr int TF_MAXCLS = 18;   // 2 s^2 phase classes, s <= 3
constexpr int TF_MAXKL = 2048;  // K-step list entries over all classes
struct TfClass {
    int cr, ccl;          // r mod s, c mod 2s of the class's pixels
    int nr, nc;           // its rows / columns per image
    int tile0, k0, kn;    // first tile, first K-step list entry, K-steps
};

struct TfParams {
    const float* x;       // gathered tensor, NCHW [B][Cx][Hin][Win]
    const float* bias;    // [Nout] or null
    const float* relu_y;  // mask source shaped like y, or null
    float* y;             // output, NCHW [B][Nout][Hout][Wout]
    int B, Cx, H, W, Hin, Win, Hout, Wout;
    int64_t plane_bytes;  // Hin * Win * 4: the stride between channel planes of x
    int Nout, s, parity, T, kc8, ksteps, relu;
    int out_lat, in_lat;  // output pixels are lattice points / the gathered tensor lives on the lattice
    int total_pix, tiles;
    int8_t dc[TF_MAXT], dr0[TF_MAXT], dr1[TF_MAXT];
    // strided bwd-data (in_lat): the output pixels are split into the 2 s^2 phase classes (r mod s, c mod 2s);
    // within a class the taps whose neighbour is a lattice centre are the same for every pixel, so a tile
    // (one class) runs only those K-steps -- s^2 times fewer MMAs than gathering every tap
    int ncls;
    TfClass cls[TF_MAXCLS];
    uint16_t klist[TF_MAXKL];  // per class, its K-steps: tap | chunk << 8
};

// tf32 rounding to nearest, ties away from zero (= cvt.rna.tf32.f32 for every non-NaN input, Inf kept): add
// half an ulp of the 10-bit mantissa to the magnitude bits and clear the 13 dropped bits -- two integer ops
// where sm_100 compiles cvt.rna.tf32 to a five-instruction sequence with an Inf / NaN test (the builders'
// split of every gathered value is on the hot path).  NaN payloads may become Inf (A10: NaN undefined).
__device__ __forceinline__ float tf32_rna(float v) {
    return __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xffffe000u);
}

// SW32 K-major shared-memory descriptor: 8-row groups 256 B apart (SBO), LBO unused, layout code 6
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
// warp-uniform issue: the whole warp runs the loop (descriptors stay in uniform registers) and one elected
// lane issues the MMA / commit
__device__ __forceinline__ void mma_tf32_ts_elect(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                  uint32_t acc) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\tsetp.ne.b32 p, %4, 0;\n\telect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(d),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc)
        : "memory");
}
__device__ __forceinline__ void mma_commit_elect(uint64_t* bar) {
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
__device__ __forceinline__ void tmem_st_wait() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t* v) {
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, "
        "%15}, [%16];"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
          "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
        : "r"(taddr));
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     ptx::smem_u32(dst)),
                 "l"((uint64_t)src), "r"(bytes), "r"(ptx::smem_u32(bar))
                 : "memory");
}

constexpr int tmem_cols(int NT, int iss) {
    return (4 * NT * iss + TF_STAGES * 16 * TF_KPS) <= 256 ? 256 : 512;
}
// two MMA-issuing warps (each takes half of every stage's K-steps into its own accumulator pair) where the
// accumulators still fit next to the A stages: the MMA front end (~45-75 cycles per tcgen05.mma for N <= 64)
// is per issuing thread
constexpr int tf_issuers(int NT) { return 4 * NT * 2 + TF_STAGES * 16 * TF_KPS <= 512 ? 2 : 1; }

// Output pixel `pix` (flattened b, R, C of the output grid) -> image, centre on the full grid, centre parity.
__device__ __forceinline__ void pixel_centre(const TfParams& p, int pix, int* b, int* rem, int* rc, int* cc) {
    const int hw = p.Hout * p.Wout;
    *b = pix / hw;
    *rem = pix - *b * hw;
    const int R = *rem / p.Wout, C = *rem - R * p.Wout;
    if (p.out_lat) {
        *rc = hex_rho(C, p.s, p.parity) + p.s * R;
        *cc = p.s * C;
    } else {
        *rc = R;
        *cc = C;
    }
}

template <int NT, bool IN_LAT, bool FULLCH>
__global__ void __launch_bounds__(tf_threads(tf_issuers(NT)), 1)
tf32_conv_kernel(const __grid_constant__ TfParams p, const float* __restrict__ wpack) {
    constexpr int ISS = tf_issuers(NT);
    constexpr int ACC_COLS = 4 * NT * ISS;  // per slot and issuer an accumulator of 2 NT columns: [D_hh + D_lh | D_hl]
    constexpr int STAGE_COLS = 16 * TF_KPS;
    constexpr int TMEM_COLS = tmem_cols(NT, ISS);
    static_assert(TF_KPS % ISS == 0, "issuers split a stage's K-steps evenly");
    constexpr uint32_t KBLK = NT * 32;  // bytes of one (K-step, hi|lo) weight block
    extern __shared__ uint8_t smem_raw[];
    uint8_t* wsm = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    const uint32_t wbytes = (uint32_t)p.ksteps * 2u * KBLK;
    uint64_t* full = reinterpret_cast<uint64_t*>(wsm + wbytes);
    uint64_t* empty = full + TF_STAGES;
    uint64_t* tfull = empty + TF_STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* wbar = tempty + 2;
    uint32_t* tslot = reinterpret_cast<uint32_t*>(wbar + 1);
    // per K-step gather entry: dc | dr(centre parity 0) << 8 | dr(parity 1) << 16 | chunk << 24, and (phase
    // classes) the K-step's weight block t * kc8 + chunk
    uint32_t* ktab = tslot + 4;
    const int nkt = IN_LAT ? p.cls[p.ncls - 1].k0 + p.cls[p.ncls - 1].kn : p.ksteps;
    uint16_t* wtab = reinterpret_cast<uint16_t*>(ktab + nkt);
    for (int i = threadIdx.x; i < nkt; i += blockDim.x) {
        int t, c8;
        if (IN_LAT) {
            t = p.klist[i] & 0xFF;
            c8 = p.klist[i] >> 8;
        } else {
            t = i / p.kc8;
            c8 = i - t * p.kc8;
        }
        ktab[i] = (uint32_t)(uint8_t)p.dc[t] | ((uint32_t)(uint8_t)p.dr0[t] << 8) |
                  ((uint32_t)(uint8_t)p.dr1[t] << 16) | ((uint32_t)c8 << 24);
        wtab[i] = (uint16_t)(t * p.kc8 + c8);
    }
    // tile -> (K-step list offset, K-steps, A stages); one class of output pixels per tile (IN_LAT)
    auto tile_class = [&](int tile) -> int {
        int c = 0;
        if (IN_LAT)
            while (c + 1 < p.ncls && tile >= p.cls[c + 1].tile0) ++c;
        return c;
    };
    auto tile_k = [&](int tile, int* k0, int* kn) {
        if (IN_LAT) {
            const TfClass& cl = p.cls[tile_class(tile)];
            *k0 = cl.k0;
            *kn = cl.kn;
        } else {
            *k0 = 0;
            *kn = p.ksteps;
        }
    };
    auto tile_stages = [&](int tile) {
        int k0, kn;
        tile_k(tile, &k0, &kn);
        return (kn + TF_KPS - 1) / TF_KPS;
    };
    // output pixel of TMEM lane `row` of `tile`: image b, offset rem in the output plane, centre (rc, cc)
    auto tile_pixel = [&](int tile, int row, int* b, int* rem, int* rc, int* cc) -> bool {
        if (!IN_LAT) {
            const int pix = tile * 128 + row;
            if (pix >= p.total_pix) return false;
            pixel_centre(p, pix, b, rem, rc, cc);
            return true;
        }
        const TfClass& cl = p.cls[tile_class(tile)];
        const int idx = (tile - cl.tile0) * 128 + row, per = cl.nr * cl.nc;
        if (idx >= p.B * per) return false;
        *b = idx / per;
        const int r2 = idx - *b * per, i = r2 / cl.nc, j = r2 - i * cl.nc;
        *rc = cl.cr + p.s * i;
        *cc = cl.ccl + 2 * p.s * j;
        *rem = *rc * p.Wout + *cc;
        return true;
    };

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if TF_PROF
    long long g_tf_prof_acc[16] = {0};
#endif
    if (warp == TF_MMA_WARP && lane == 0) {
        for (int s = 0; s < TF_STAGES; ++s) {
            ptx::mbar_init(&full[s], 4);   // the 4 builder warps of the group that wrote the stage
            ptx::mbar_init(&empty[s], ISS);  // tcgen05.commit of the stage's MMAs (each issuer)
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(&tfull[a], ISS);
            ptx::mbar_init(&tempty[a], TF_EPI_WARPS);
        }
        ptx::mbar_init(wbar, 1);
        ptx::fence_barrier_init();
        ptx::mbar_arrive_expect_tx(wbar, wbytes);
        constexpr uint32_t CH = 32768;
        for (uint32_t off = 0; off < wbytes; off += CH)
            bulk_g2s(wsm + off, reinterpret_cast<const uint8_t*>(wpack) + off, wbytes - off < CH ? wbytes - off : CH,
                     wbar);
    }
    if (warp == TF_MMA_WARP) ptx::tmem_alloc(tslot, TMEM_COLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = *tslot;

    if (warp >= TF_MMA_WARP) {
        // per K-step: D[0, 2NT) += A_hi . [B_hi ; B_lo]  (one N = 2 NT MMA: hi.hi and hi.lo side by side)
        //             D[0, NT)  += A_lo . B_hi
        // The whole warp runs this loop (its values stay warp-uniform) and an elected lane issues.  A tile's
        // last stage always issues TF_KPS K-steps: the builders write zeros into the A columns of K-steps
        // past the tile's count, and those K-steps read weight block 0 (finite), so they add exact zeros --
        // no per-MMA bounds test in the issue stream.
        // Issuer i (warp TF_MMA_WARP + i) takes K-steps kk = i, i + ISS, ... of every stage into its own
        // accumulator (slot acc, issuer i); the epilogue adds the issuers' accumulators.
        constexpr uint32_t idesc2 = idesc_tf32(128, 2 * NT), idesc1 = idesc_tf32(128, NT);
        const int iss = warp - TF_MMA_WARP;
        ptx::mbar_wait(wbar, 0);
        const uint64_t bdesc0 = desc_sw32(ptx::smem_u32(wsm));
        constexpr uint64_t BSTEP = (2 * KBLK) >> 4;  // descriptor address units (16 B)
        int sglob = 0, acc = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            ptx::mbar_wait(&tempty[acc], aphase ^ 1);
            ptx::tc_fence_after();
            const uint32_t d = tm + (acc * ISS + iss) * 2 * NT;
            int k0, kn;
            tile_k(tile, &k0, &kn);
            const int tst = (kn + TF_KPS - 1) / TF_KPS;
            uint64_t bd = bdesc0;
            for (int js = 0; js < tst; ++js, ++sglob) {
                const int st = sglob & (TF_STAGES - 1);
                PROF_T0();
                ptx::mbar_wait(&full[st], (sglob / TF_STAGES) & 1);
                PROF_ACC(0);
                ptx::tc_fence_after();
                const uint32_t a0 = tm + ACC_COLS + st * STAGE_COLS;
                const bool last = js + 1 == tst;
#pragma unroll
                for (int k2 = 0; k2 < TF_KPS / ISS; ++k2) {
                    const int kk = k2 * ISS + iss;
                    const int ks = js * TF_KPS + kk;
                    uint64_t b = bd + (uint64_t)kk * BSTEP;
                    if (IN_LAT) b = bdesc0 + (uint64_t)wtab[k0 + (ks < kn ? ks : 0)] * BSTEP;
                    else if (last && ks >= kn) b = bdesc0;
                    mma_tf32_ts_elect(d, a0 + 16 * kk, b, idesc2, (js | k2) ? 1u : 0u);
                    mma_tf32_ts_elect(d, a0 + 16 * kk + 8, b, idesc1, 1u);
                }
                bd += (uint64_t)TF_KPS * BSTEP;
                mma_commit_elect(&empty[st]);
                PROF_ACC(1);
            }
            mma_commit_elect(&tfull[acc]);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    } else if (warp >= TF_EPI_WARPS) {
        // builders: group g fills the A stages sglob = g (mod TF_GROUPS) -- every use of a TMEM stage
        // (sglob mod TF_STAGES) belongs to the same group, so its empty-barrier parity waits are never more
        // than one phase ahead.  A stage holds TF_KPS consecutive K-steps of one tile (the last stage of a
        // tile may hold fewer).  Warp quadrant q fills TMEM lanes 32q .. 32q+31 = pixels 32q .. 32q+31 of the
        // tile; all 8 * TF_KPS loads of a stage are issued before any is used.
        const int g = (warp - TF_EPI_WARPS) >> 2, q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const int hw_in = p.Hin * p.Win;
        int sglob = g, js = g, tile = blockIdx.x;
        while (tile < p.tiles && js >= tile_stages(tile)) {
            js -= tile_stages(tile);
            tile += gridDim.x;
        }
        int cur_tile = -1, pc = 0, rc = 0, cc = 0, k0 = 0, kn = 0;
        bool valid = false;
        const float* xb = p.x;
        for (; tile < p.tiles; sglob += TF_GROUPS) {
            if (tile != cur_tile) {
                cur_tile = tile;
                int b = 0, rem = 0;
                rc = cc = 0;
                valid = tile_pixel(tile, q * 32 + lane, &b, &rem, &rc, &cc);
                if (!valid) b = 0;
                pc = (cc + p.parity) & 1;
                xb = p.x + (size_t)b * p.Cx * hw_in;
                tile_k(tile, &k0, &kn);
            }
            PROF_T0();
            const int ks0 = js * TF_KPS;
            float v[TF_KPS][8];
#pragma unroll
            for (int kk = 0; kk < TF_KPS; ++kk) {
                const int ks = ks0 + kk;
                const bool in_k = ks < kn;
                const uint32_t e = ktab[k0 + (in_k ? ks : 0)];
                const int dc = (int8_t)(e & 0xFF), dr = (int8_t)((pc ? e >> 16 : e >> 8) & 0xFF);
                const int c0 = (int)(e >> 24) * 8;
                const int qr = rc + dr, qc = cc + dc;
                bool ok = in_k && valid && (unsigned)qr < (unsigned)p.H && (unsigned)qc < (unsigned)p.W;
                int idx = qr * p.Win + qc;
                if constexpr (IN_LAT) {  // the neighbour must be a centre of the stride-s lattice (dy lives there)
                    const int Cq = qc / p.s;
                    const int rr = qr - hex_rho(Cq, p.s, p.parity);
                    const int Rq = rr / p.s;
                    ok = ok && qc == Cq * p.s && rr >= 0 && rr == Rq * p.s && Rq < p.Hin && Cq < p.Win;
                    idx = Rq * p.Win + Cq;
                }
                // unconditional loads from a valid address (the image's first pixel when the neighbour is
                // off-grid or off-lattice), zeroed afterwards: no predicated loads in the hot loop
                // channel k of the chunk is k plane strides (p.plane_bytes, a kernel parameter) past the first:
                // the 8 offsets are warp-uniform, so each load is one LDG [base + uniform offset]
                const char* src = reinterpret_cast<const char*>(xb + (ok ? idx : 0) + c0 * hw_in);
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float* sk = reinterpret_cast<const float*>(src + (int64_t)k * p.plane_bytes);
                    float u;
                    if constexpr (FULLCH) {
                        u = __ldg(sk);
                    } else {
                        u = c0 + k < p.Cx ? __ldg(sk) : 0.f;
                    }
                    v[kk][k] = ok ? u : 0.f;
                }
            }
            PROF_ACC(4);
            const int st = sglob & (TF_STAGES - 1);
            ptx::mbar_wait(&empty[st], ((sglob / TF_STAGES) & 1) ^ 1);
            PROF_ACC(6);
            ptx::tc_fence_after();
            const uint32_t ta = tm + lane_base + ACC_COLS + st * STAGE_COLS;
#pragma unroll
            for (int kk = 0; kk < TF_KPS; ++kk) {
                uint32_t hi[8], lo[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float h = tf32_rna(v[kk][k]);
                    hi[k] = __float_as_uint(h);
                    lo[k] = __float_as_uint(v[kk][k] - h);
                }
                tmem_st8(ta + 16 * kk, hi);
                tmem_st8(ta + 16 * kk + 8, lo);
            }
            tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&full[st]);
            PROF_ACC(7);
            js += TF_GROUPS;
            while (tile < p.tiles && js >= tile_stages(tile)) {
                js -= tile_stages(tile);
                tile += gridDim.x;
            }
        }
    } else {
        // epilogue: warp q drains TMEM lanes 32q .. 32q+31 (its 32 pixels): out = D[c] + D[NT + c]
        const int q = warp;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const int hw_out = p.Hout * p.Wout;
        int acc = 0;
        uint32_t aphase = 0;
        for (int tile = blockIdx.x; tile < p.tiles; tile += gridDim.x) {
            PROF_T0();
            ptx::mbar_wait(&tfull[acc], aphase);
            PROF_ACC(10);
            ptx::tc_fence_after();
            int b = 0, rem = 0, rcx, ccx;
            const bool vpix = tile_pixel(tile, q * 32 + lane, &b, &rem, &rcx, &ccx);
            float* yo = p.y + (size_t)b * p.Nout * hw_out + rem;
            const float* mo = p.relu_y ? p.relu_y + (size_t)b * p.Nout * hw_out + rem : nullptr;
            const uint32_t dbase = tm + lane_base + acc * ISS * 2 * NT;
#pragma unroll
            for (int c0 = 0; c0 < NT; c0 += 16) {
                uint32_t u[16], w[16];
                tmem_ld16(dbase + c0, u);
                tmem_ld16(dbase + NT + c0, w);
                if constexpr (ISS == 2) {
                    uint32_t u2[16], w2[16];
                    tmem_ld16(dbase + 2 * NT + c0, u2);
                    tmem_ld16(dbase + 3 * NT + c0, w2);
                    ptx::tmem_ld_wait();
#pragma unroll
                    for (int j = 0; j < 16; ++j) {  // fixed order: (hh + lh + hl of issuer 0) + (... of issuer 1)
                        u[j] = __float_as_uint((__uint_as_float(u[j]) + __uint_as_float(w[j])) +
                                               (__uint_as_float(u2[j]) + __uint_as_float(w2[j])));
                        w[j] = 0u;
                    }
                }
                ptx::tmem_ld_wait();
                if (c0 + 16 >= NT) {  // the accumulator is drained: hand it back to the MMA warp
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&tempty[acc]);
                }
                if (vpix) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int c = c0 + j;
                        if (c < p.Nout) {
                            float o = __uint_as_float(u[j]) + __uint_as_float(w[j]);
                            if (p.bias) o += __ldg(p.bias + c);
                            if (p.relu) o = fmaxf(o, 0.f);
                            if (mo && !(__ldg(mo + (size_t)c * hw_out) > 0.f)) o = 0.f;
                            yo[(size_t)c * hw_out] = o;
                        }
                    }
                }
            }
            PROF_ACC(11);
            acc ^= 1;
            if (acc == 0) aphase ^= 1;
        }
    }
#if TF_PROF
    if (blockIdx.x == 0 && lane == 0 && (warp == TF_MMA_WARP || warp == TF_EPI_WARPS || warp == 0))
        for (int i = 0; i < 16; ++i)
            if (g_tf_prof_acc[i]) g_tf_prof[i] = g_tf_prof_acc[i];
#endif
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == TF_MMA_WARP) ptx::tmem_dealloc(tm, TMEM_COLS);
}

// Weights -> [K-step][hi|lo][NT rows][8] fp32 in the SW32 K-major layout the MMA reads.
//   forward : row n = co, K-step (t, c8), k -> ci = 8 c8 + k :  w[co][ci][t]
//   bwd-data: row n = ci, K-step (t, c8), k -> co = 8 c8 + k :  w[co][ci][T-1-t]   (pin P18)
__global__ void tf32_pack_kernel(const float* __restrict__ w, float* __restrict__ wp, int Cout, int Cin, int T,
                                 int NT, int kc8, int ksteps, int transpose) {
    const int total = ksteps * 2 * NT * 8;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < total; e += gridDim.x * blockDim.x) {
        const int k = e & 7, n = (e >> 3) % NT, half = (e / (8 * NT)) & 1, ks = e / (16 * NT);
        const int t = ks / kc8, ch = (ks - t * kc8) * 8 + k;
        float v = 0.f;
        if (!transpose) {
            if (n < Cout && ch < Cin) v = w[((size_t)n * Cin + ch) * T + t];
        } else {
            if (n < Cin && ch < Cout) v = w[((size_t)ch * Cin + n) * T + (T - 1 - t)];
        }
        const float hi = tf32_rna(v);
        const float out = half ? v - hi : hi;
        const int off = ks * 2 * NT * 8 + half * NT * 8 + n * 8 + (((k >> 2) ^ ((n >> 2) & 1)) << 2) + (k & 3);
        wp[off] = out;
    }
}

struct TfPlan {
    int NT, kc8, ksteps, smem;
    bool ok;
};
TfPlan tf_plan(const Geom& g, int Cx, int Nout) {
    TfPlan pl{};
    if (g.T > TF_MAXT || Cx < 1 || Nout < 1) return pl;
    pl.NT = (Nout + 15) / 16 * 16;
    if (pl.NT > TF_MAX_NT) return pl;
    pl.kc8 = (Cx + 7) / 8;
    pl.ksteps = g.T * pl.kc8;
    pl.smem = pl.ksteps * 2 * pl.NT * 32 + 1024 + 256 + 4 * pl.ksteps;
    pl.ok = pl.smem <= TF_SMEM_MAX;
    return pl;
}

template <int NT, bool IN_LAT, bool FULLCH>
hex_status_t launch_tf_k(const TfParams& p, const float* wpack, int smem, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(tf32_conv_kernel<NT, IN_LAT, FULLCH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 TF_SMEM_MAX) != cudaSuccess)
            return HEX_ERR_CUDA;
        attr = true;
    }
    const int grid = p.tiles < num_sms() ? p.tiles : num_sms();
    tf32_conv_kernel<NT, IN_LAT, FULLCH><<<grid, tf_threads(tf_issuers(NT)), smem, st>>>(p, wpack);
    count_launch();
    return last_launch_status();
}

template <int NT>
hex_status_t launch_tf(const TfParams& p, const float* wpack, int smem, cudaStream_t st) {
    const bool full = (p.Cx & 7) == 0;
    if (p.in_lat) return full ? launch_tf_k<NT, true, true>(p, wpack, smem, st) : launch_tf_k<NT, true, false>(p, wpack, smem, st);
    return full ? launch_tf_k<NT, false, true>(p, wpack, smem, st) : launch_tf_k<NT, false, false>(p, wpack, smem, st);
}

}  // namespace

// Which fp32 NCHW convolutions run on the 3xTF32 tensor-core kernel: enough input channels to fill a K-step
// (Cx >= 8), <= 64 output channels, n <= 3, weights resident in shared memory.  HEXCONV_NO_TF32 forces the
// FFMA kernels.
bool tf32_conv_supported(const Geom& g, int Cx, int Nout, int dtype, int layout) {
    if (dtype != HEX_F32 || layout != HEX_NCHW || Cx < 8 || sw_on("HEXCONV_NO_TF32")) return false;
    return tf_plan(g, Cx, Nout).ok;
}

size_t tf32_conv_ws_bytes(const Geom& g, int Cx, int Nout) {
    const TfPlan pl = tf_plan(g, Cx, Nout);
    return pl.ok ? (size_t)pl.ksteps * 2 * pl.NT * 32 + 256 : 0;
}

// mode 0: forward of x [B][Cin][H][W] -> y [B][Cout][Ho][Wo];  mode 1: bwd-data of dy [B][Cout][Ho][Wo] ->
// dx [B][Cin][H][W] (masked by relu_y > 0 when given).  ws holds the packed weights.
hex_status_t tf32_conv(const Geom& g, int Cin, int Cout, int mode, const float* in, const float* w,
                       const float* bias, const float* relu_y, int relu, float* out, void* ws, size_t ws_bytes,
                       cudaStream_t st) {
    const int Cx = mode ? Cout : Cin, Nout = mode ? Cin : Cout;
    const TfPlan pl = tf_plan(g, Cx, Nout);
    if (!pl.ok) return HEX_ERR_UNSUPPORTED;
    const size_t need = (size_t)pl.ksteps * 2 * pl.NT * 32;
    if (!ws || ws_bytes < need + 256) return HEX_ERR_WORKSPACE;
    float* wp = reinterpret_cast<float*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    {
        const int total = pl.ksteps * 2 * pl.NT * 8;
        tf32_pack_kernel<<<ceil_div(total, 256), 256, 0, st>>>(w, wp, Cout, Cin, g.T, pl.NT, pl.kc8, pl.ksteps, mode);
        count_launch();
        if (last_launch_status() != HEX_OK) return HEX_ERR_CUDA;
    }
    TfParams p{};
    p.x = in;
    p.bias = mode ? nullptr : bias;
    p.relu_y = relu_y;
    p.y = out;
    p.Cx = Cx;
    p.H = g.H;
    p.W = g.W;
    if (mode == 0) {
        p.Hin = g.H; p.Win = g.W; p.Hout = g.Ho; p.Wout = g.Wo;
        p.out_lat = g.s > 1; p.in_lat = 0;
    } else {
        p.Hin = g.Ho; p.Win = g.Wo; p.Hout = g.H; p.Wout = g.W;
        p.out_lat = 0; p.in_lat = g.s > 1;
    }
    p.plane_bytes = (int64_t)p.Hin * p.Win * 4;
    p.Nout = Nout;
    p.s = g.s;
    p.parity = g.parity;
    p.T = g.T;
    p.kc8 = pl.kc8;
    p.ksteps = pl.ksteps;
    p.relu = mode ? 0 : relu;
    p.B = g.B;
    p.total_pix = g.B * p.Hout * p.Wout;
    p.tiles = ceil_div(p.total_pix, 128);
    for (int t = 0; t < g.T; ++t) {
        int dc, dr0, dr1;
        tap_offset(g.n, 0, t, &dc, &dr0);
        tap_offset(g.n, 1, t, &dc, &dr1);
        p.dc[t] = (int8_t)dc;
        p.dr0[t] = (int8_t)dr0;
        p.dr1[t] = (int8_t)dr1;
    }
    int smem = pl.smem;
    if (p.in_lat) {
        // phase classes (r mod s, c mod 2s): the taps whose neighbour q = y + off_t(y) is a lattice centre
        // depend only on the class (q's column parity mod s, its rho(C) (period 2 in C) and its row mod s);
        // decided on a representative pixel far from the borders (the borders are checked per pixel)
        const int s = g.s;
        int nk = 0, tile0 = 0;
        p.ncls = 0;
        for (int cr = 0; cr < s; ++cr)
            for (int ccl = 0; ccl < 2 * s; ++ccl) {
                const int nr = cr < g.H ? (g.H - cr + s - 1) / s : 0, nc = ccl < g.W ? (g.W - ccl + 2 * s - 1) / (2 * s) : 0;
                if (nr * nc == 0) continue;
                TfClass& cl = p.cls[p.ncls++];
                cl.cr = cr;
                cl.ccl = ccl;
                cl.nr = nr;
                cl.nc = nc;
                cl.tile0 = tile0;
                cl.k0 = nk;
                const int r_rep = cr + 8 * s, c_rep = ccl + 16 * s, pc = (c_rep + g.parity) & 1;
                for (int t = 0; t < g.T; ++t) {
                    const int qc = c_rep + p.dc[t], qr = r_rep + (pc ? p.dr1[t] : p.dr0[t]);
                    if (qc % s) continue;
                    if ((qr - hex_rho(qc / s, s, g.parity)) % s) continue;
                    for (int c8 = 0; c8 < pl.kc8; ++c8) {
                        if (nk >= TF_MAXKL) return HEX_ERR_UNSUPPORTED;
                        p.klist[nk++] = (uint16_t)(t | (c8 << 8));
                    }
                }
                cl.kn = nk - cl.k0;
                if (cl.kn == 0) {  // no tap reaches a lattice centre: the class's dx is all zero, but it still
                    p.klist[nk++] = (uint16_t)0;  // needs one (zero-contributing) K-step to write its tile
                    cl.kn = 1;
                }
                tile0 += ceil_div((int64_t)g.B * nr * nc, 128);
            }
        p.tiles = tile0;
        smem += 6 * nk + 16;
        if (smem > TF_SMEM_MAX) return HEX_ERR_UNSUPPORTED;
    } else {
        p.ncls = 0;
        smem += 2 * pl.ksteps + 16;
    }
    switch (pl.NT) {
        case 16: return launch_tf<16>(p, wp, smem, st);
        case 32: return launch_tf<32>(p, wp, smem, st);
        case 48: return launch_tf<48>(p, wp, smem, st);
        case 64: return launch_tf<64>(p, wp, smem, st);
    }
    return HEX_ERR_UNSUPPORTED;
}


// ====================================================================================================
// Weight gradient (+ dbias) in 3xTF32:  dW[co][ci][t] = sum_{b,o} dy[b][co][o] * x[b][ci][centre(o) + off_t]
// (the adjoint of the forward with respect to the weights).
//
// GEMM view: M = (ci, t) rows (m = ci * T + t, up to 3 M-tiles of 128), N = Cout (padded to 16, <= 64),
// K = output pixels.  A K-step is 8 consecutive output pixels of one output row (b, R): C0 .. C0+7.
//   * The x rows an output row needs (all Cin channels, every tap's row, W + 2n columns with zero halo)
//     are staged as one TMA box per output row ("band", OOB rows / columns zero-filled), double-buffered.
//     The box's rows x columns are padded so that one channel plane is 4 x odd words: the 32 lanes of a
//     warp (32 (t, ci) rows) then spread over the banks (16 channels of a plane-multiple-of-16 box sat on
//     2 banks).
//   * A builders (one thread per TMEM lane = per (t, ci) row, two groups alternating K-steps) read their
//     8 values from the band -- two base addresses per K-step (the two column parities of the centres)
//     plus compile-time offsets -- split them hi / lo and tcgen05.st them.
//   * The same group's first 2 Cout threads load dy[b][co][R][C0 .. C0+7] (two threads per output
//     channel, one K-step ahead), split it and write the K-major SW32 hi / lo block to shared memory
//     (fence.proxy.async before signalling), keeping the dbias partial sums.
//   * Per K-step and M-tile: D += A_hi . [B_hi ; B_lo] (N = 2 Cout) and D += A_lo . B_hi (N = Cout).
//   * Split-K: CTA c takes a contiguous range of output rows; it writes its partial dW [co][m] and dbias
//     to the workspace, and a fixed-order reduction kernel sums the partials (deterministic).
namespace {

constexpr int WG_G = 2;   // A-builder groups (K-steps alternate)
constexpr int WG_HL = 4;  // left halo columns of a band (16 bytes: TMA needs the innermost start 16-byte aligned)

struct WgParams {
    const float* dy;      // [B][Cout][Ho][Wo]
    float* part;          // [grid][Cout][Mrows] partial dW
    float* part_b;        // [grid][Cout] partial dbias
    int Cin, Cout, H, W, Ho, Wo, s, parity, n, T, Mrows;
    int rows, rows_per_cta, cblk;  // output rows B*Ho, per CTA, K-steps per output row
    int rmin, NR, BW;              // band: input rows s*R + rmin .. + NR - 1, columns -WG_HL .. BW - WG_HL - 1

    int8_t dc[TF_MAXT], dr0[TF_MAXT], dr1[TF_MAXT];
    int dbg;  // development probe only (TF_PROF builds): bit 0 no MMA, 1 no tcgen05.st, 2 no TMA, 3 no tcgen05.ld
};
#if TF_PROF
#define WG_SKIP(bit) (p.dbg & (1 << (bit)))
#else
#define WG_SKIP(bit) false
#endif

template <int NT, int MT>
struct WgCfg {
    static constexpr int AWARPS = 4 * MT * WG_G;           // A builders
    static constexpr int TWARP = 4 + AWARPS;               // TMA (x bands)
    static constexpr int MWARP = TWARP + 1;                // MMA issue
    static constexpr int THREADS = (MWARP + 1) * 32;
    static constexpr int ACC = MT * 2 * NT;                // accumulators
    static constexpr int STAGES = (ACC + 4 * MT * 16 <= 512) ? 4 : 2;
    static constexpr int TCOLS = (ACC + STAGES * MT * 16) <= 256 ? 256 : 512;
    static constexpr int BBYTES = 2 * NT * 32;             // one stage's B block (hi | lo)
};

template <int NT, int MT, int S>
__global__ void __launch_bounds__(WgCfg<NT, MT>::THREADS, 1)
tf32_wgrad_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ WgParams p) {
    using Cfg = WgCfg<NT, MT>;
    constexpr int STAGES = Cfg::STAGES;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* base = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* bsm = base;                                             // STAGES x B blocks (1024-aligned)
    float* band = reinterpret_cast<float*>(base + STAGES * Cfg::BBYTES);
    const int band_elems = (p.Cin * p.NR * p.BW + 31) & ~31;  // buffer pitch: 128-byte aligned TMA destinations
    uint64_t* bars = reinterpret_cast<uint64_t*>(band + 2 * band_elems);
    uint64_t* full = bars;               // STAGES
    uint64_t* empty = full + STAGES;     // STAGES
    uint64_t* xfull = empty + STAGES;    // 2
    uint64_t* xempty = xfull + 2;        // 2
    uint64_t* dfull = xempty + 2;        // 1
    uint32_t* tslot = reinterpret_cast<uint32_t*>(dfull + 1);
    float* bpart = reinterpret_cast<float*>(tslot + 4);  // [WG_G][2 NT] dbias partial sums

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
#if TF_PROF
    long long g_tf_prof_acc[16] = {0};
#endif
    const int row0 = blockIdx.x * p.rows_per_cta;
    const int row1 = min(p.rows, row0 + p.rows_per_cta);
    const int nrows = max(0, row1 - row0);
    const int nk = nrows * p.cblk;  // K-steps of this CTA
    if (warp == Cfg::MWARP && lane == 0) {
        for (int st = 0; st < STAGES; ++st) {
            ptx::mbar_init(&full[st], 4 * MT);  // the owning group's warps (A in TMEM, B in smem)
            ptx::mbar_init(&empty[st], 1);
        }
        for (int b = 0; b < 2; ++b) {
            ptx::mbar_init(&xfull[b], 1);
            ptx::mbar_init(&xempty[b], Cfg::AWARPS);
        }
        ptx::mbar_init(dfull, 1);
        ptx::fence_barrier_init();
    }
    if (warp == Cfg::MWARP) ptx::tmem_alloc(tslot, Cfg::TCOLS);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tm = *tslot;
    const int hwo = p.Ho * p.Wo;
    (void)hwo;

    if (warp == Cfg::TWARP) {
        if (lane == 0) {
            ptx::prefetch_tmap(&map_x);
            for (int r = 0; r < nrows; ++r) {
                const int buf = r & 1;
                ptx::mbar_wait(&xempty[buf], ((r >> 1) & 1) ^ 1);
                const int row = row0 + r, b = row / p.Ho, R = row - b * p.Ho;
                ptx::mbar_arrive_expect_tx(&xfull[buf], (uint32_t)(p.Cin * p.NR * p.BW) * 4u);
                ptx::tma_load_4d(&map_x, &xfull[buf], band + buf * band_elems, -WG_HL, p.s * R + p.rmin, 0, b);
            }
        }
    } else if (warp == Cfg::MWARP) {
        // the whole warp runs the issue loop (warp-uniform values), one elected lane issues
        constexpr uint32_t idesc2 = idesc_tf32(128, 2 * NT), idesc1 = idesc_tf32(128, NT);
        const uint64_t b0 = desc_sw32(ptx::smem_u32(bsm));
        for (int kg = 0; kg < nk; ++kg) {
            const int st = kg % STAGES;
            PROF_T0();
            ptx::mbar_wait(&full[st], (kg / STAGES) & 1);
            PROF_ACC(0);
            ptx::tc_fence_after();
            const uint64_t bd = b0 + (uint64_t)((st * Cfg::BBYTES) >> 4);
#pragma unroll
            for (int mt = 0; mt < MT; ++mt) {
                const uint32_t d = tm + mt * 2 * NT;
                const uint32_t a = tm + Cfg::ACC + (st * MT + mt) * 16;
                if (WG_SKIP(0)) continue;
                mma_tf32_ts_elect(d, a, bd, idesc2, kg > 0 ? 1u : 0u);
                mma_tf32_ts_elect(d, a + 8, bd, idesc1, 1u);
            }
            mma_commit_elect(&empty[st]);
            PROF_ACC(1);
        }
        mma_commit_elect(dfull);
    } else if (warp >= 4) {
        // A builders: warp index within the group -> (M-tile, lane quadrant = warp % 4).  Row m = ci * T + t
        // (channel-major: the 32 lanes of a warp are mostly the taps of one channel, whose band addresses
        // differ by the tap offsets -- spread over the banks -- instead of 16 channel planes 4 x odd words
        // apart).
        const int wi = warp - 4, g = wi / (4 * MT), wg = wi - g * 4 * MT;
        const int mt = wg >> 2, q = warp & 3;
        const uint32_t lane_base = (uint32_t)(q * 32) << 16;
        const int m = mt * 128 + q * 32 + lane;
        const bool mvalid = m < p.Mrows;
        const int ci = mvalid ? m / p.T : 0, t = mvalid ? m - ci * p.T : 0;
        const int ss = S ? S : p.s;
        // band offsets of this row's 8 values, per centre-column parity cp of C = C0 + cp (C0 is a multiple of
        // 8 and rho has period 2, so they do not depend on C0 beyond the + ss * C0 column shift):
        //   value k of a K-step sits at  off[k & 1] + ss * (C0 + k)
        int off[2];
#pragma unroll
        for (int cp = 0; cp < 2; ++cp) {
            const int pc = (ss * cp + p.parity) & 1;
            const int srow = hex_rho(cp, ss, p.parity) + (pc ? p.dr1[t] : p.dr0[t]) - p.rmin;
            off[cp] = ci * p.NR * p.BW + srow * p.BW + p.dc[t] + WG_HL;
        }
        // B role: thread bi of the group (bi < 2 NT) loads dy[b][co = bi / 2][R][C0 + 4 (bi & 1) .. + 3] of the
        // group's K-steps, one K-step ahead, splits it and writes its half row of the SW32 hi / lo blocks;
        // it also sums those dy values for dbias
        const int bi = wg * 32 + lane, bn = bi >> 1, bh = bi & 1;
        const bool brole = bi < 2 * NT, bload_ok = brole && bn < p.Cout;
        const bool vec = (p.Wo & 3) == 0 && ((uintptr_t)p.dy & 15) == 0;
        const int boff = bn * 32 + ((bh ^ ((bn >> 2) & 1)) << 4);  // SW32 chunk of this thread's half row
        float bsum = 0.f;
        // the group's K-steps kg = g, g + WG_G, ...: (row r, column block j) walked without division
        int r = 0, j = g;
        while (j >= p.cblk && r < nrows) { j -= p.cblk; ++r; }
        auto dy_row = [&](int rr) -> const float* {
            const int row = row0 + rr, b = row / p.Ho, R = row - b * p.Ho;
            return p.dy + ((size_t)(b * p.Cout + (bload_ok ? bn : 0)) * p.Ho + R) * p.Wo + 4 * bh;
        };
        auto bload = [&](const float* rowp, int C0, float* v) {
            v[0] = v[1] = v[2] = v[3] = 0.f;
            if (!bload_ok) return;
            const float* src = rowp + C0;
            if (vec && C0 + 4 * bh + 4 <= p.Wo) {
                const float4 a = __ldg(reinterpret_cast<const float4*>(src));
                v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
            } else {
#pragma unroll
                for (int k = 0; k < 4; ++k) v[k] = C0 + 4 * bh + k < p.Wo ? __ldg(src + k) : 0.f;
            }
        };
        float bnext[4] = {0.f, 0.f, 0.f, 0.f};
        if (r < nrows) bload(dy_row(r), j * 8, bnext);
        int cur_r = -1;
        const float* bx = band;
        for (int kg = g; r < nrows; kg += WG_G) {
            PROF_T0();
            if (r != cur_r) {  // entering row r: release the bands of the rows passed, wait for row r's
                // (a row is released only after its band was seen loaded, so an arrival always counts toward
                // that row's phase of the empty barrier -- also for rows this group had no K-step in)
                for (int rr = cur_r < 0 ? 0 : cur_r; rr < r; ++rr) {
                    if (rr > cur_r) ptx::mbar_wait(&xfull[rr & 1], (rr >> 1) & 1);
                    __syncwarp();
                    if (lane == 0) ptx::mbar_arrive(&xempty[rr & 1]);
                }
                ptx::mbar_wait(&xfull[r & 1], (r >> 1) & 1);
                PROF_ACC(6);
                cur_r = r;
                bx = band + (r & 1) * band_elems;
            }
            const int C0 = j * 8;
            const int nv = min(8, p.Wo - C0);
            uint32_t hi[8], lo[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float u = (mvalid && k < nv) ? bx[off[k & 1] + ss * (C0 + k)] : 0.f;
                const float h = tf32_rna(u);
                hi[k] = __float_as_uint(h);
                lo[k] = __float_as_uint(u - h);
            }
            // advance to the group's next K-step and prefetch its dy
            int nr = r, nj = j + WG_G;
            while (nj >= p.cblk && nr < nrows) { nj -= p.cblk; ++nr; }
            float bv[4] = {bnext[0], bnext[1], bnext[2], bnext[3]};
            if (nr < nrows) bload(dy_row(nr), nj * 8, bnext);
            const int st = kg % STAGES;
            PROF_ACC(7);
            ptx::mbar_wait(&empty[st], ((kg / STAGES) & 1) ^ 1);
            PROF_ACC(8);
            ptx::tc_fence_after();
            const uint32_t ta = tm + lane_base + Cfg::ACC + (st * MT + mt) * 16;
            if (!WG_SKIP(1)) {
                tmem_st8(ta, hi);
                tmem_st8(ta + 8, lo);
            }
            if (brole) {
                float bhv[4], blv[4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    bsum += bv[k];
                    bhv[k] = tf32_rna(bv[k]);
                    blv[k] = bv[k] - bhv[k];
                }
                uint8_t* blk = bsm + st * Cfg::BBYTES;
                *reinterpret_cast<float4*>(blk + boff) = make_float4(bhv[0], bhv[1], bhv[2], bhv[3]);
                *reinterpret_cast<float4*>(blk + NT * 32 + boff) = make_float4(blv[0], blv[1], blv[2], blv[3]);
                ptx::fence_proxy_async();  // generic-proxy smem writes -> visible to the tensor core
            }
            if (!WG_SKIP(1)) tmem_st_wait();
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&full[st]);
            PROF_ACC(9);
            r = nr;
            j = nj;
        }
        // release the bands of the remaining rows (including ones this group had no K-step in)
        for (int rr = cur_r < 0 ? 0 : cur_r; rr < nrows; ++rr) {
            if (rr > cur_r) ptx::mbar_wait(&xfull[rr & 1], (rr >> 1) & 1);
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(&xempty[rr & 1]);
        }
        if (brole) bpart[g * 2 * NT + bi] = bsum;
    } else {
        // epilogue (warps 0-3): D rows of lane quadrant q -> partial [co][m] = D[c] + D[NT + c]
        const int q = warp;
        ptx::mbar_wait(dfull, 0);
        ptx::tc_fence_after();
#pragma unroll
        for (int mt = 0; mt < MT; ++mt) {
            const int m = mt * 128 + q * 32 + lane;
            const uint32_t dbase = tm + ((uint32_t)(q * 32) << 16) + mt * 2 * NT;
#pragma unroll
            for (int c0 = 0; c0 < NT; c0 += 16) {
                uint32_t u[16] = {}, w[16] = {};
                if (!WG_SKIP(3)) {
                    tmem_ld16(dbase + c0, u);
                    tmem_ld16(dbase + NT + c0, w);
                    ptx::tmem_ld_wait();
                }
                if (m < p.Mrows) {
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const int co = c0 + j;
                        if (co < p.Cout)
                            p.part[((size_t)blockIdx.x * p.Cout + co) * p.Mrows + m] =
                                nk ? __uint_as_float(u[j]) + __uint_as_float(w[j]) : 0.f;
                    }
                }
            }
        }
    }
#if TF_PROF
    if (blockIdx.x == 0 && lane == 0 && (warp == Cfg::MWARP || warp == 4))
        for (int i = 0; i < 16; ++i)
            if (g_tf_prof_acc[i]) g_tf_prof[16 + i] = g_tf_prof_acc[i];
#endif
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == Cfg::MWARP) ptx::tmem_dealloc(tm, Cfg::TCOLS);
    if (warp == 0) {  // dbias partial of this CTA: the B threads' sums in fixed order
        for (int co = lane; co < p.Cout; co += 32) {
            float acc = 0.f;
            for (int gg = 0; gg < WG_G; ++gg) acc += bpart[gg * 2 * NT + 2 * co] + bpart[gg * 2 * NT + 2 * co + 1];
            p.part_b[(size_t)blockIdx.x * p.Cout + co] = nk ? acc : 0.f;
        }
    }
}

// dw[co][ci][t] (+)= sum_c part[c][co][ci * T + t]; dbias[co] (+)= sum_c part_b[c][co]  (fixed order)
__global__ void tf32_wgrad_reduce_kernel(const float* __restrict__ part, const float* __restrict__ part_b, int nparts,
                                         int Cout, int Cin, int T, float* __restrict__ dw, float* __restrict__ dbias,
                                         int accumulate) {
    // 8 lanes per output: lane l sums the partials c = l (mod 8), then a fixed shuffle tree (deterministic)
    const int Mrows = T * Cin;
    const int total = Cout * Mrows;
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    const int e = gid >> 3, l = gid & 7;
    const bool is_db = e >= total;
    const float* src = is_db ? part_b : part;
    const int stride = is_db ? Cout : total, off = is_db ? e - total : e;
    float s = 0.f;
    if (e < total + Cout) {
#pragma unroll 4
        for (int c = l; c < nparts; c += 8) s += src[(size_t)c * stride + off];
    }
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (l != 0 || e >= total + Cout) return;
    if (!is_db) {
        float* o = dw + (size_t)e;  // e = co * Mrows + ci * T + t: dw's own [co][ci][t] order
        *o = accumulate ? *o + s : s;
    } else if (dbias) {
        dbias[off] = accumulate ? dbias[off] + s : s;
    }
}

struct WgPlan {
    int NT, MT, grid, rows_per_cta, cblk, rmin, NR, BW, smem;
    bool ok;
};
WgPlan wg_plan(const Geom& g, int Cin, int Cout) {
    WgPlan pl{};
    if (g.T > TF_MAXT || Cin < 1 || Cout < 1 || g.n > 3) return pl;
    pl.NT = (Cout + 15) / 16 * 16;
    const int Mrows = g.T * Cin;
    pl.MT = (Mrows + 127) / 128;
    if (pl.NT > TF_MAX_NT || pl.MT > 3) return pl;
    // band rows: s*R + min/max over the two centre-column parities of (rho(C) + dr)
    int mn = 1 << 20, mx = -(1 << 20);
    for (int cp = 0; cp < 2; ++cp) {
        const int rho = hex_rho(cp, g.s, g.parity), pc = (g.s * cp + g.parity) & 1;
        for (int t = 0; t < g.T; ++t) {
            int dc, dr;
            tap_offset(g.n, pc, t, &dc, &dr);
            mn = std::min(mn, rho + dr);
            mx = std::max(mx, rho + dr);
        }
    }
    pl.rmin = mn;
    // box rows x columns (columns a multiple of 4: 16-byte TMA rows) padded until one channel plane is
    // 4 x odd words (bank spread of the 32 (t, ci) lanes of a warp)
    pl.NR = mx - mn + 1;
    pl.BW = (g.W + WG_HL + g.n + 3) / 4 * 4;
    for (int tries = 0; tries < 16 && ((pl.NR * pl.BW) % 8) != 4; ++tries) {
        if (tries & 1) ++pl.NR; else pl.BW += 4;
    }
    if (pl.BW > 256 || pl.NR > 256 || Cin > 256) return pl;
    pl.cblk = (g.Wo + 7) / 8;
    const int rows = g.B * g.Ho;
    pl.grid = std::min(rows, num_sms());
    pl.rows_per_cta = (rows + pl.grid - 1) / pl.grid;
    pl.grid = (rows + pl.rows_per_cta - 1) / pl.rows_per_cta;
    const int stages = (pl.MT * 2 * pl.NT + 4 * pl.MT * 16 <= 512) ? 4 : 2;
    pl.smem = 1024 + stages * 2 * pl.NT * 32 + 2 * ((Cin * pl.NR * pl.BW + 31) & ~31) * 4 + 256 + WG_G * 2 * pl.NT * 4;
    pl.ok = pl.smem <= TF_SMEM_MAX && (g.W * 4) % 16 == 0;  // TMA: 16-byte multiple row pitch of x
    return pl;
}

template <int NT, int MT, int S>
hex_status_t launch_wg_k(const CUtensorMap& mx, const WgParams& p, int grid, int smem, cudaStream_t st) {
    static bool attr = false;
    if (!attr) {
        if (cudaFuncSetAttribute(tf32_wgrad_kernel<NT, MT, S>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 TF_SMEM_MAX) != cudaSuccess)
            return HEX_ERR_CUDA;
        attr = true;
    }
    tf32_wgrad_kernel<NT, MT, S><<<grid, WgCfg<NT, MT>::THREADS, smem, st>>>(mx, p);
    count_launch();
    return last_launch_status();
}

template <int NT, int MT>
hex_status_t launch_wg_s(const CUtensorMap& mx, const WgParams& p, int grid, int smem, cudaStream_t st) {
    if (p.s == 1) return launch_wg_k<NT, MT, 1>(mx, p, grid, smem, st);
    if (p.s == 2) return launch_wg_k<NT, MT, 2>(mx, p, grid, smem, st);
    return launch_wg_k<NT, MT, 0>(mx, p, grid, smem, st);
}

template <int NT>
hex_status_t launch_wg_m(const CUtensorMap& mx, const WgParams& p, int MT, int grid, int smem, cudaStream_t st) {
    switch (MT) {
        case 1: return launch_wg_s<NT, 1>(mx, p, grid, smem, st);
        case 2: return launch_wg_s<NT, 2>(mx, p, grid, smem, st);
        case 3: return launch_wg_s<NT, 3>(mx, p, grid, smem, st);
    }
    return HEX_ERR_UNSUPPORTED;
}

}  // namespace

bool tf32_wgrad_supported(const Geom& g, int Cin, int Cout, int dtype, int layout) {
    if (dtype != HEX_F32 || layout != HEX_NCHW || Cin < 8 || sw_on("HEXCONV_NO_TF32")) return false;
    return wg_plan(g, Cin, Cout).ok;
}

size_t tf32_wgrad_ws_bytes(const Geom& g, int Cin, int Cout) {
    const WgPlan pl = wg_plan(g, Cin, Cout);
    if (!pl.ok) return 0;
    return (size_t)pl.grid * Cout * (g.T * Cin + 1) * sizeof(float) + 512;
}

hex_status_t tf32_wgrad(const Geom& g, int Cin, int Cout, const float* x, const float* dy, float* dw, float* dbias,
                        int accumulate, void* ws, size_t ws_bytes, cudaStream_t st, int dbg) {
    const WgPlan pl = wg_plan(g, Cin, Cout);
    if (!pl.ok) return HEX_ERR_UNSUPPORTED;
    const size_t need = (size_t)pl.grid * Cout * (g.T * Cin + 1) * sizeof(float) + 512;
    if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
    float* part = reinterpret_cast<float*>(((uintptr_t)ws + 255) & ~(uintptr_t)255);
    float* part_b = part + (size_t)pl.grid * Cout * g.T * Cin;
    static PFN_cuTensorMapEncodeTiled_v12000 enc = nullptr;
    if (!enc) {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            enc = (PFN_cuTensorMapEncodeTiled_v12000)ptr;
    }
    if (!enc) return HEX_ERR_CUDA;
    if ((uintptr_t)x & 15) return HEX_ERR_ALIGNMENT;  // TMA global address
    CUtensorMap mx;
    cuuint64_t dims[4] = {(cuuint64_t)g.W, (cuuint64_t)g.H, (cuuint64_t)Cin, (cuuint64_t)g.B};
    cuuint64_t strides[3] = {(cuuint64_t)g.W * 4, (cuuint64_t)g.H * g.W * 4, (cuuint64_t)Cin * g.H * g.W * 4};
    cuuint32_t box[4] = {(cuuint32_t)pl.BW, (cuuint32_t)pl.NR, (cuuint32_t)Cin, 1};
    cuuint32_t es[4] = {1, 1, 1, 1};
    if (enc(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, (void*)x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
        return HEX_ERR_CUDA;
    WgParams p{};
    p.dbg = dbg;
    p.dy = dy;
    p.part = part;
    p.part_b = part_b;
    p.Cin = Cin;
    p.Cout = Cout;
    p.H = g.H;
    p.W = g.W;
    p.Ho = g.Ho;
    p.Wo = g.Wo;
    p.s = g.s;
    p.parity = g.parity;
    p.n = g.n;
    p.T = g.T;
    p.Mrows = g.T * Cin;
    p.rows = g.B * g.Ho;
    p.rows_per_cta = pl.rows_per_cta;
    p.cblk = pl.cblk;
    p.rmin = pl.rmin;
    p.NR = pl.NR;
    p.BW = pl.BW;
    for (int t = 0; t < g.T; ++t) {
        int dc, dr0, dr1;
        tap_offset(g.n, 0, t, &dc, &dr0);
        tap_offset(g.n, 1, t, &dc, &dr1);
        p.dc[t] = (int8_t)dc;
        p.dr0[t] = (int8_t)dr0;
        p.dr1[t] = (int8_t)dr1;
    }
    hex_status_t r = HEX_ERR_UNSUPPORTED;
    switch (pl.NT) {
        case 16: r = launch_wg_m<16>(mx, p, pl.MT, pl.grid, pl.smem, st); break;
        case 32: r = launch_wg_m<32>(mx, p, pl.MT, pl.grid, pl.smem, st); break;
        case 48: r = launch_wg_m<48>(mx, p, pl.MT, pl.grid, pl.smem, st); break;
        case 64: r = launch_wg_m<64>(mx, p, pl.MT, pl.grid, pl.smem, st); break;
    }
    if (r != HEX_OK) return r;
    const int total = Cout * g.T * Cin + Cout;
    tf32_wgrad_reduce_kernel<<<ceil_div((int64_t)total * 8, 256), 256, 0, st>>>(part, part_b, pl.grid, Cout, Cin, g.T,
                                                                               dw, dbias, accumulate);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
