// tc_wgrad_tr.cu -- tcgen05 hexagonal-convolution weight gradient with TAP
// REUSE (bf16 NHWC, stride 1, fp32 accumulation in tensor memory).
//
//   dW[t][co][ci] = sum_px dy[px][co] * x[px + off_t][ci]     (pixels are K)
//   dbias[co]     = sum_px dy[px][co]
// (the hexagonal convolution is the sum over the taps of the
// kernel footprint; its weight gradient correlates dy with the tap-shifted
// input.  Off-grid neighbours are TMA's zero fill, A4.)
//
// Pixel tiles are RB rows x JB = 8 sub-columns of ONE parity view of one image,
// ordered row-major ([row][sub-column], so 8 pixels = one 1024-byte SW128
// atom).  For a tile of view P, all taps of one kernel column dc read the SAME
// view P' = (P + dc) mod 2 at the same sub-column shift and differ only by
// their row offset dr = top(dc) + k, k < len(dc).  A row shift is exactly one
// swizzle atom, so ONE x box (RB + 2n rows) per (column, 64-channel chunk)
// serves every tap of the column: the MMA's B operand for tap k starts k atoms
// into the box.  Better still, the taps of a column form one MMA: with the
// MN-major B layout the 64-wide N blocks sit LBO = 1024 B (= one row) apart, so
// N = 64 * len(dc) covers all len(dc) taps of the column in one instruction.
// Per 128-pixel stage that is 3 x-box loads (n = 1) instead of 7, each about
// (RB+2)/RB of a plain box: ~2x less x traffic and 2.3x fewer TMA ops than the
// one-box-per-tap kernel (tc_conv.cu), whose K loop is bound by both.
//
// Work unit = (Cout tile of 128, 64-channel input chunk, column group, pixel
// chunk).  A column group is a set of kernel columns whose taps fit the 512
// TMEM columns (n = 1: all three columns, 7 taps; n = 2: {-2,-1}, {0}, {1,2}).
// Warp 0 issues TMA, warp 1 the MMAs (dbias as an extra block of ones), warps
// 2-5 drain TMEM into a per-pixel-chunk fp32 workspace, summed in a fixed
// order afterwards: deterministic.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hexconv {

namespace {

constexpr int TR_JB = 8;        // sub-columns per pixel tile (one 1024-byte atom per image row)
constexpr int TR_MAXCOLS = 3;   // kernel columns per group
constexpr int TR_SMEM_MAX = 220 * 1024;

struct TrParams {
    int B, H, W, Cin, Cout, T, n, parity, RB;
    int rt, jt0, jt1, tiles0, ptiles;  // pixel tiles per view / in total
    int kchunks, groups, co_tiles, chunks, tiles_per_chunk;
    int stages, xrows;                 // pipeline depth; x box rows = RB + 2n
    int gcols[4][TR_MAXCOLS];          // kernel columns dc of each group (unused slots: 99)
    int ncols[4];
    // 3-D: pixel tile image b is an OUTPUT slice b = vol * Do + zo (dy image); the units'
    // channel chunk kc runs over (depth tap kz, 64-channel chunk of x) = kz * kchunks_x + kcx, reading x image
    // vol * D + sd * zo + kz - pd (all zero fill outside the volume), and the partials are laid out with
    // Cin = kd * Cin_x channels ordered (kz, ci).  2-D: kd = D = Do = sd = 1, pd = 0, kchunks_x = kchunks.
    int kd, D, Do, sd, pd, kchunks_x;
    float* part;     // [chunks][T][Cout][Cin]
    float* db_part;  // [chunks][Cout] or NULL
    int dbg;         // development (HEXCONV_WG_DEBUG): 1 = no TMA loads, 2 = no MMAs (results invalid)
};

__host__ __device__ __forceinline__ int col_len(int n, int dc) { return 2 * n + 1 - (dc < 0 ? -dc : dc); }
__host__ __device__ __forceinline__ int col_tap_base(int n, int dc) {  // canonical index of the column's first tap
    int t = 0;
    for (int c = -n; c < dc; ++c) t += col_len(n, c);
    return t;
}

__device__ __forceinline__ void tr_decode(const TrParams& p, int m, int* P, int* r0, int* j0, int* b) {
    int jt;
    if (p.jt0 == p.jt1) { *P = m & 1; m >>= 1; jt = p.jt0; }  // views interleaved: L2 reuse across views
    else if (m < p.tiles0) { *P = 0; jt = p.jt0; }
    else { *P = 1; m -= p.tiles0; jt = p.jt1; }
    const int rti = m % p.rt;
    m /= p.rt;
    const int jti = m % jt;
    *b = m / jt;
    *r0 = rti * p.RB;
    *j0 = jti * TR_JB;
}

}  // namespace

struct MmaLoopArgs {
    uint64_t* full;
    uint64_t* empty;
    uint64_t* tfull;
    uint32_t tmem_base;
    uint64_t a_desc0, x_desc0, ones_desc;
    uint32_t stage16, xbox16;  // stage stride and x box size in descriptor units (16 B)
    int stages, pt_begin, pt_end, dbg;
};

// Column c of group GRP (compile time): length, TMEM column offset (in 64-column blocks).
template <int N, int GRP>
struct GroupCols {
    static constexpr int ncol = N == 1 ? 3 : (GRP == 1 ? 1 : 2);
    static constexpr int L0 = N == 1 ? 2 : (GRP == 0 ? 3 : GRP == 1 ? 5 : 4);
    static constexpr int L1 = N == 1 ? 3 : (GRP == 0 ? 4 : GRP == 1 ? 0 : 3);
    static constexpr int L2 = N == 1 ? 2 : 0;
};

// MMAs of column C (tap blocks LBO = one row apart; a 5-tap column splits 4 + 1)
template <int LEN, int OFF>
__device__ __forceinline__ void issue_col(uint32_t tmem_base, uint64_t ad, uint64_t bd, uint32_t acc) {
    if constexpr (LEN > 0) {
        constexpr int n0 = LEN > 4 ? 4 : LEN;
        ptx::mma_bf16(tmem_base + 64 * OFF, ad, bd, ptx::idesc_bf16(128, 64 * n0, 1, 1), acc);
        if constexpr (LEN > 4)
            ptx::mma_bf16(tmem_base + 64 * (OFF + 4), ad, bd + 256, ptx::idesc_bf16(128, 64 * (LEN - 4), 1, 1),
                          acc);
    }
}

// The MMA issuer (one thread).  Every shape is a compile-time constant so the issue
// stream is straight-line: measured, a single issuing thread with per-MMA predicates
// or descriptor arithmetic needs ~150 cycles per MMA -- slower than the 64-cycle
// tensor time of an N = 128 MMA -- while this form issues at the tensor-core rate.
template <int RB, int N, int GRP, bool DB>
__device__ __forceinline__ void mma_loop(const MmaLoopArgs& m) {
    using G = GroupCols<N, GRP>;
    constexpr int KSTEPS = TR_JB * RB / 16;
    int stage = 0;
    uint32_t phase = 0;
    uint32_t acc0 = 0;  // the first k-step of the unit initialises the accumulators
    for (int pt = m.pt_begin; pt < m.pt_end; ++pt) {
        ptx::mbar_wait(&m.full[stage], phase);
        ptx::tc_fence_after();
        const uint64_t soff = (uint64_t)stage * m.stage16;
        const uint64_t ad0 = m.a_desc0 + soff, xd0 = m.x_desc0 + soff;
        if (HEX_DBG(m.dbg) != 2) {
#pragma unroll
            for (int k = 0; k < KSTEPS; ++k) {
                const uint64_t ad = ad0 + (uint64_t)(k * 128);  // 16 pixels = 2048 B
                const uint64_t xk = xd0 + (uint64_t)(k * 128);
                const uint32_t acc = k ? 1u : acc0;
                issue_col<G::L0, 0>(m.tmem_base, ad, xk, acc);
                issue_col<G::L1, G::L0>(m.tmem_base, ad, xk + m.xbox16, acc);
                issue_col<G::L2, G::L0 + G::L1>(m.tmem_base, ad, xk + 2 * (uint64_t)m.xbox16, acc);
                if (DB) ptx::mma_bf16(m.tmem_base + 448, ad, m.ones_desc, ptx::idesc_bf16(128, 64, 1, 1), acc);
            }
        }
        acc0 = 1u;
        ptx::mma_commit(&m.empty[stage]);
        if (++stage == m.stages) { stage = 0; phase ^= 1; }
    }
    ptx::mma_commit(m.tfull);
}

template <int RB>
__global__ void __launch_bounds__(192, 1)
tc_wgrad_tr_kernel(const __grid_constant__ CUtensorMap map_x0, const __grid_constant__ CUtensorMap map_x1,
                   const __grid_constant__ CUtensorMap map_dy0, const __grid_constant__ CUtensorMap map_dy1,
                   const __grid_constant__ TrParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = smem_raw + ((1024u - (ptx::smem_u32(smem_raw) & 1023u)) & 1023u);  // 1024-aligned, shared space
    constexpr int TR_PIX = TR_JB * RB;
    constexpr int DY_BOX = TR_PIX * 128;  // one 64-channel dy box
    const int xbox = p.xrows * TR_JB * 128;

    // unit decode
    int u = blockIdx.x;
    const int chunk = u % p.chunks; u /= p.chunks;
    const int grp = u % p.groups; u /= p.groups;
    const int kc = u % p.kchunks;
    const int cot = u / p.kchunks;
    const int co0 = cot * 128;
    const int pt_begin = chunk * p.tiles_per_chunk;
    const int pt_end = min(p.ptiles, pt_begin + p.tiles_per_chunk);
    const int ncol = p.ncols[grp];
    const int stage_bytes = 2 * DY_BOX + ncol * xbox;
    const int stage_stride = (2 * DY_BOX + (p.n == 1 ? 3 : 2) * xbox + 1023) & ~1023;  // = tr_stage_stride
    uint8_t* ones = smem + p.stages * stage_stride;  // 16 K rows x 64 N of bf16 1.0: the dbias column block
    uint64_t* full = (uint64_t*)(ones + 2048);
    uint64_t* empty = full + p.stages;
    uint64_t* tfull = empty + p.stages;
    uint32_t* tmem_slot = (uint32_t*)(tfull + 1);

    // dbias rides on the MMA: units of chunk 0 of one group add an N = 64 block of ones to B, whose
    // accumulator columns are sum_px dy[px][co] (a group's taps use at most 448 of the 512 columns).
    // n = 2: the centre-column group (5 taps + the block = 7 blocks like the two side groups, so every
    // unit carries equal MMA work).  (Summing the staged dy tiles in the idle epilogue warps instead
    // measured slower for n = 1: the stage release then waits for them.)
    const bool do_db = p.db_part != nullptr && grp == (p.n == 1 ? 0 : 1) && kc == 0;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    for (int i = threadIdx.x; i < 512; i += blockDim.x) reinterpret_cast<uint32_t*>(ones)[i] = 0x3F803F80u;
    ptx::fence_proxy_async();  // generic smem writes -> visible to the tensor core (async proxy)
    if (warp == 0 && lane == 0) {
        for (int s = 0; s < p.stages; ++s) {
            ptx::mbar_init(&full[s], 1);
            ptx::mbar_init(&empty[s], 1);
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

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int pt = pt_begin; pt < pt_end; ++pt) {
                int P, r0, j0, b;
                tr_decode(p, pt, &P, &r0, &j0, &b);
                const int pc = (P + p.parity) & 1;  // centre column parity
                ptx::mbar_wait(&empty[stage], phase ^ 1);
                uint8_t* s = smem + stage * stage_stride;
                if (HEX_DBG(p.dbg) == 1) {
                    ptx::mbar_arrive(&full[stage]);
                    if (++stage == p.stages) { stage = 0; phase ^= 1; }
                    continue;
                }
                ptx::mbar_arrive_expect_tx(&full[stage], stage_bytes);
                // dy: both 64-channel chunks of the Cout tile in one op
                ptx::tma_load_5d(P ? &map_dy1 : &map_dy0, &full[stage], s, 0, j0, r0, b, co0 / 64);
                const int kz = kc / p.kchunks_x, kcx = kc - kz * p.kchunks_x;
                const int vol = b / p.Do, zo = b - vol * p.Do;
                const int z = p.sd * zo + kz - p.pd;
                const bool zin = z >= 0 && z < p.D;
                const int ximg = vol * p.D + (zin ? z : 0);
                const int roff = zin ? 0 : p.H + 64;  // outside the volume: the x boxes are all zero fill
                for (int c = 0; c < ncol; ++c) {
                    const int dc = p.gcols[grp][c];
                    const int Pv = (P + dc) & 1;
                    const int jsh = (P + dc - Pv) / 2;
                    const int top = -p.n + (((dc < 0 ? -dc : dc) + pc) >> 1);
                    ptx::tma_load_5d(Pv ? &map_x1 : &map_x0, &full[stage], s + 2 * DY_BOX + c * xbox, 0, j0 + jsh,
                                     r0 + top + roff, ximg, kcx);
                }
                if (++stage == p.stages) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint64_t ones_desc = ptx::smem_desc_sw128(ptx::smem_u32(ones), 1024, 1024);
            const uint64_t a_desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smem), DY_BOX, 1024);
            const uint64_t x_desc0 = ptx::smem_desc_sw128(ptx::smem_u32(smem) + 2 * DY_BOX, 1024, 1024);
            const int key = (p.n == 1 ? 0 : 1 + grp) * 2 + (do_db ? 1 : 0);
            MmaLoopArgs m{full, empty, tfull, tmem_base, a_desc0, x_desc0, ones_desc, (uint32_t)(stage_stride >> 4),
                          (uint32_t)(xbox >> 4), p.stages, pt_begin, pt_end, p.dbg};
            switch (key) {
                case 0: mma_loop<RB, 1, 0, false>(m); break;
                case 1: mma_loop<RB, 1, 0, true>(m); break;
                case 2: case 3: mma_loop<RB, 2, 0, false>(m); break;
                case 4: mma_loop<RB, 2, 1, false>(m); break;
                case 5: mma_loop<RB, 2, 1, true>(m); break;  // dbias rides on the centre-column group
                default: mma_loop<RB, 2, 2, false>(m); break;
            }
        }
    } else {
        const int q = warp & 3;
        const int row = q * 32 + lane;  // co local (TMEM lane)
        ptx::mbar_wait(tfull, 0);
        ptx::tc_fence_after();
        const int co = co0 + row;
        const bool empty_chunk = pt_end <= pt_begin;
        if (do_db) {
            uint32_t v[32];
            ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + 448, v);
            ptx::tmem_ld_wait();
            p.db_part[(int64_t)chunk * p.Cout + co] = empty_chunk ? 0.f : __uint_as_float(v[0]);
        }
        int col_off = 0;
        for (int c = 0; c < ncol; ++c) {
            const int dc = p.gcols[grp][c];
            const int len = col_len(p.n, dc), tb = col_tap_base(p.n, dc);
            for (int k = 0; k < len; ++k) {
                const int t = tb + k;
                float* dst = p.part + (((int64_t)chunk * p.T + t) * p.Cout + co) * p.Cin + kc * 64;
#pragma unroll 1
                for (int ch = 0; ch < 2; ++ch) {
                    uint32_t v[32];
                    ptx::tmem_ld32(tmem_base + ((uint32_t)(q * 32) << 16) + (col_off + k) * 64 + ch * 32, v);
                    ptx::tmem_ld_wait();
                    float4* d4 = reinterpret_cast<float4*>(dst + ch * 32);
#pragma unroll
                    for (int jj = 0; jj < 8; ++jj) {
                        float4 f;
                        f.x = empty_chunk ? 0.f : __uint_as_float(v[4 * jj]);
                        f.y = empty_chunk ? 0.f : __uint_as_float(v[4 * jj + 1]);
                        f.z = empty_chunk ? 0.f : __uint_as_float(v[4 * jj + 2]);
                        f.w = empty_chunk ? 0.f : __uint_as_float(v[4 * jj + 3]);
                        d4[jj] = f;
                    }
                }
            }
            col_off += len;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem_base, 512);
    }
}

// ------------------------------------------------------------------ host side
static PFN_cuTensorMapEncodeTiled_v12000 tr_encode() {
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

// Parity view P of an NHWC bf16 tensor, sub-columns BEFORE rows:
// dims {64, ceil((W-P)/2), H, B, C/64}, box {64, JB, rows, 1, KC}.
static bool make_rowmajor_view(CUtensorMap* m, const void* base, int B, int H, int W, int C, int P, int rows,
                               int KC) {
    auto enc = tr_encode();
    if (!enc) return false;
    const int Wp = (W - P + 1) / 2;
    if (Wp < 1 || C % 64) return false;
    cuuint64_t dims[5] = {64, (cuuint64_t)Wp, (cuuint64_t)H, (cuuint64_t)B, (cuuint64_t)(C / 64)};
    cuuint64_t strides[4] = {(cuuint64_t)2 * C * 2, (cuuint64_t)W * C * 2, (cuuint64_t)H * W * C * 2, 128};
    cuuint32_t box[5] = {64, (cuuint32_t)TR_JB, (cuuint32_t)rows, 1, (cuuint32_t)KC};
    cuuint32_t es[5] = {1, 1, 1, 1, 1};
    void* addr = (void*)((const char*)base + (size_t)P * C * 2);
    return enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, addr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
               CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

struct TrPlan {
    int RB;
    int rt, jt0, jt1, tiles0, ptiles, kchunks, groups, co_tiles, chunks, tiles_per_chunk, stages;
    int gcols[4][TR_MAXCOLS], ncols[4];
};

static int tr_max_cols(int n) { return n == 1 ? 3 : 2; }
static int tr_stage_stride(int n, int RB) {
    return (2 * TR_JB * RB * 128 + tr_max_cols(n) * (RB + 2 * n) * TR_JB * 128 + 1023) & ~1023;
}
static int tr_smem_bytes(int n, int RB, int stages) { return stages * tr_stage_stride(n, RB) + 2048 + 1024 + 256; }
// Rows per pixel tile: 16 (fewer, larger stages) by default; HEXCONV_WG_TR_RB=8 for experiments.
static int tr_rb() {
    static const int rb = (sw_int("HEXCONV_WG_TR_RB", 16) == 8) ? 8 : 16;
    return rb;
}

static TrPlan tr_plan(const Geom& g, int Cin, int Cout, int kd = 1) {
    TrPlan w{};
    w.RB = tr_rb();
    w.rt = ceil_div(g.H, w.RB);
    w.jt0 = ceil_div((g.W + 1) / 2, TR_JB);
    w.jt1 = ceil_div(g.W / 2, TR_JB);
    w.tiles0 = w.rt * w.jt0 * g.B;
    w.ptiles = w.tiles0 + w.rt * w.jt1 * g.B;
    w.kchunks = kd * (Cin / 64);  // (depth tap, channel chunk) units
    w.co_tiles = Cout / 128;
    for (auto& r : w.gcols)
        for (int& c : r) c = 99;
    if (g.n == 1) {
        w.groups = 1;
        w.ncols[0] = 3; w.gcols[0][0] = -1; w.gcols[0][1] = 0; w.gcols[0][2] = 1;
    } else {  // n == 2: {-2,-1} (7 taps), {0} (5), {1,2} (7)
        w.groups = 3;
        w.ncols[0] = 2; w.gcols[0][0] = -2; w.gcols[0][1] = -1;
        w.ncols[1] = 1; w.gcols[1][0] = 0;
        w.ncols[2] = 2; w.gcols[2][0] = 1; w.gcols[2][1] = 2;
    }
    const int base_units = w.co_tiles * w.kchunks * w.groups;
    // one wave of 148 CTAs (one per SM); a fixed SM count keeps the split-K order identical on every B200
    int chunks = 148 / base_units;
    if (chunks < 1) chunks = 1;
    if (chunks > w.ptiles) chunks = w.ptiles;
    w.tiles_per_chunk = ceil_div(w.ptiles, chunks);
    w.chunks = ceil_div(w.ptiles, w.tiles_per_chunk);
    w.stages = 6;
    while (w.stages > 2 && tr_smem_bytes(g.n, w.RB, w.stages) > TR_SMEM_MAX) --w.stages;
    return w;
}

}  // namespace hexconv

namespace hexconv {

// Taken when the tiles are well filled (sub-column and row padding waste <= 15%)
// and the 8-row x boxes divide evenly; HEXCONV_NO_WG_TR disables it.
bool tc_wgrad_tr_supported(const Geom& g, int Cin, int Cout) {
    if (sw_on("HEXCONV_NO_WG_TR")) return false;
    if (g.s != 1 || (g.n != 1 && g.n != 2) || Cout % 128 || Cin % 64 || g.W < 2) return false;
    if (g.B > 65535) return false;
    const double fill_c = (double)((g.W + 1) / 2) / (ceil_div((g.W + 1) / 2, TR_JB) * TR_JB);
    const double fill_r = (double)g.H / (ceil_div(g.H, tr_rb()) * tr_rb());
    const double min_fill = sw_double("HEXCONV_WG_TR_MINFILL", 0.85);
    if (fill_c * fill_r < min_fill) return false;
    if (tr_smem_bytes(g.n, tr_rb(), 2) > TR_SMEM_MAX) return false;
    return tr_encode() != nullptr;
}

size_t tc_wgrad_tr_ws_bytes(const Geom& g, int Cin, int Cout, int kd) {
    const TrPlan w = tr_plan(g, Cin, Cout, kd);
    return (size_t)w.chunks * g.T * Cout * kd * Cin * sizeof(float) + (size_t)w.chunks * Cout * sizeof(float) + 256;
}

hex_status_t tc_wgrad_tr(const TcWgradArgs& a, void* ws, size_t ws_bytes, int* chunks_out, float** db_part_out,
                         cudaStream_t st, const TrDepth* dz) {
    const Geom& g = a.g;  // 3-D: g.B = B * Do output slices
    const int kd = dz ? dz->kd : 1;
    const TrPlan w = tr_plan(g, a.Cin, a.Cout, kd);
    if (ws_bytes < tc_wgrad_tr_ws_bytes(g, a.Cin, a.Cout, kd)) return HEX_ERR_WORKSPACE;
    TrParams p{};
    p.RB = w.RB;
    p.B = g.B; p.H = g.H; p.W = g.W; p.Cin = kd * a.Cin; p.Cout = a.Cout; p.T = g.T; p.n = g.n; p.parity = g.parity;
    p.kd = kd;
    p.D = dz ? dz->D : 1;
    p.Do = dz ? dz->Do : 1;
    p.sd = dz ? dz->sd : 1;
    p.pd = (kd - 1) / 2;
    p.kchunks_x = a.Cin / 64;
    const int Bx = dz ? (g.B / p.Do) * p.D : g.B;  // x images
    p.rt = w.rt; p.jt0 = w.jt0; p.jt1 = w.jt1; p.tiles0 = w.tiles0; p.ptiles = w.ptiles;
    p.kchunks = w.kchunks; p.groups = w.groups; p.co_tiles = w.co_tiles; p.chunks = w.chunks;
    p.tiles_per_chunk = w.tiles_per_chunk; p.stages = w.stages; p.xrows = w.RB + 2 * g.n;
    for (int i = 0; i < 4; ++i) {
        p.ncols[i] = w.ncols[i];
        for (int j = 0; j < TR_MAXCOLS; ++j) p.gcols[i][j] = w.gcols[i][j];
    }
    p.dbg = debug_mode("HEXCONV_WG_DEBUG");
    p.part = (float*)ws;
    p.db_part = a.dbias ? (float*)ws + (size_t)w.chunks * g.T * a.Cout * p.Cin : nullptr;
    CUtensorMap mx0, mx1, md0, md1;
    if (!make_rowmajor_view(&mx0, a.x, Bx, g.H, g.W, a.Cin, 0, p.xrows, 1)) return HEX_ERR_CUDA;
    if (!make_rowmajor_view(&mx1, a.x, Bx, g.H, g.W, a.Cin, 1, p.xrows, 1)) return HEX_ERR_CUDA;
    if (!make_rowmajor_view(&md0, a.dy, g.B, g.H, g.W, a.Cout, 0, w.RB, 2)) return HEX_ERR_CUDA;
    if (!make_rowmajor_view(&md1, a.dy, g.B, g.H, g.W, a.Cout, 1, w.RB, 2)) return HEX_ERR_CUDA;
    const int smem = tr_smem_bytes(g.n, w.RB, w.stages);
    const int units = w.co_tiles * w.kchunks * w.groups * w.chunks;
    if (w.RB == 8) {
        if (cudaFuncSetAttribute(tc_wgrad_tr_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
            cudaSuccess)
            return HEX_ERR_CUDA;
        tc_wgrad_tr_kernel<8><<<units, 192, smem, st>>>(mx0, mx1, md0, md1, p);
    } else {
        if (cudaFuncSetAttribute(tc_wgrad_tr_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) !=
            cudaSuccess)
            return HEX_ERR_CUDA;
        tc_wgrad_tr_kernel<16><<<units, 192, smem, st>>>(mx0, mx1, md0, md1, p);
    }
    count_launch();
    *chunks_out = w.chunks;
    *db_part_out = p.db_part;
    return last_launch_status();
}

}  // namespace hexconv
