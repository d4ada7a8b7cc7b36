// smallc_mma.cu -- single-input-channel hexagonal convolution on the tensor
// cores (bf16 NHWC, stride 1; BASELINE config 5 layer 1: 1 -> 64, n = 2).
//
// With Cin = 1 the layer is a contraction over the T = 3n(n+1)+1 taps only
// (Sec. 2.2): per output pixel p,
//     y[p][co]  = relu?(bias[co] + sum_t w[co][t] * x[p + off_t(parity(p))])
//     dw[co][t] = sum_p dy[p][co] * x[p + off_t],   dbias[co] = sum_p dy[p][co]
// (off-grid neighbours = 0, A4).  On CUDA-core FFMA this layer is
// compute-bound (19 FMAs per output element against 2 bytes written); as a
// [pixels x taps] x [taps x Cout] product with K = T padded to 8/24 it runs on
// the warp-level bf16 tensor-core MMA (mma.sync m16n8k16 / m16n8k8, fp32
// accumulate) and the kernels become bound by the HBM stream of y / dy.
// tcgen05 buys nothing here: K is at most 24, so a 128-row UMMA tile would be
// fed entirely by per-thread gathers anyway.
//
// Both kernels work on bands of RB image rows: the band plus an n-row /
// n-column zero halo of x is staged in shared memory once, and each warp walks
// "items" of 16 consecutive pixels of one row.  The hexagonal gather is a
// per-thread table of shared-memory offsets: a thread's pixels share one column
// parity (forward) or split into the two parities of its pixel pairs (weight
// gradient), so every tap's offset is fixed per thread.
//
//   forward: A = gathered x [16 pixels x K taps] (per-thread LDS.U16 gathers),
//            B = weights [K x 64 channels] held in registers for the whole
//            kernel, accumulators start at the fp32 bias.  Output channels are
//            permuted in B so that each thread ends with 8 + 8 CONSECUTIVE
//            channels of its two pixels: the epilogue is two 16-byte stores per
//            pixel, each warp store instruction covering 4 whole 64-byte
//            half-rows.
//   weight gradient: dW^T [taps (+ a ones row for dbias) x 64] accumulates
//            A = gathered x^T [taps x 16 pixels] times B = dy [16 pixels x 64]
//            loaded by cp.async into a per-warp double-buffered, XOR-swizzled
//            tile and read with ldmatrix.trans.  Fixed-order reductions: warps
//            of a block in warp order, then blocks in block order.
#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"
#include "tc_ptx.cuh"

namespace hexconv {

namespace {

constexpr int MM_WARPS = 8;
constexpr int MM_RB = 16;              // image rows per band (maximum; the host picks rb <= MM_RB)
constexpr int MM_CP = 8;               // zero column pad on each side of a staged row (elements)
constexpr int MM_WG_STAGES = 3;        // dy tiles in flight per warp (weight gradient)
constexpr int MM_TILE = 2048;          // one dy tile: 16 pixels x 64 channels x bf16

__device__ __forceinline__ void mma_16816(float* c, const uint32_t* a, uint32_t b0, uint32_t b1) {
    asm volatile(
        "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
        "{%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

__device__ __forceinline__ void mma_1688(float* c, uint32_t a0, uint32_t a1, uint32_t b0) {
    asm volatile(
        "mma.sync.aligned.m16n8k8.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};\n"
        : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
        : "r"(a0), "r"(a1), "r"(b0));
}

__device__ __forceinline__ uint32_t pack2(uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); }

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
    const int sz = valid ? 16 : 0;  // src-size 0: zero fill
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory"); }

__device__ __forceinline__ void ldsm_x4_trans(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
    asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];\n"
                 : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                 : "r"(addr)
                 : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
            ptx::smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(ptx::smem_u32(bar))
        : "memory");
}

__host__ __device__ __forceinline__ int band_wp(int W) { return (W + 15) / 16 * 16 + 2 * MM_CP; }

// Stage rows r0-N .. r0+rows+N-1 of image plane xb into a band buffer laid out
// xs[(r - r0 + N) * Wp + (c + MM_CP)] (Wp = roundup(W, 16) + 16; the pads stay
// zero, ragged items read zeros).  Rows outside the image are zeroed with plain
// stores; in-image rows are one bulk async copy each (16-byte aligned rows,
// W % 8 == 0) completing on `bar`, else plain copies.  Every thread calls this;
// completion = mbarrier phase + __syncthreads.
template <int N>
__device__ __forceinline__ void stage_band(const uint16_t* __restrict__ xb, uint16_t* xs, uint64_t* bar, int H, int W,
                                           int r0, int rows, bool bulk) {
    const int Wp = band_wp(W);
    const int nr = rows + 2 * N;
    const int rlo = max(0, N - r0), rhi = min(nr, H - r0 + N);  // in-image staged rows [rlo, rhi)
    for (int i = threadIdx.x; i < nr * Wp; i += blockDim.x) {
        const int rr = i / Wp;
        if (rr < rlo || rr >= rhi) {
            xs[i] = 0;
        } else if (!bulk) {
            const int c = i - rr * Wp - MM_CP;
            xs[i] = (c >= 0 && c < W) ? __ldg(xb + (int64_t)(r0 - N + rr) * W + c) : (uint16_t)0;
        }
    }
    if (threadIdx.x == 0) {
        if (bulk) {
            ptx::fence_proxy_async();
            ptx::mbar_arrive_expect_tx(bar, (uint32_t)((rhi - rlo) * W * 2));
            for (int rr = rlo; rr < rhi; ++rr)
                bulk_g2s(xs + rr * Wp + MM_CP, xb + (int64_t)(r0 - N + rr) * W, (uint32_t)(W * 2), bar);
        } else {
            ptx::mbar_arrive(bar);
        }
    }
}

// smem offset of tap t for a centre of column parity p (tap t >= T: 0, unused).
template <int N>
__device__ __forceinline__ int tap_smem_off(int t, int p, int Wp) {
    constexpr int T = 3 * N * (N + 1) + 1;
    if (t >= T) return 0;
    int dc, dr;
    tap_offset(N, p, t, &dc, &dr);
    return dr * Wp + dc;
}

// Forward output-channel permutation: MMA column L = 8j + 2*tig + e of the 64-wide
// block holds channel phys(j, tig, e) so that thread tig owns channels
// 8*tig .. 8*tig+7 (tiles 0-3) and 32 + 8*tig .. (tiles 4-7).
__device__ __forceinline__ int fwd_phys(int j, int tig, int e) {
    return (j < 4 ? 8 * tig + 2 * j : 32 + 8 * tig + 2 * (j - 4)) + e;
}

}  // namespace

// ---------------------------------------------------------------------------
// Forward.  Persistent grid = (min(bands, blocks resident), Cout / 64), 8 warps;
// block k processes bands k, k + gridDim.x, ... with the next band's x staged
// (bulk async copies) while the current one is computed.
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(MM_WARPS * 32, 2)
smallc_mma_fwd_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ w, const float* __restrict__ bias,
                      uint16_t* __restrict__ y, int B, int H, int W, int parity, int Cout, int relu, int bulk, int rb) {
    constexpr int T = 3 * N * (N + 1) + 1;
    constexpr int K16 = N >= 2 ? 1 : 0;  // one k16 step covers taps 0..15
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint16_t* xs = reinterpret_cast<uint16_t*>(smem + 128);
    const int Wp = band_wp(W);
    const int band_elems = (rb + 2 * N) * Wp;
    const int co0 = blockIdx.y * 64;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int bands_per_img = (H + rb - 1) / rb;
    const int nbands = B * bands_per_img;
    const int segs = (W + 15) / 16;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars[0], 1);
        ptx::mbar_init(&bars[1], 1);
        ptx::fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 2 * band_elems; i += blockDim.x) xs[i] = 0;  // pads stay zero
    __syncthreads();

    // B fragments (weights), resident for the whole kernel.  Column n = g of tile j
    // is channel co0 + phys(j, g >> 1, g & 1); tap k rows beyond T are zero.
    uint32_t bk16[8][2], bk8[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int co = co0 + fwd_phys(j, g >> 1, g & 1);
        const uint16_t* wr = w + (int64_t)co * T;
        auto wv = [&](int t) -> uint16_t { return t < T ? __ldg(wr + t) : (uint16_t)0; };
        if (K16) {
            bk16[j][0] = pack2(wv(2 * tig), wv(2 * tig + 1));
            bk16[j][1] = pack2(wv(2 * tig + 8), wv(2 * tig + 9));
        } else {
            bk16[j][0] = bk16[j][1] = 0u;
        }
        bk8[j] = pack2(wv(16 * K16 + 2 * tig), wv(16 * K16 + 2 * tig + 1));
    }
    // accumulator init = bias of the thread's channels (identical for both pixel rows)
    float bi[8][2];
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
        for (int e = 0; e < 2; ++e) bi[j][e] = bias ? __ldg(bias + co0 + fwd_phys(j, tig, e)) : 0.f;

    // the thread's two pixels (columns c0+g, c0+g+8 of an item) share the parity of g;
    // offsets are relative to the smem cell of the centre
    const int p = (g + parity) & 1;
    int off[6];
    off[0] = tap_smem_off<N>(16 * K16 + 2 * tig, p, Wp);
    off[1] = tap_smem_off<N>(16 * K16 + 2 * tig + 1, p, Wp);
    off[2] = tap_smem_off<N>(2 * tig, p, Wp);
    off[3] = tap_smem_off<N>(2 * tig + 1, p, Wp);
    off[4] = tap_smem_off<N>(2 * tig + 8, p, Wp);
    off[5] = tap_smem_off<N>(2 * tig + 9, p, Wp);
    const bool ok0 = 16 * K16 + 2 * tig < T;  // tap index < T (offsets may be negative)
    const bool ok1 = 16 * K16 + 2 * tig + 1 < T;

    int band = blockIdx.x, buf = 0;
    uint32_t phases = 0u;  // bit k: parity of the next completion of bars[k]
    if (band < nbands) {
        const int b = band / bands_per_img, r0 = (band - b * bands_per_img) * rb;
        stage_band<N>(x + (int64_t)b * H * W, xs, &bars[0], H, W, r0, min(rb, H - r0), bulk);
    }
    for (; band < nbands; band += gridDim.x, buf ^= 1) {
        const int nb = band + gridDim.x;
        if (nb < nbands) {  // buffer buf^1 was released by the __syncthreads that ended the previous band
            const int b2 = nb / bands_per_img, r2 = (nb - b2 * bands_per_img) * rb;
            stage_band<N>(x + (int64_t)b2 * H * W, xs + (buf ^ 1) * band_elems, &bars[buf ^ 1], H, W, r2,
                          min(rb, H - r2), bulk);
        }
        ptx::mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        const int b = band / bands_per_img;
        const int r0 = (band - b * bands_per_img) * rb;
        const int rows = min(rb, H - r0);
        const uint16_t* xb = xs + buf * band_elems;
        const int items = rows * segs;
        for (int it = warp; it < items; it += MM_WARPS) {
            const int rl = it / segs;
            const int c0 = (it - rl * segs) * 16;
            const uint16_t* p0 = xb + (rl + N) * Wp + c0 + g + MM_CP;  // centre of pixel g
            const uint16_t* p1 = p0 + 8;                               // centre of pixel g + 8
            uint32_t a16[4] = {0u, 0u, 0u, 0u};
            if (K16) {
                a16[0] = pack2(p0[off[2]], p0[off[3]]);
                a16[1] = pack2(p1[off[2]], p1[off[3]]);
                a16[2] = pack2(p0[off[4]], p0[off[5]]);
                a16[3] = pack2(p1[off[4]], p1[off[5]]);
            }
            const uint32_t a8_0 = pack2(ok0 ? p0[off[0]] : (uint16_t)0, ok1 ? p0[off[1]] : (uint16_t)0);
            const uint32_t a8_1 = pack2(ok0 ? p1[off[0]] : (uint16_t)0, ok1 ? p1[off[1]] : (uint16_t)0);
            float acc[8][4];
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                acc[j][0] = bi[j][0]; acc[j][1] = bi[j][1];
                acc[j][2] = bi[j][0]; acc[j][3] = bi[j][1];
            }
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (K16) mma_16816(acc[j], a16, bk16[j][0], bk16[j][1]);
                mma_1688(acc[j], a8_0, a8_1, bk8[j]);
            }
            // epilogue: relu, bf16 (RNE), two 16-byte stores per pixel
            const int r = r0 + rl;
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = c0 + g + 8 * h;
                if (c >= W) continue;
                uint32_t pk[8];
                if (relu) {  // ReLU inside the conversion (cvt.rn.relu: negatives and -0 give +0)
#pragma unroll
                    for (int j = 0; j < 8; ++j) pk[j] = ptx::pack_bf16x2_relu(acc[j][2 * h], acc[j][2 * h + 1]);
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        __nv_bfloat162 hv = __floats2bfloat162_rn(acc[j][2 * h], acc[j][2 * h + 1]);
                        pk[j] = *reinterpret_cast<uint32_t*>(&hv);
                    }
                }
                uint4* dst = reinterpret_cast<uint4*>(y + (((int64_t)b * H + r) * W + c) * Cout + co0);
                dst[tig] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                dst[4 + tig] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
            }
        }
        __syncthreads();  // everyone is done with buffer `buf` before it is restaged
    }
}

// ---------------------------------------------------------------------------
// Weight gradient.  Persistent grid = (min(bands, blocks resident), Cout / 64);
// block k processes bands k, k + gridDim.x, ...  Per warp, the dy tiles of its
// items stream through an MM_WG_STAGES-deep cp.async ring; the next band's x is
// staged by bulk copies meanwhile.  Partials part[block][co][T + 1] (last column
// = dbias) are reduced in block order by smallc_mma_reduce_kernel.
// ---------------------------------------------------------------------------
template <int N>
__global__ void __launch_bounds__(MM_WARPS * 32, 2)
smallc_mma_wgrad_kernel(const uint16_t* __restrict__ x, const uint16_t* __restrict__ dy, float* __restrict__ part,
                        int B, int H, int W, int parity, int Cout, int bulk, int rb) {
    constexpr int T = 3 * N * (N + 1) + 1;
    constexpr int MT = (T + 1 + 15) / 16;  // m-tiles of 16 tap rows (incl. the ones row)
    constexpr int NA = T + 1;
    constexpr int ST = MM_WG_STAGES;
    extern __shared__ __align__(128) uint8_t smem[];
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem);
    uint8_t* dyt = smem + 128;                                           // [warp][ST][16 px][128 B], swizzled
    uint16_t* xs = reinterpret_cast<uint16_t*>(dyt + MM_WARPS * ST * MM_TILE);
    const int Wp = band_wp(W);
    const int band_elems = (rb + 2 * N) * Wp;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int g = lane >> 2, tig = lane & 3;
    const int co0 = blockIdx.y * 64;
    const int bands_per_img = (H + rb - 1) / rb;
    const int nbands = B * bands_per_img;
    const int segs = (W + 15) / 16;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bars[0], 1);
        ptx::mbar_init(&bars[1], 1);
        ptx::fence_barrier_init();
    }
    for (int i = threadIdx.x; i < 2 * band_elems; i += blockDim.x) xs[i] = 0;  // pads stay zero
    __syncthreads();

    // A gather table: taps m = 16*mt + g (+8), pixels 2tig (+8) of parity pe, 2tig+1 (+9) of parity po.
    // code: >= 0 smem offset from the item's band origin, -1 zero, -2 the ones row (dbias)
    const int pe = parity & 1, po = pe ^ 1;
    int offe[MT][2], offo[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int t = 16 * mt + g + 8 * h;
            if (t == T) { offe[mt][h] = -2; offo[mt][h] = -2; }
            else if (t > T) { offe[mt][h] = -1; offo[mt][h] = -1; }
            else {
                int dc, dr;
                tap_offset(N, pe, t, &dc, &dr);
                offe[mt][h] = (dr + N) * Wp + dc + MM_CP;
                tap_offset(N, po, t, &dc, &dr);
                offo[mt][h] = (dr + N) * Wp + dc + MM_CP;
            }
        }

    float acc[MT][8][4];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int j = 0; j < 8; ++j)
#pragma unroll
            for (int e = 0; e < 4; ++e) acc[mt][j][e] = 0.f;

    const uint32_t ring = ptx::smem_u32(dyt + warp * ST * MM_TILE);
    // ldmatrix.x4.trans lane address: matrix mi = lane >> 3 (pixels +8 for odd mi, tile +1 for mi >= 2)
    const int lm_pix = ((lane >> 3) & 1) * 8 + (lane & 7);
    const int lm_tile = lane >> 4;

    int band = blockIdx.x, buf = 0;
    uint32_t phases = 0u;  // bit k: parity of the next completion of bars[k]
    if (band < nbands) {
        const int b = band / bands_per_img, r0 = (band - b * bands_per_img) * rb;
        stage_band<N>(x + (int64_t)b * H * W, xs, &bars[0], H, W, r0, min(rb, H - r0), bulk);
    }
    for (; band < nbands; band += gridDim.x, buf ^= 1) {
        const int b = band / bands_per_img;
        const int r0 = (band - b * bands_per_img) * rb;
        const int rows = min(rb, H - r0);
        const int items = rows * segs;
        const uint16_t* dimg = dy + (int64_t)b * H * W * Cout + co0;
        // dy tile of item `it` into ring slot `slot`: 16 pixels x 128 B = 128 16-byte chunks, 4 per lane;
        // one commit group per call (possibly empty) keeps the group count uniform
        auto issue = [&](int it, int rl, int sg, int slot) {  // item it = rl * segs + sg
            if (it < items) {
                const int c0 = sg * 16;
                const int r = r0 + rl;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int ch = lane + 32 * q;  // chunk id: pixel = ch >> 3, tile = ch & 7
                    const int px = ch >> 3, tl = ch & 7;
                    const int c = c0 + px;
                    const bool ok = c < W;
                    const uint16_t* src = dimg + ((int64_t)r * W + (ok ? c : 0)) * Cout + tl * 8;
                    cp_async16(ring + slot * MM_TILE + px * 128 + ((tl ^ (px & 7)) << 4), src, ok);
                }
            }
            cp_async_commit();
        };
#pragma unroll
        for (int s = 0; s < ST - 1; ++s) {
            const int it0 = warp + s * MM_WARPS;
            issue(it0, it0 / segs, it0 % segs, s);
        }
        const int nb = band + gridDim.x;
        if (nb < nbands) {  // buffer buf^1 was released by the __syncthreads that ended the previous band
            const int b2 = nb / bands_per_img, r2 = (nb - b2 * bands_per_img) * rb;
            stage_band<N>(x + (int64_t)b2 * H * W, xs + (buf ^ 1) * band_elems, &bars[buf ^ 1], H, W, r2,
                          min(rb, H - r2), bulk);
        }
        ptx::mbar_wait(&bars[buf], (phases >> buf) & 1u);
        phases ^= 1u << buf;
        __syncthreads();
        const uint16_t* xb = xs + buf * band_elems;
        int slot = 0;
        int rl = warp / segs, sg = warp % segs;  // item it = rl * segs + sg, stepped by MM_WARPS
        const int pit0 = warp + (ST - 1) * MM_WARPS;  // the item prefetched ST - 1 steps ahead
        int prl = pit0 / segs, psg = pit0 % segs;
        for (int it = warp; it < items; it += MM_WARPS) {
            issue(it + (ST - 1) * MM_WARPS, prl, psg, (slot + ST - 1) % ST);
            psg += MM_WARPS;
            while (psg >= segs) { psg -= segs; ++prl; }
            cp_async_wait<ST - 1>();
            __syncwarp();
            const int c0 = sg * 16;
            const uint16_t* base = xb + rl * Wp + c0;
            // A fragments: a0 = {m g: px 2tig, 2tig+1}, a1 = {m g+8: ...}, a2 = {m g: px 2tig+8, +9}, a3 = {m g+8: ...}
            uint32_t a[MT][4];
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // branch-free (the tap rows differ per lane): load from a valid offset, then select
                    const int oe = offe[mt][h], oo = offo[mt][h];
                    const bool tap = oe >= 0;
                    const uint16_t cst = oe == -2 ? (uint16_t)0x3F80 : (uint16_t)0;  // 1.0 (dbias row) or 0
                    const uint16_t* pe_ = base + 2 * tig + (tap ? oe : 0);
                    const uint16_t* po_ = base + 2 * tig + 1 + (tap ? oo : 0);
                    const uint16_t e0 = tap ? pe_[0] : cst, e1 = tap ? pe_[8] : cst;
                    const uint16_t o0 = tap ? po_[0] : cst, o1 = tap ? po_[8] : cst;
                    a[mt][h] = pack2(e0, o0);
                    a[mt][2 + h] = pack2(e1, o1);
                }
            // B fragments from the swizzled dy tile, two n-tiles per ldmatrix.x4.trans
            const uint32_t tb = ring + slot * MM_TILE + lm_pix * 128;
#pragma unroll
            for (int jj = 0; jj < 4; ++jj) {
                const int tl = 2 * jj + lm_tile;
                uint32_t b00, b01, b10, b11;
                ldsm_x4_trans(tb + ((tl ^ (lm_pix & 7)) << 4), b00, b01, b10, b11);
#pragma unroll
                for (int mt = 0; mt < MT; ++mt) {
                    mma_16816(acc[mt][2 * jj], a[mt], b00, b01);
                    mma_16816(acc[mt][2 * jj + 1], a[mt], b10, b11);
                }
            }
            __syncwarp();  // slot `slot` is refilled ST - 1 items later
            slot = (slot + 1 == ST) ? 0 : slot + 1;
            sg += MM_WARPS;
            while (sg >= segs) { sg -= segs; ++rl; }
        }
        cp_async_wait<0>();  // drain the (empty) tail groups
        __syncthreads();     // everyone is done with buffer `buf` before it is restaged
    }

    // fixed-order block reduction: warps add their dW^T fragments into red[m][co] in warp order
    float* red = reinterpret_cast<float*>(dyt);  // [MT*16][64] (aliases the dy rings, now idle)
    for (int i = threadIdx.x; i < MT * 16 * 64; i += blockDim.x) red[i] = 0.f;
    __syncthreads();
    for (int wv = 0; wv < MM_WARPS; ++wv) {
        if (warp == wv) {
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const int m0 = 16 * mt + g, col = 8 * j + 2 * tig;
                    red[m0 * 64 + col] += acc[mt][j][0];
                    red[m0 * 64 + col + 1] += acc[mt][j][1];
                    red[(m0 + 8) * 64 + col] += acc[mt][j][2];
                    red[(m0 + 8) * 64 + col + 1] += acc[mt][j][3];
                }
        }
        __syncthreads();
    }
    // part[block][co][t]; t = T is the dbias column
    float* pp = part + ((int64_t)blockIdx.x * Cout + co0) * NA;
    for (int i = threadIdx.x; i < 64 * NA; i += blockDim.x) {
        const int cl = i / NA, t = i - cl * NA;
        pp[i] = red[t * 64 + cl];
    }
}

// Deterministic reduction of the per-block partials: 8 lanes per output, each
// summing a fixed strided subset of blocks, then a fixed shuffle tree.
__global__ void smallc_mma_reduce_kernel(const float* __restrict__ part, int nblocks, int Cout, int NA,
                                         float* __restrict__ dw, float* __restrict__ dbias, int accumulate) {
    const int gid = blockIdx.x * blockDim.x + threadIdx.x;
    const int o = gid >> 3, sub = gid & 7;
    const int total = Cout * NA;
    float s = 0.f;
    if (o < total)
        for (int k = sub; k < nblocks; k += 8) s += part[(int64_t)k * total + o];
    s += __shfl_xor_sync(0xffffffffu, s, 4);
    s += __shfl_xor_sync(0xffffffffu, s, 2);
    s += __shfl_xor_sync(0xffffffffu, s, 1);
    if (o >= total || sub != 0) return;
    const int co = o / NA, t = o - co * NA;
    if (t == NA - 1) {
        if (dbias) dbias[co] = accumulate ? dbias[co] + s : s;
    } else {
        float* d = dw + (int64_t)co * (NA - 1) + t;
        *d = accumulate ? *d + s : s;
    }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
static size_t band_bytes(const Geom& g) { return (size_t)(MM_RB + 2 * g.n) * band_wp(g.W) * 2; }
static size_t fwd_smem(const Geom& g) { return 128 + 2 * band_bytes(g); }
static size_t wgrad_smem(const Geom& g) { return 128 + (size_t)MM_WARPS * MM_WG_STAGES * MM_TILE + 2 * band_bytes(g); }
static bool bulk_ok(const Geom& g, const void* x) { return g.W % 8 == 0 && ((uintptr_t)x & 15) == 0; }

bool smallc_mma_supported(const Geom& g, int Cin, int Cout) {
    return Cin == 1 && Cout % 64 == 0 && (g.n == 1 || g.n == 2) && g.s == 1 && g.B <= 65535 &&
           wgrad_smem(g) <= 100 * 1024;
}

// rows per band: the persistent grid's last round should be nearly full (H = 96, B = 256: 16 rows give
// 1536 bands = 5.2 rounds of 296 blocks, 12 rows 2048 = 6.9 rounds); a band's fixed cost ~ one row
static int pick_rb(const Geom& g) {
    const int slots = 2 * num_sms();
    int best = MM_RB;
    double best_score = 0.0;
    for (int rb = MM_RB; rb >= 8; --rb) {
        const int per = (g.H + rb - 1) / rb;
        const long bands = (long)g.B * per;
        const long rounds = (bands + slots - 1) / slots;
        const double fill = bands < slots ? 1.0 : (double)bands / (double)(rounds * slots);
        const double score = fill * ((double)g.H / (per * rb)) * rb / (rb + 1.0);
        if (score > best_score + 1e-9) { best_score = score; best = rb; }
    }
    return best;
}

static int resident_blocks(const Geom& g) {
    const int rb = pick_rb(g);
    const int nbands = g.B * ((g.H + rb - 1) / rb);
    const int cap = 2 * num_sms();  // 2 blocks of 8 warps per SM (launch bounds)
    return nbands < cap ? nbands : cap;
}

size_t smallc_mma_wgrad_ws_bytes(const Geom& g, int Cout) {
    return (size_t)resident_blocks(g) * Cout * (g.T + 1) * sizeof(float);
}

template <int N>
static void launch_fwd(const Geom& g, dim3 grid, size_t smem, cudaStream_t st, const uint16_t* x, const uint16_t* w,
                       const float* bias, uint16_t* y, int Cout, int relu, int bulk) {
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(smallc_mma_fwd_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smallc_mma_fwd_kernel<N><<<grid, MM_WARPS * 32, smem, st>>>(x, w, bias, y, g.B, g.H, g.W, g.parity, Cout, relu,
                                                               bulk, pick_rb(g));
}

template <int N>
static void launch_wgrad(const Geom& g, dim3 grid, size_t smem, cudaStream_t st, const uint16_t* x, const uint16_t* dy,
                         float* part, int Cout, int bulk) {
    if (smem > 48 * 1024)
        cudaFuncSetAttribute(smallc_mma_wgrad_kernel<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    smallc_mma_wgrad_kernel<N><<<grid, MM_WARPS * 32, smem, st>>>(x, dy, part, g.B, g.H, g.W, g.parity, Cout, bulk,
                                                                   pick_rb(g));
}

hex_status_t smallc_mma_fwd(const void* x, const void* w, const float* bias, void* y, const Geom& g, int Cout,
                            int relu, cudaStream_t st) {
    dim3 grid(resident_blocks(g), Cout / 64);
    const int bulk = bulk_ok(g, x);
    if (g.n == 1)
        launch_fwd<1>(g, grid, fwd_smem(g), st, (const uint16_t*)x, (const uint16_t*)w, bias, (uint16_t*)y, Cout,
                      relu, bulk);
    else
        launch_fwd<2>(g, grid, fwd_smem(g), st, (const uint16_t*)x, (const uint16_t*)w, bias, (uint16_t*)y, Cout,
                      relu, bulk);
    count_launch();
    return last_launch_status();
}

hex_status_t smallc_mma_wgrad(const void* x, const void* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                              int Cout, void* ws, cudaStream_t st) {
    const int nb = resident_blocks(g);
    dim3 grid(nb, Cout / 64);
    const int bulk = bulk_ok(g, x);
    if (g.n == 1)
        launch_wgrad<1>(g, grid, wgrad_smem(g), st, (const uint16_t*)x, (const uint16_t*)dy, (float*)ws, Cout, bulk);
    else
        launch_wgrad<2>(g, grid, wgrad_smem(g), st, (const uint16_t*)x, (const uint16_t*)dy, (float*)ws, Cout, bulk);
    count_launch();
    const int NA = g.T + 1;
    const int outs = Cout * NA;
    smallc_mma_reduce_kernel<<<ceil_div((int64_t)outs * 8, 256), 256, 0, st>>>((const float*)ws, nb, Cout, NA, dw,
                                                                               dbias, accumulate);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
