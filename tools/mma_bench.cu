// mma_bench.cu -- development microbenchmark: issue rate of tcgen05.mma (kind::f16,
// cta_group::1, M = 128) for the operand layouts the hexconv kernels use.  One CTA
// per SM, one thread issues ITERS MMAs (data is whatever is in shared memory), and
// the kernel reports cycles per MMA and MACs per cycle per SM.
//
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_1903_01814_b200/csrc \
//        tools/mma_bench.cu -o /tmp/mma_bench -lcuda
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "tc_ptx.cuh"

using namespace hexconv;

struct Cfg {
    int M, N, a_mn, b_mn, a_lbo, b_lbo, b_sbo, nmma;  // nmma: MMAs per k-step with distinct N blocks (D offsets)
    const char* name;
};

__global__ void __launch_bounds__(128, 1) bench(Cfg c, int iters, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_init(&bar2, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc(&slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (c.nmma == -3 && warp == 0) {  // whole warp runs the loop, one elected lane issues
        const uint32_t s = ptx::smem_u32(smem);
        const uint32_t idesc = ptx::idesc_bf16(c.M, c.N, c.a_mn, c.b_mn);
        const uint64_t ad0 = ptx::smem_desc_sw128(s, 16, 1024);
        const uint64_t bd0 = ptx::smem_desc_sw128(s + 65536, 16, 1024);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t ad = ad0 + (uint64_t)((i & 7) * 2), bd = bd0 + (uint64_t)((i & 7) * 2);
            const uint32_t d = tmem + (uint32_t)((i & 1) * c.N);
            uint32_t pred;
            asm volatile("{\n\t.reg .pred P;\n\telect.sync _|P, 0xffffffff;\n\tselp.u32 %0, 1, 0, P;\n\t}" : "=r"(pred));
            if (pred) ptx::mma_bf16(d, ad, bd, idesc, 1);
            __syncwarp();
        }
        if (threadIdx.x == 0) {
            ptx::mma_commit(&bar);
            ptx::mbar_wait(&bar, 0);
            out[blockIdx.x] = clock64() - t0;
        }
    } else if (c.nmma == -2 && threadIdx.x == 0) {  // lane 0 alone, 64-bit descriptor adds per MMA
        const uint32_t s = ptx::smem_u32(smem);
        const uint32_t idesc = ptx::idesc_bf16(c.M, c.N, c.a_mn, c.b_mn);
        const uint64_t ad0 = ptx::smem_desc_sw128(s, 16, 1024);
        const uint64_t bd0 = ptx::smem_desc_sw128(s + 65536, 16, 1024);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t ad = ad0 + (uint64_t)((i & 7) * 2), bd = bd0 + (uint64_t)((i & 7) * 2);
            ptx::mma_bf16(tmem + (uint32_t)((i & 1) * c.N), ad, bd, idesc, 1);
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    } else if (c.nmma > -2 && threadIdx.x == 0) {
        const uint32_t s = ptx::smem_u32(smem);
        const uint32_t idesc = ptx::idesc_bf16(c.M, c.N, c.a_mn, c.b_mn);
        if (c.nmma < 0) {  // lean issue loop: descriptors built once, 8 MMAs per iteration, 8 D tiles
            // (nmma = -4: all MMAs into ONE accumulator; -5: two accumulators alternating)
            const uint64_t ad = ptx::smem_desc_sw128(s, 16, 1024);
            const uint64_t bd = ptx::smem_desc_sw128(s + 65536, 16, 1024);
            const uint32_t step = c.nmma == -4 ? 0u : (c.nmma == -5 ? (uint32_t)(c.N * 4) : (uint32_t)c.N);
            const long long t0 = clock64();
            for (int i = 0; i < iters; i += 8) {
#pragma unroll
                for (int j = 0; j < 8; ++j) ptx::mma_bf16(tmem + ((j * step) & 511), ad, bd, idesc, 1);
                if (c.nmma == -6) ptx::mma_commit(&bar2);  // a commit every 8 MMAs (nobody waits)
            }
            ptx::mma_commit(&bar);
            ptx::mbar_wait(&bar, 0);
            out[blockIdx.x] = clock64() - t0;
        } else {
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int k = i & 7;
            // A: MN-major -> 64-row blocks LBO apart, K groups 1024 B apart; K-major -> k*32 B advance
            const uint64_t ad = c.a_mn ? ptx::smem_desc_sw128(s + k * 2048, c.a_lbo, 1024)
                                       : ptx::smem_desc_sw128(s + (k & 3) * 32, 16, 1024);
            const uint32_t bs = s + 65536;
            const uint64_t bd = c.b_mn ? ptx::smem_desc_sw128(bs + k * 2048, c.b_lbo, c.b_sbo)
                                       : ptx::smem_desc_sw128(bs + (k & 3) * 32, 16, 1024);
            const int j = i % c.nmma;
            ptx::mma_bf16(tmem + (uint32_t)(j * c.N), ad, bd, idesc, 1);
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        const long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// A fixed sequence of MMAs per k-step (MN-major A and B, B blocks 1024 B apart), lean issue.
template <int N0, int N1, int N2, int N3>
__global__ void __launch_bounds__(128, 1) bench_seq(int iters, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc(&slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t s = ptx::smem_u32(smem);
        const uint64_t ad0 = ptx::smem_desc_sw128(s, 16384, 1024);
        const uint64_t bd0 = ptx::smem_desc_sw128(s + 32768, 1024, 1024);
        const long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const uint64_t ad = ad0 + (uint64_t)((i & 7) * 128), bd = bd0 + (uint64_t)((i & 7) * 128);
            ptx::mma_bf16(tmem, ad, bd, ptx::idesc_bf16(128, N0, 1, 1), 1);
            if (N1) ptx::mma_bf16(tmem + N0, ad, bd + 1152, ptx::idesc_bf16(128, N1 ? N1 : 64, 1, 1), 1);
            if (N2) ptx::mma_bf16(tmem + N0 + N1, ad, bd + 2304, ptx::idesc_bf16(128, N2 ? N2 : 64, 1, 1), 1);
            if (N3) ptx::mma_bf16(tmem + N0 + N1 + N2, ad, bd + 3456, ptx::idesc_bf16(128, N3 ? N3 : 64, 1, 1), 1);
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// Shared-memory bandwidth contention: thread 0 issues ITERS lean K-major MMAs (M = 128, N) while
// LW warps stream LDS.128 over a separate 32 KB area until the MMAs are done.
template <int N, int LW>
__global__ void __launch_bounds__(64 + 32 * LW, 1) bench_contend(int iters, long long* out, long long* lds_bytes) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar;
    __shared__ uint32_t slot;
    __shared__ volatile int done;
    __shared__ unsigned long long nbytes;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::fence_barrier_init();
        done = 0;
        nbytes = 0;
    }
    if (warp == 1) ptx::tmem_alloc(&slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t s = ptx::smem_u32(smem);
        const uint32_t idesc = ptx::idesc_bf16(128, N, 0, 0);
        const uint64_t ad = ptx::smem_desc_sw128(s, 16, 1024);
        const uint64_t bd = ptx::smem_desc_sw128(s + 65536, 16, 1024);
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += 8) {
#pragma unroll
            for (int j = 0; j < 8; ++j) ptx::mma_bf16(tmem + ((j * N) & 511), ad, bd, idesc, 1);
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
        done = 1;
    } else if (warp >= 2) {
        const uint4* src = reinterpret_cast<const uint4*>(smem + 131072);
        uint32_t acc = 0;
        unsigned long long cnt = 0;
        int i = threadIdx.x & 31;
        while (!done) {
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                const uint4 v = src[(i + u * 32 + (warp - 2) * 512) & 2047];
                acc ^= v.x ^ v.y ^ v.z ^ v.w;
            }
            i += 7;
            cnt += 16 * 16;
        }
        atomicAdd(&nbytes, cnt);
        if (acc == 0x12345678u) out[0] = 0;  // keep the loads
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (threadIdx.x == 0) lds_bytes[blockIdx.x] = (long long)nbytes;
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

// Compile-time commit frequency: EVERY MMAs (M = 128, N, K-major, two D tiles) then one tcgen05.commit.
template <int N, int EVERY>
__global__ void __launch_bounds__(128, 1) bench_commit(int iters, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t slot;
    const int warp = threadIdx.x / 32;
    if (threadIdx.x == 0) {
        ptx::mbar_init(&bar, 1);
        ptx::mbar_init(&bar2, 1);
        ptx::fence_barrier_init();
    }
    if (warp == 1) ptx::tmem_alloc(&slot, 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = slot;
    if (threadIdx.x == 0) {
        const uint32_t s = ptx::smem_u32(smem);
        constexpr uint32_t idesc = ptx::idesc_bf16(128, N, 0, 0);
        const uint64_t ad = ptx::smem_desc_sw128(s, 16, 1024);
        const uint64_t bd = ptx::smem_desc_sw128(s + 65536, 16, 1024);
        const long long t0 = clock64();
        for (int i = 0; i < iters; i += EVERY) {
#pragma unroll
            for (int j = 0; j < EVERY; ++j) ptx::mma_bf16(tmem + (uint32_t)((j & 1) * 256), ad, bd, idesc, 1);
            if (EVERY < 1024) ptx::mma_commit(&bar2);
        }
        ptx::mma_commit(&bar);
        ptx::mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
    }
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == 1) {
        ptx::tc_fence_after();
        ptx::tmem_dealloc(tmem, 512);
    }
}

template <int N, int EVERY>
static void run_commit(long long* d_out) {
    const int smem = 200 * 1024, iters = 8192;
    cudaFuncSetAttribute(bench_commit<N, EVERY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench_commit<N, EVERY><<<148, 128, smem>>>(iters, d_out);
    bench_commit<N, EVERY><<<148, 128, smem>>>(iters, d_out);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    printf("commit N=%3d every %4d MMAs: %7.1f cyc/MMA\n", N, EVERY, avg / 148 / iters);
}

template <int N, int LW>
static void run_contend(long long* d_out, long long* d_lds) {
    const int smem = 200 * 1024, iters = 16384;
    cudaFuncSetAttribute(bench_contend<N, LW>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench_contend<N, LW><<<148, 64 + 32 * LW, smem>>>(iters, d_out, d_lds);
    bench_contend<N, LW><<<148, 64 + 32 * LW, smem>>>(iters, d_out, d_lds);
    cudaDeviceSynchronize();
    long long h[148], l[148];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    cudaMemcpy(l, d_lds, sizeof(l), cudaMemcpyDeviceToHost);
    double avg = 0, lb = 0;
    for (int i = 0; i < 148; ++i) { avg += h[i]; lb += l[i]; }
    avg /= 148;
    lb /= 148;
    printf("contend N=%3d lds_warps=%2d  %7.1f cyc/MMA (ideal %5.1f)  LDS %6.1f B/clk  MMA operands %6.1f B/clk\n", N,
           LW, avg / iters, N / 2.0, lb / avg, (double)iters * (128 + N) * 32 / avg);
}

template <int N0, int N1, int N2, int N3>
static void run_seq(const char* name, long long* d_out) {
    const int smem = 200 * 1024, iters = 4096;
    cudaFuncSetAttribute(bench_seq<N0, N1, N2, N3>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench_seq<N0, N1, N2, N3><<<148, 128, smem>>>(iters, d_out);
    bench_seq<N0, N1, N2, N3><<<148, 128, smem>>>(iters, d_out);
    cudaDeviceSynchronize();
    long long h[148];
    cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < 148; ++i) avg += h[i];
    avg /= 148;
    const double cyc = avg / iters;
    const int N = N0 + N1 + N2 + N3;
    printf("%-36s %7.1f cyc/step (ideal %5.1f)  %7.0f MAC/clk/SM\n", name, cyc, N / 2.0, 128.0 * N * 16 / cyc);
}

int main() {
    Cfg cfgs[] = {
        {128, 128, 0, 0, 16, 16, 1024, -2, "lane0 loop desc-add N=128"},
        {128, 128, 0, 0, 16, 16, 1024, -3, "warp loop + elect N=128"},
        {128, 256, 0, 0, 16, 16, 1024, -3, "warp loop + elect N=256"},
        {128, 256, 0, 0, 16, 16, 1024, -1, "lean K-major N=256"},
        {128, 128, 0, 0, 16, 16, 1024, -1, "lean K-major N=128"},
        {128, 64, 0, 0, 16, 16, 1024, -1, "lean K-major N=64"},
        {128, 32, 0, 0, 16, 16, 1024, -1, "lean K-major N=32"},
        {64, 256, 0, 0, 16, 16, 1024, 1, "M=64 K-major A,B  N=256"},
        {64, 128, 0, 0, 16, 16, 1024, 2, "M=64 K-major A,B  N=128"},
        {128, 256, 0, 0, 16, 16, 1024, 1, "K-major A,B  N=256"},
        {128, 128, 0, 0, 16, 16, 1024, 2, "K-major A,B  N=128 (2 D)"},
        {128, 64, 0, 0, 16, 16, 1024, 4, "K-major A,B  N=64 (4 D)"},
        {128, 256, 1, 1, 16384, 8192, 1024, 1, "MN-major A,B N=256 LBO 8K"},
        {128, 192, 1, 1, 16384, 1024, 1024, 2, "MN-major A,B N=192 LBO 1K"},
        {128, 128, 1, 1, 16384, 1024, 1024, 4, "MN-major A,B N=128 LBO 1K"},
        {128, 64, 1, 1, 16384, 1024, 1024, 8, "MN-major A,B N=64"},
        {128, 256, 1, 1, 16384, 1024, 1024, 2, "MN-major A,B N=256 LBO 1K"},
        {128, 256, 1, 1, 16384, 1024, 3072, 2, "MN-major A,B N=256 LBO 1K SBO 3K"},
        {128, 256, 1, 0, 16384, 16, 1024, 1, "MN-major A, K-major B N=256"},
        {128, 256, 0, 1, 16, 8192, 1024, 1, "K-major A, MN-major B N=256"},
    };
    long long* d_out;
    cudaMalloc(&d_out, 148 * sizeof(long long));
    if (getenv("MMA_CONTEND")) {
        long long* d_lds;
        cudaMalloc(&d_lds, 148 * sizeof(long long));
        {
            Cfg extra[] = {
                {128, 64, 0, 0, 16, 16, 1024, -1, "lean N=64, 8 D tiles"},
                {128, 64, 0, 0, 16, 16, 1024, -4, "lean N=64, one D"},
                {128, 64, 0, 0, 16, 16, 1024, -5, "lean N=64, two D alternating"},
                {128, 128, 0, 0, 16, 16, 1024, -1, "lean N=128, 8 D tiles"},
                {128, 128, 0, 0, 16, 16, 1024, -4, "lean N=128, one D"},
                {128, 256, 0, 0, 16, 16, 1024, -4, "lean N=256, one D"},
                {128, 64, 0, 0, 16, 16, 1024, -6, "lean N=64, commit every 8"},
                {128, 128, 0, 0, 16, 16, 1024, -6, "lean N=128, commit every 8"},
                {128, 256, 0, 0, 16, 16, 1024, -1, "lean N=256, 2 D"},
            };
            const int smem = 200 * 1024;
            cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            for (const Cfg& c : extra) {
                bench<<<148, 128, smem>>>(c, 8192, d_out);
                bench<<<148, 128, smem>>>(c, 8192, d_out);
                cudaDeviceSynchronize();
                long long h[148];
                cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
                double avg = 0;
                for (int i = 0; i < 148; ++i) avg += h[i];
                printf("%-36s %7.1f cyc/MMA\n", c.name, avg / 148 / 8192);
            }
        }
        run_commit<64, 1024>(d_out);
        run_commit<64, 32>(d_out);
        run_commit<64, 16>(d_out);
        run_commit<64, 8>(d_out);
        run_commit<64, 4>(d_out);
        run_commit<64, 2>(d_out);
        run_commit<128, 1024>(d_out);
        run_commit<128, 8>(d_out);
        run_commit<128, 4>(d_out);
        run_commit<128, 2>(d_out);
        run_commit<256, 1024>(d_out);
        run_commit<256, 4>(d_out);
        run_commit<256, 2>(d_out);
        run_contend<128, 0>(d_out, d_lds);
        run_contend<128, 2>(d_out, d_lds);
        run_contend<128, 4>(d_out, d_lds);
        run_contend<128, 8>(d_out, d_lds);
        run_contend<128, 16>(d_out, d_lds);
        run_contend<256, 0>(d_out, d_lds);
        run_contend<256, 4>(d_out, d_lds);
        run_contend<256, 16>(d_out, d_lds);
        run_contend<64, 0>(d_out, d_lds);
        run_contend<64, 4>(d_out, d_lds);
        run_contend<64, 16>(d_out, d_lds);
        run_contend<32, 0>(d_out, d_lds);
        run_contend<16, 0>(d_out, d_lds);
        run_contend<8, 0>(d_out, d_lds);
        return 0;
    }
    run_seq<128, 192, 128, 64>("seq n1: 128 192 128 64", d_out);
    run_seq<128, 192, 128, 0>("seq n1: 128 192 128", d_out);
    run_seq<192, 256, 64, 0>("seq n2 g0: 192 256 64", d_out);
    run_seq<256, 64, 0, 0>("seq n2 g1: 256 64", d_out);
    run_seq<256, 192, 0, 0>("seq n2 g2: 256 192", d_out);
    run_seq<128, 128, 128, 128>("seq 4x128", d_out);
    run_seq<192, 0, 0, 0>("seq 192", d_out);
    run_seq<256, 256, 0, 0>("seq 256 256", d_out);
    const int smem = 200 * 1024;
    cudaFuncSetAttribute(bench, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 8192;
    for (const Cfg& c : cfgs) {
        bench<<<148, 128, smem>>>(c, iters, d_out);
        bench<<<148, 128, smem>>>(c, iters, d_out);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("%s: %s\n", c.name, cudaGetErrorString(e)); return 1; }
        long long h[148];
        cudaMemcpy(h, d_out, sizeof(h), cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < 148; ++i) avg += h[i];
        avg /= 148;
        const double cyc = avg / iters;
        printf("%-36s %7.1f cyc/MMA  %7.0f MAC/clk/SM\n", c.name, cyc, (double)c.M * c.N * 16 / cyc);
    }
    return 0;
}
