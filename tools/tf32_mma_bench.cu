// tf32_mma_bench.cu -- development microbenchmark: cost of tcgen05.mma.kind::tf32 (M = 128, K = 8) with A in
// TMEM or shared memory, by N and by the number of independent accumulators the issue loop rotates over
// (a dependent chain on one accumulator exposes the MMA latency; independent chains expose its throughput).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_mma_bench.bin tools/tf32_mma_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int NACC, bool A_TMEM, int MODE = 0>
__global__ void bench(long long* cycles, int iters) {
    __shared__ __align__(1024) uint8_t bsm[256 * 32];
    __shared__ __align__(1024) uint8_t asm_[128 * 32];
    __shared__ uint64_t bar, bar2;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x;
    for (int i = tid; i < 256 * 8; i += blockDim.x) reinterpret_cast<float*>(bsm)[i] = 0.5f;
    for (int i = tid; i < 128 * 8; i += blockDim.x) reinterpret_cast<float*>(asm_)[i] = 0.25f;
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1000000;" ::"r"(smem_u32(&bar2)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (tid < 32) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    if (MODE == 6 && tid >= 32) {  // other warps: dependent FMA chains (issue-slot competition)
        float a = tid * 1e-3f, b = 1.0001f;
        for (int it = 0; it < iters * 64; ++it) {
#pragma unroll
            for (int r = 0; r < 16; ++r) a = fmaf(a, b, 0.5f);
        }
        if (a == 1.2345f) cycles[blockIdx.x + 1000] = 1;
    }
    if (MODE == 5 && tid >= 32) {  // warps 1-3: continuous tcgen05.st traffic to other TMEM columns
        const int w = tid / 32;
        uint32_t v[8] = {1, 2, 3, 4, 5, 6, 7, 8};
        for (int it = 0; it < iters * 4; ++it) {
            const uint32_t ta = tm + ((uint32_t)(w * 32) << 16) + 320 + (it & 7) * 16;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(v[0]),
                         "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + 8), "r"(v[0]),
                         "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]));
            asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        }
    }
    if (MODE == 4 && tid == 32) {  // a second issuing warp on its own accumulator (columns 256..)
        constexpr uint32_t idesc = idesc_tf32(128, N);
        const uint64_t bd = desc_sw32(smem_u32(bsm));
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int a = 0; a < NACC; ++a)
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm + 256 + a * N), "r"(tm + 496), "l"(bd), "r"(idesc), "r"(1));
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar2)));
    }
    if (tid == 0) {
        constexpr uint32_t idesc = idesc_tf32(128, N);
        const uint64_t bd = desc_sw32(smem_u32(bsm));
        const uint64_t ad = desc_sw32(smem_u32(asm_));
        extern __shared__ __align__(1024) uint8_t dyn[];
        const uint64_t bdyn = desc_sw32(smem_u32(dyn));
        const uint32_t a_t = tm + 480;  // A in TMEM columns 480..487 (contents irrelevant for timing)
        long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
            if constexpr (MODE >= 1 && MODE != 4) {  // the kernel's per-K-step handshake: wait on a barrier, fence
                asm volatile("{.reg .pred P1; W2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 1; @!P1 bra W2;}" ::"r"(
                    smem_u32(&bar)));
                asm volatile("tcgen05.fence::after_thread_sync;");
            }
            if constexpr (MODE == 3 || MODE == 5 || MODE == 6 || MODE == 7) {
                constexpr uint32_t id2 = idesc_tf32(128, 2 * N), id1 = idesc_tf32(128, N);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk) {
                    const uint64_t bk = MODE == 7 ? bdyn + (uint64_t)(((it * 4 + kk) % 24) * (2 * N * 32 >> 4))
                                                  : bd + (uint64_t)((kk & 1) * (2 * N * 32 >> 4));
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                                 ::"r"(tm), "r"(tm + 256 + 16 * kk), "l"(bk), "r"(id2), "r"(1));
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                                 ::"r"(tm), "r"(tm + 256 + 16 * kk + 8), "l"(bk), "r"(id1), "r"(1));
                }
            }
#pragma unroll
            for (int a = 0; a < (MODE == 3 || MODE == 5 || MODE == 6 || MODE == 7 ? 0 : NACC); ++a) {
                const uint32_t d = tm + a * N;
                if constexpr (A_TMEM)
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                                 ::"r"(d), "r"(a_t), "l"(bd), "r"(idesc), "r"(1));
                else
                    asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;}"
                                 ::"r"(d), "l"(ad), "l"(bd), "r"(idesc), "r"(1));
            }
            if constexpr (MODE >= 2 && MODE != 4)  // commit to a second barrier every iteration
                asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                    smem_u32(&bar2)));
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W;}" ::"r"(
            smem_u32(&bar)));
        long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tm));
}

template <int N, int NACC, bool AT, int MODE = 0>
void run() {
    long long* c;
    cudaMallocManaged(&c, 148 * sizeof(long long));
    const int iters = 2048 / NACC;
    bench<N, NACC, AT, MODE><<<148, 128>>>(c, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("{\"N\": %d, \"acc_chains\": %d, \"A\": \"%s\", \"mode\": %d, \"cycles_per_mma\": %.1f, \"status\": \"%s\"}\n", N,
           NACC, AT ? "tmem" : "smem", MODE, (double)mx / (iters * NACC), cudaGetErrorString(e));
    cudaFree(c);
}

template <int N>
void run6() {  // mode 6 with 24 competing warps (768 threads)
    long long* c;
    cudaMallocManaged(&c, 2000 * sizeof(long long));
    const int iters = 2048 / 8;
    bench<N, 8, true, 6><<<148, 768>>>(c, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("{\"N\": %d, \"mode\": 6, \"competing_warps\": 23, \"cycles_per_mma\": %.1f, \"status\": \"%s\"}\n", N,
           (double)mx / (iters * 8), cudaGetErrorString(e));
    cudaFree(c);
}

template <int N>
void run7() {  // mode 7: B blocks of successive K-steps from a 24-block region (as the conv kernel's resident weights)
    long long* c;
    cudaMallocManaged(&c, 2000 * sizeof(long long));
    const int iters = 2048 / 8;
    const int smem = 24 * 2 * N * 32 + 1024;
    cudaFuncSetAttribute(bench<N, 8, true, 7>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    bench<N, 8, true, 7><<<148, 128, smem>>>(c, iters);
    cudaError_t e = cudaDeviceSynchronize();
    long long mx = 0;
    for (int i = 0; i < 148; ++i) mx = c[i] > mx ? c[i] : mx;
    printf("{\"N\": %d, \"mode\": 7, \"cycles_per_mma\": %.1f, \"status\": \"%s\"}\n", N,
           (double)mx / (iters * 8), cudaGetErrorString(e));
    cudaFree(c);
}

int main() {
    run<16, 1, true>(); run<32, 1, true>(); run<64, 1, true>(); run<128, 1, true>(); run<256, 1, true>();
    run<16, 4, true>(); run<32, 4, true>(); run<64, 4, true>(); run<128, 2, true>();
    run<32, 8, true>(); run<16, 8, true>();
    run<32, 1, false>(); run<32, 4, false>(); run<64, 4, false>(); run<16, 8, false>();
    run<32, 3, true, 1>(); run<32, 3, true, 2>(); run<64, 3, true, 2>(); run<32, 6, true, 2>();
    run<32, 8, true, 3>(); run<16, 8, true, 3>(); run<64, 8, true, 3>();
    run<32, 2, true, 4>(); run<64, 2, true, 4>(); run<16, 2, true, 4>();
    run<32, 8, true, 5>(); run<64, 8, true, 5>();
    run6<32>();
    run7<32>(); run7<64>(); run7<16>();
    return 0;
}
