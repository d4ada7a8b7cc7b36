// tf32_pair_probe.cu -- development probe: does a CTA-pair (cta_group::2, M = 256) tcgen05.mma.kind::tf32 take
// its A operand from tensor memory (each CTA's own 128 lanes) with B split across the pair, as the 3xTF32
// conv kernel would use it?  D[0, 2N) += A_hi . [B_hi ; B_lo] (CTA 0 holds B_hi, CTA 1 B_lo at the same
// offset), D[0, N) += A_lo . B_hi (each CTA holds half of B_hi's rows).  Prints the normwise error.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_pair_probe.bin tools/tf32_pair_probe.cu
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ float tf32_rna(float x) {
    uint32_t r;
    asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
    return __uint_as_float(r);
}
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)1 << 16) | ((uint64_t)(256 >> 4) << 32) |
           ((uint64_t)1 << 46) | ((uint64_t)6 << 61);
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) probe(const float* A, const float* B, float* D) {
    // A: [256][8], B: [N][8], D: [256][N]
    __shared__ __align__(1024) uint8_t bx[N * 32];      // rank 0: B_hi rows 0..N-1; rank 1: B_lo rows
    __shared__ __align__(1024) uint8_t by[N / 2 * 32];  // rank r: B_hi rows r*N/2 ..
    __shared__ uint64_t full, done;
    __shared__ uint32_t tslot;
    const uint32_t rank = ctarank();
    const int tid = threadIdx.x, warp = tid / 32;
    auto put = [&](uint8_t* blk, int row, int k, float v) {
        const int chunk = (k / 4) ^ ((row >> 2) & 1);
        *reinterpret_cast<float*>(blk + row * 32 + chunk * 16 + (k % 4) * 4) = v;
    };
    for (int i = tid; i < N * 8; i += blockDim.x) {
        const int n = i / 8, k = i % 8;
        const float v = B[n * 8 + k], h = tf32_rna(v);
        put(bx, n, k, rank == 0 ? h : v - h);
        if ((int)(n / (N / 2)) == (int)rank) put(by, n % (N / 2), k, h);
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 2;" ::"r"(smem_u32(&full)));
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&done)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    {  // A rows of this CTA (global rows rank*128 + tid): hi at column 128, lo at 136
        uint32_t h[8], l[8];
        for (int k = 0; k < 8; ++k) {
            const float v = A[(rank * 128 + tid) * 8 + k], hv = tf32_rna(v);
            h[k] = __float_as_uint(hv);
            l[k] = __float_as_uint(v - hv);
        }
        const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + 128;
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta), "r"(h[0]),
                     "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]));
        asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + 8), "r"(l[0]),
                     "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]));
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (tid == 0) {  // both CTAs signal the leader's barrier (the follower remotely)
        uint32_t a = smem_u32(&full), ra;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(a), "r"(0));
        asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(ra) : "memory");
    }
    if (rank == 0 && tid == 0) {
        asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W;}" ::"r"(
            smem_u32(&full)));
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint64_t dx = desc_sw32(smem_u32(bx)), dyd = desc_sw32(smem_u32(by));
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;}"
                     ::"r"(tm), "r"(tm + 128), "l"(dx), "r"(idesc_tf32(256, 2 * N)), "r"(0));
        asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::2.kind::tf32 [%0], [%1], %2, %3, p;}"
                     ::"r"(tm), "r"(tm + 136), "l"(dyd), "r"(idesc_tf32(256, N)), "r"(1));
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&done)), "h"((uint16_t)3));
    }
    asm volatile("{.reg .pred P1; W2: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W2;}" ::"r"(
        smem_u32(&done)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < N; c += 8) {
        uint32_t u[8], w[8];
        const uint32_t ta = tm + ((uint32_t)(warp * 32) << 16) + c;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(u[0]), "=r"(u[1]), "=r"(u[2]), "=r"(u[3]), "=r"(u[4]), "=r"(u[5]), "=r"(u[6]), "=r"(u[7])
                     : "r"(ta));
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(w[0]), "=r"(w[1]), "=r"(w[2]), "=r"(w[3]), "=r"(w[4]), "=r"(w[5]), "=r"(w[6]), "=r"(w[7])
                     : "r"(ta + N));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int k = 0; k < 8; ++k) D[(rank * 128 + tid) * N + c + k] = __uint_as_float(u[k]) + __uint_as_float(w[k]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    cluster_sync();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

template <int N>
static void run() {
    float *A, *B, *D;
    cudaMallocManaged(&A, 256 * 8 * 4);
    cudaMallocManaged(&B, N * 8 * 4);
    cudaMallocManaged(&D, 256 * N * 4);
    srand(3);
    for (int i = 0; i < 256 * 8; ++i) A[i] = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    for (int i = 0; i < N * 8; ++i) B[i] = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    for (int i = 0; i < 256 * N; ++i) D[i] = 12345.f;
    probe<N><<<2, 128>>>(A, B, D);
    cudaError_t e = cudaDeviceSynchronize();
    double me = 0, mr = 0;
    for (int m = 0; m < 256; ++m)
        for (int n = 0; n < N; ++n) {
            double r = 0;
            for (int k = 0; k < 8; ++k) r += (double)A[m * 8 + k] * B[n * 8 + k];
            me = fmax(me, fabs(r - D[m * N + n]));
            mr = fmax(mr, fabs(r));
        }
    printf("{\"N\": %d, \"status\": \"%s\", \"normwise_rel_err\": %.3e}\n", N, cudaGetErrorString(e), me / mr);
}

int main() {
    run<16>();
    run<32>();
    run<64>();
    return 0;
}
