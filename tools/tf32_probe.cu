// tf32_probe.cu -- development probe for the 3xTF32 tensor-core path: validates, on one
// CTA, the conventions the fp32 implicit-GEMM kernels rely on:
//   * tcgen05.mma.cta_group::1.kind::tf32 with A read from TMEM ([a_tmem], lane = M row, 8 columns = K)
//     and B from shared memory, K-major SWIZZLE_32B (one 32-byte row = the 8 K values of one N row);
//   * A written by the threads with tcgen05.st.32x32b.x8 (thread = TMEM lane);
//   * the split x = hi + lo (hi = cvt.rna.tf32(x), lo = x - hi) and D += Ahi.Bhi + Ahi.Blo + Alo.Bhi
//     giving ~fp32 accuracy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/tf32_probe.bin tools/tf32_probe.cu
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

// SW32 K-major descriptor: start>>4, LBO (unused) = 1, SBO = 256 B (8 rows x 32 B), version 1, layout 6
__device__ __forceinline__ uint64_t desc_sw32(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)(256 >> 4) << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)6 << 61;
    return d;
}
__host__ __device__ constexpr uint32_t idesc_tf32(int M, int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int KSTEPS>
__global__ void probe(const float* A, const float* B, float* D, int mode) {
    // A: [128][KSTEPS*8] row-major, B: [N][KSTEPS*8] row-major, D: [128][N]
    __shared__ __align__(1024) uint8_t bsm[2][KSTEPS][N * 32];  // [hi/lo][kstep] SW32 K-major
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
    for (int i = tid; i < N * KSTEPS * 8; i += blockDim.x) {
        const int n = i / (KSTEPS * 8), k = i % (KSTEPS * 8), ks = k / 8, kk = k % 8;
        const float v = B[n * KSTEPS * 8 + k];
        const float hi = tf32_rna(v), lo = v - hi;
        const int chunk = (kk / 4) ^ ((n >> 2) & 1);
        const int off = n * 32 + chunk * 16 + (kk % 4) * 4;
        *reinterpret_cast<float*>(&bsm[0][ks][off]) = hi;
        *reinterpret_cast<float*>(&bsm[1][ks][off]) = mode == 1 ? v : lo;
    }
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tslot)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // generic smem writes -> async proxy (MMA)
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t tm = tslot;
    // A: thread = lane (M row); columns [128 + 16 ks, +8) hi, [+8, +16) lo
    {
        const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
        for (int ks = 0; ks < KSTEPS; ++ks) {
            uint32_t h[8], l[8];
            for (int k = 0; k < 8; ++k) {
                const float v = A[tid * KSTEPS * 8 + ks * 8 + k];
                const float hi = tf32_rna(v);
                h[k] = __float_as_uint(mode == 1 ? v : hi);
                l[k] = __float_as_uint(v - hi);
            }
            const uint32_t ta = tm + lane_base + 128 + 16 * ks;
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta),
                         "r"(h[0]), "r"(h[1]), "r"(h[2]), "r"(h[3]), "r"(h[4]), "r"(h[5]), "r"(h[6]), "r"(h[7]));
            asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(ta + 8),
                         "r"(l[0]), "r"(l[1]), "r"(l[2]), "r"(l[3]), "r"(l[4]), "r"(l[5]), "r"(l[6]), "r"(l[7]));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (tid == 0) {
        constexpr uint32_t idesc = idesc_tf32(128, N);
        for (int ks = 0; ks < KSTEPS; ++ks) {
            const uint32_t ahi = tm + 128 + 16 * ks, alo = ahi + 8;
            const uint64_t bhi = desc_sw32(smem_u32(&bsm[0][ks][0])), blo = desc_sw32(smem_u32(&bsm[1][ks][0]));
            const uint32_t acc0 = ks > 0;
            asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                         ::"r"(tm), "r"(ahi), "l"(bhi), "r"(idesc), "r"(acc0));
            if (mode != 2) {
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm), "r"(ahi), "l"(blo), "r"(idesc), "r"(1));
                asm volatile("{.reg .pred p; setp.ne.b32 p, %4, 0; tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;}"
                             ::"r"(tm), "r"(alo), "l"(bhi), "r"(idesc), "r"(1));
            }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)));
    }
    asm volatile("{.reg .pred P1; W: mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], 0; @!P1 bra W;}" ::"r"(
        smem_u32(&bar)));
    asm volatile("tcgen05.fence::after_thread_sync;");
    for (int c = 0; c < N; c += 8) {
        uint32_t v[8];
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7])
                     : "r"(tm + ((uint32_t)(warp * 32) << 16) + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        for (int k = 0; k < 8; ++k) D[tid * N + c + k] = __uint_as_float(v[k]);
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tm));
}

template <int N, int KS>
static void run(int mode) {
    const int K = KS * 8;
    float *A, *B, *D;
    cudaMallocManaged(&A, 128 * K * 4);
    cudaMallocManaged(&B, N * K * 4);
    cudaMallocManaged(&D, 128 * N * 4);
    srand(1);
    for (int i = 0; i < 128 * K; ++i) A[i] = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    for (int i = 0; i < N * K; ++i) B[i] = (rand() / (float)RAND_MAX - 0.5f) * 2.f;
    probe<N, KS><<<1, 128>>>(A, B, D, mode);
    cudaError_t e = cudaDeviceSynchronize();
    double maxerr = 0, maxref = 0;
    for (int m = 0; m < 128; ++m)
        for (int n = 0; n < N; ++n) {
            double r = 0;
            for (int k = 0; k < K; ++k) r += (double)A[m * K + k] * B[n * K + k];
            maxerr = fmax(maxerr, fabs(r - D[m * N + n]));
            maxref = fmax(maxref, fabs(r));
        }
    printf("{\"N\": %d, \"K\": %d, \"mode\": \"%s\", \"status\": \"%s\", \"normwise_rel_err\": %.3e}\n", N, K,
           mode == 0 ? "3xtf32" : mode == 1 ? "raw fp32 operands (hw tf32)" : "1xtf32 (hi only)",
           cudaGetErrorString(e), maxerr / maxref);
    cudaFree(A);
    cudaFree(B);
    cudaFree(D);
}

int main() {
    for (int mode = 0; mode < 3; ++mode) {
        run<32, 1>(mode);
        run<16, 4>(mode);
        run<64, 2>(mode);
        run<128, 4>(mode);
    }
    return 0;
}
