// wbw.cu -- development microbenchmark: HBM write bandwidth of store flavours on B200
// (st.global.v4, st.global.cs.v4, 32-byte st.global.v8, TMA bulk smem->global, cudaMemsetAsync).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void st_v4(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(1u, 2u, 3u, 4u);
}
__global__ void st_cs_v4(uint4* p, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        __stcs(p + i, make_uint4(1u, 2u, 3u, 4u));
}
__global__ void st_v8(uint4* p, size_t n2) {  // n2 = number of 32-byte units
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
        float* a = reinterpret_cast<float*>(p + 2 * i);
        asm volatile("st.global.v8.f32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(a), "f"(1.f), "f"(2.f), "f"(3.f),
                     "f"(4.f), "f"(5.f), "f"(6.f), "f"(7.f), "f"(8.f)
                     : "memory");
    }
}
__global__ void bulk_store(uint8_t* p, size_t bytes) {
    extern __shared__ __align__(128) uint8_t sm[];
    constexpr int CH = 32768;
    for (int i = threadIdx.x; i < CH / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(sm)[i] = i;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t s = (uint32_t)__cvta_generic_to_shared(sm);
        int inflight = 0;
        for (size_t off = (size_t)blockIdx.x * CH; off < bytes; off += (size_t)gridDim.x * CH) {
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(p + off), "r"(s),
                         "r"(CH)
                         : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (++inflight >= 6) {
                asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
                inflight = 4;
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

int main() {
    const size_t bytes = (size_t)2 << 30;
    uint8_t* d;
    cudaMalloc(&d, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    auto run = [&](const char* name, auto fn) {
        fn();
        cudaDeviceSynchronize();
        cudaEventRecord(a);
        for (int i = 0; i < 10; ++i) fn();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        printf("%-28s %8.1f GB/s  (%s)\n", name, bytes * 10 / (ms / 1e3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    };
    const size_t n16 = bytes / 16;
    run("st.global.v4 (148x8 x 256)", [&] { st_v4<<<148 * 8, 256>>>((uint4*)d, n16); });
    run("st.global.v4 (148x16 x 512)", [&] { st_v4<<<148 * 16, 512>>>((uint4*)d, n16); });
    run("st.global.cs.v4", [&] { st_cs_v4<<<148 * 8, 256>>>((uint4*)d, n16); });
    run("st.global.v4 16 warps/SM", [&] { st_v4<<<148 * 2, 256>>>((uint4*)d, n16); });
    run("st.global.v4 8 warps/SM", [&] { st_v4<<<148, 256>>>((uint4*)d, n16); });
    run("st.global.v8 16 warps/SM", [&] { st_v8<<<148 * 2, 256>>>((uint4*)d, n16 / 2); });
    run("st.global.v8 (32 B)", [&] { st_v8<<<148 * 8, 256>>>((uint4*)d, n16 / 2); });
    cudaFuncSetAttribute(bulk_store, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    run("TMA bulk store 32 KB x148", [&] { bulk_store<<<148, 128, 32768>>>(d, bytes); });
    run("TMA bulk store 32 KB x296", [&] { bulk_store<<<296, 128, 32768>>>(d, bytes); });
    run("cudaMemsetAsync", [&] { cudaMemsetAsync(d, 0, bytes); });
    return 0;
}
