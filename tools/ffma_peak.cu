// ffma_peak.cu -- FP32 FFMA throughput of this B200 (the CUDA-core roofline of the fp32 conv layers,
// SURVEY.md 8(d) "FFMA 74.4 derived, to be re-measured").
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/ffma_peak.bin tools/ffma_peak.cu
//   tools/ffma_peak.bin            -> one JSON line
//
// Two forms, each with 16 independent accumulator chains per thread (latency hidden by ILP and
// 8 warps per scheduler) and a persistent grid of 148 x 2 CTAs of 512 threads:
//   reg : acc_i = fma(a_i, b, acc_i) with a_i, b in registers -- the form of a convolution's inner loop
//         (weight x activation), three register source operands;
//   imm : acc_i = fma(acc_i, 1.0001f, 0.5f) -- immediate operands.
// FLOPs = 2 per FFMA lane; time = CUDA events around the launch (best of 10 after 3 warm-ups).
// Clocks are whatever the driver gives (no locking); the caller samples nvidia-smi alongside.
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 16;

__global__ void __launch_bounds__(512) ffma_reg(float* out, const float* in, int iters, float b) {
    float acc[CHAINS], a[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) {
        acc[i] = threadIdx.x * 1e-3f + i;
        a[i] = in[(threadIdx.x + i) & 63];  // opaque to the compiler: register operands, not immediates
    }
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(a[i], b, acc[i]);
        b = b * 0.999999f;  // keeps b live across iterations (one FMUL per 128 FFMA)
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += acc[i];
    if (s == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void __launch_bounds__(512) ffma_imm(float* out, int iters) {
    float acc[CHAINS];
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) acc[i] = threadIdx.x * 1e-3f + i;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int r = 0; r < 8; ++r)
#pragma unroll
            for (int i = 0; i < CHAINS; ++i) acc[i] = fmaf(acc[i], 1.0001f, 0.5f);
    }
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) s += acc[i];
    if (s == 1.2345f) out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <typename K>
static float best_ms(K launch) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int i = 0; i < 3; ++i) launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int i = 0; i < 10; ++i) {
        cudaEventRecord(e0);
        launch();
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (ms < best) best = ms;
    }
    return best;
}

int main() {
    int dev = 0, sms = 0, clk_khz = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, dev);
    const int blocks = sms * 2, threads = 512, iters = 4096;
    float *out, *in;
    cudaMalloc(&out, (size_t)blocks * threads * sizeof(float));
    cudaMalloc(&in, 64 * sizeof(float));
    float h[64];
    for (int i = 0; i < 64; ++i) h[i] = 1.0f + i * 1e-5f;
    cudaMemcpy(in, h, sizeof(h), cudaMemcpyHostToDevice);
    const double ffma = (double)blocks * threads * iters * 8 * CHAINS;
    const float ms_reg = best_ms([&] { ffma_reg<<<blocks, threads>>>(out, in, iters, 1.0f); });
    const float ms_imm = best_ms([&] { ffma_imm<<<blocks, threads>>>(out, iters); });
    cudaError_t err = cudaDeviceSynchronize();
    const double tf_reg = 2.0 * ffma / (ms_reg * 1e-3) / 1e12, tf_imm = 2.0 * ffma / (ms_imm * 1e-3) / 1e12;
    const double nominal = 2.0 * sms * 128 * (clk_khz * 1e3) / 1e12;
    printf("{\"ffma_tflops_reg\": %.3f, \"ffma_tflops_imm\": %.3f, \"ms_reg\": %.4f, \"ms_imm\": %.4f, "
           "\"sms\": %d, \"clock_rate_mhz\": %.0f, \"nominal_128_lanes_tflops\": %.3f, \"status\": \"%s\", "
           "\"how\": \"148x2 CTAs x 512 threads, 16 independent FFMA chains per thread, %d x 128 FFMA per "
           "thread; best of 10 CUDA-event timings after 3 warm-ups\"}\n",
           tf_reg, tf_imm, ms_reg, ms_imm, sms, clk_khz / 1e3, nominal, cudaGetErrorString(err), iters);
    cudaFree(out);
    cudaFree(in);
    return err == cudaSuccess ? 0 : 1;
}
