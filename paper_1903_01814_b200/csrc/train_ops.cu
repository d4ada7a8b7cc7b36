// train_ops.cu -- small kernels of the data-parallel training step (BASELINE
// config 5): the network head (global average pool + linear + softmax
// cross-entropy, forward and backward), SGD with momentum, fp32->bf16 casts.
// Not part of the paper's method; deterministic plain reductions.
#include "common.cuh"

namespace hexconv {

// gap[b][c] = mean_hw feat[b][hw][c]   (feat bf16 NHWC)
__global__ void gap_kernel(const __nv_bfloat16* __restrict__ feat, float* __restrict__ gap, int HW, int C) {
    const int b = blockIdx.x;
    for (int c = threadIdx.x; c < C; c += blockDim.x) {
        const __nv_bfloat16* p = feat + (int64_t)b * HW * C + c;
        float s = 0.f;
        for (int i = 0; i < HW; ++i) s += __bfloat162float(p[(int64_t)i * C]);
        gap[(int64_t)b * C + c] = s / (float)HW;
    }
}

// One block: logits, softmax CE, dlogits, dwl, dbl, dgap.
__global__ void head_kernel(const float* __restrict__ gap, const float* __restrict__ wl, const float* __restrict__ bl,
                            const int32_t* __restrict__ labels, float* __restrict__ loss, float* __restrict__ dwl,
                            float* __restrict__ dbl, float* __restrict__ dlog, float* __restrict__ dgap,
                            int B, int C, int K) {
    extern __shared__ float sh[];  // [B*K] dlogits, then [blockDim] reduction scratch
    float* dl = sh;
    float* red = sh + B * K;
    // logits and per-sample loss
    float my_loss = 0.f;
    for (int b = threadIdx.x; b < B; b += blockDim.x) {
        float lg[8];
        float mx = -INFINITY;
        for (int k = 0; k < K; ++k) {
            float s = bl[k];
            for (int c = 0; c < C; ++c) s = fmaf(gap[(int64_t)b * C + c], wl[(int64_t)k * C + c], s);
            lg[k] = s;
            mx = fmaxf(mx, s);
        }
        float z = 0.f;
        for (int k = 0; k < K; ++k) z += expf(lg[k] - mx);
        const int y = labels[b];
        my_loss += (logf(z) + mx - lg[y]);
        for (int k = 0; k < K; ++k) {
            const float pk = expf(lg[k] - mx) / z;
            dl[b * K + k] = (pk - (k == y ? 1.f : 0.f)) / (float)B;
        }
    }
    red[threadIdx.x] = my_loss;
    __syncthreads();
    if (threadIdx.x == 0) {
        float s = 0.f;
        for (int i = 0; i < (int)blockDim.x; ++i) s += red[i];
        *loss = s / (float)B;
    }
    // dwl[k][c] = sum_b dl[b][k] gap[b][c]; dbl[k] = sum_b dl[b][k]
    for (int i = threadIdx.x; i < K * C; i += blockDim.x) {
        const int k = i / C, c = i % C;
        float s = 0.f;
        for (int b = 0; b < B; ++b) s = fmaf(dl[b * K + k], gap[(int64_t)b * C + c], s);
        dwl[i] = s;
    }
    for (int k = threadIdx.x; k < K; k += blockDim.x) {
        float s = 0.f;
        for (int b = 0; b < B; ++b) s += dl[b * K + k];
        dbl[k] = s;
    }
    // dgap[b][c] = sum_k dl[b][k] wl[k][c]
    for (int i = threadIdx.x; i < B * C; i += blockDim.x) {
        const int b = i / C, c = i % C;
        float s = 0.f;
        for (int k = 0; k < K; ++k) s = fmaf(dl[b * K + k], wl[(int64_t)k * C + c], s);
        dgap[i] = s;
    }
    for (int i = threadIdx.x; i < B * K; i += blockDim.x) dlog[i] = dl[i];
}

// dfeat[b][hw][c] = dgap[b][c] / HW * (feat > 0)   (8 channels per thread)
__global__ void head_dfeat_kernel(const uint4* __restrict__ feat, const float* __restrict__ dgap,
                                  uint4* __restrict__ dfeat, int B, int HW, int C8) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)B * HW * C8;
    if (idx >= total) return;
    const int c8 = (int)(idx % C8);
    const int b = (int)(idx / ((int64_t)HW * C8));
    uint4 f4 = feat[idx];
    const __nv_bfloat16* f = reinterpret_cast<const __nv_bfloat16*>(&f4);
    uint4 o4;
    __nv_bfloat16* o = reinterpret_cast<__nv_bfloat16*>(&o4);
    const float inv = 1.f / (float)HW;
    const float* dg = dgap + (int64_t)b * C8 * 8 + c8 * 8;
#pragma unroll
    for (int j = 0; j < 8; ++j) o[j] = __float2bfloat16_rn(__bfloat162float(f[j]) > 0.f ? dg[j] * inv : 0.f);
    dfeat[idx] = o4;
}

size_t head_ws_bytes(int B, int K, int C) {
    return (size_t)(B * C + B * C + B * K) * sizeof(float);
}

hex_status_t head_fwd_bwd(int B, int HW, int C, int K, const void* feat, const float* wl, const float* bl,
                          const int32_t* labels, float* loss, void* dfeat, float* dwl, float* dbl, void* ws,
                          cudaStream_t st) {
    float* gap = (float*)ws;
    float* dgap = gap + (size_t)B * C;
    float* dlog = dgap + (size_t)B * C;
    gap_kernel<<<B, 256, 0, st>>>((const __nv_bfloat16*)feat, gap, HW, C);
    const int threads = 256;
    head_kernel<<<1, threads, (B * K + threads) * sizeof(float), st>>>(gap, wl, bl, labels, loss, dwl, dbl, dlog,
                                                                         dgap, B, C, K);
    const int64_t total = (int64_t)B * HW * (C / 8);
    head_dfeat_kernel<<<ceil_div(total, 256), 256, 0, st>>>((const uint4*)feat, dgap, (uint4*)dfeat, B, HW, C / 8);
    count_launch(3);
    return last_launch_status();
}

__global__ void sgd_kernel(int64_t n, float* __restrict__ p, const float* __restrict__ g, float* __restrict__ m,
                           float lr, float mu, float gs, __nv_bfloat16* __restrict__ pb) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    const float gi = g[i] * gs;
    const float mi = fmaf(mu, m[i], gi);
    m[i] = mi;
    const float pi = p[i] - lr * mi;
    p[i] = pi;
    if (pb) pb[i] = __float2bfloat16_rn(pi);
}

hex_status_t sgd_momentum(int64_t n, float* p, const float* g, float* m, float lr, float mu, float gs, void* pb,
                          cudaStream_t st) {
    if (n == 0) return HEX_OK;
    sgd_kernel<<<ceil_div(n, 256), 256, 0, st>>>(n, p, g, m, lr, mu, gs, (__nv_bfloat16*)pb);
    count_launch();
    return last_launch_status();
}

__global__ void cast_kernel(int64_t n, const float* __restrict__ s, __nv_bfloat16* __restrict__ d) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) d[i] = __float2bfloat16_rn(s[i]);
}

hex_status_t cast_f32_bf16(int64_t n, const float* s, void* d, cudaStream_t st) {
    if (n == 0) return HEX_OK;
    cast_kernel<<<ceil_div(n, 256), 256, 0, st>>>(n, s, (__nv_bfloat16*)d);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
