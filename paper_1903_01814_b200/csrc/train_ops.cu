// train_ops.cu -- small kernels of the data-parallel training step (BASELINE
// config 5): the network head (global average pool + linear + softmax
// cross-entropy, forward and backward), SGD with momentum, fp32->bf16 casts.
// Not part of the paper's method; deterministic plain reductions.
#include "common.cuh"

namespace hexconv {

// Per-sample block: global average pool (8 channels per thread, HW split over
// thread slices, fixed-order smem reduction), logits, softmax cross-entropy,
// dlogits.  gap[b][C], dlog[b][K], loss_b[b].
constexpr int HEAD_THREADS = 512;  // C = 256: 16 pixel slices x 32 channel groups per image; 2 blocks per SM
constexpr int HEAD_BATCH = 9;      // loads in flight per thread (C5: 576 pixels / 16 slices = 4 batches)

__global__ void __launch_bounds__(HEAD_THREADS)
head_sample_kernel(const uint4* __restrict__ feat, const float* __restrict__ wl, const float* __restrict__ bl,
                   const int32_t* __restrict__ labels, float* __restrict__ gap, float* __restrict__ dlog,
                   float* __restrict__ loss_b, int B, int HW, int C, int K) {
    extern __shared__ float sh[];  // [slices][C] partial sums, then logits
    const int b = blockIdx.x;
    const int C8 = C / 8;
    const int slices = HEAD_THREADS / C8 > 0 ? HEAD_THREADS / C8 : 1;
    const int tid = threadIdx.x;
    const int c8 = tid % C8, sl = tid / C8;
    if (sl < slices && tid < slices * C8) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        // batches of HEAD_BATCH independent 16-byte loads in flight per thread (latency-bound otherwise: one
        // block per image, a few loads per thread); the sums stay in pixel order
        int i = sl;
        for (; i + (HEAD_BATCH - 1) * slices < HW; i += HEAD_BATCH * slices) {
            uint4 q[HEAD_BATCH];
#pragma unroll
            for (int u = 0; u < HEAD_BATCH; ++u) q[u] = __ldg(feat + ((int64_t)b * HW + i + u * slices) * C8 + c8);
#pragma unroll
            for (int u = 0; u < HEAD_BATCH; ++u) {
                const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&q[u]);
#pragma unroll
                for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(v[j]);
            }
        }
        for (; i < HW; i += slices) {
            const uint4 v4 = __ldg(feat + ((int64_t)b * HW + i) * C8 + c8);
            const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&v4);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(v[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) sh[sl * C + c8 * 8 + j] = acc[j];
    }
    // C8 > HEAD_THREADS: loop the remaining channel groups with one slice
    for (int cc = HEAD_THREADS + tid; cc < C8; cc += HEAD_THREADS) {
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        for (int i = 0; i < HW; ++i) {
            const uint4 v4 = feat[((int64_t)b * HW + i) * C8 + cc];
            const __nv_bfloat16* v = reinterpret_cast<const __nv_bfloat16*>(&v4);
#pragma unroll
            for (int j = 0; j < 8; ++j) acc[j] += __bfloat162float(v[j]);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) sh[cc * 8 + j] = acc[j];
    }
    __syncthreads();
    float* g = sh;  // reduce slices into row 0
    for (int c = tid; c < C; c += HEAD_THREADS) {
        float s = 0.f;
        const int ns = (C8 <= HEAD_THREADS) ? slices : 1;
        for (int k = 0; k < ns; ++k) s += sh[k * C + c];
        g[c] = s / (float)HW;
    }
    __syncthreads();
    for (int c = tid; c < C; c += HEAD_THREADS) gap[(int64_t)b * C + c] = g[c];
    // logits: warp k computes logit k
    float* lg = sh + C;
    const int warp = tid / 32, lane = tid % 32;
    for (int k = warp; k < K; k += HEAD_THREADS / 32) {
        float s = 0.f;
        for (int c = lane; c < C; c += 32) s = fmaf(g[c], wl[(int64_t)k * C + c], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) lg[k] = s + bl[k];
    }
    __syncthreads();
    if (tid == 0) {
        float mx = -INFINITY;
        for (int k = 0; k < K; ++k) mx = fmaxf(mx, lg[k]);
        float z = 0.f;
        for (int k = 0; k < K; ++k) z += expf(lg[k] - mx);
        const int y = labels[b];
        loss_b[b] = logf(z) + mx - lg[y];
        for (int k = 0; k < K; ++k)
            dlog[(int64_t)b * K + k] = (expf(lg[k] - mx) / z - (k == y ? 1.f : 0.f)) / (float)B;
    }
}

// dwl[k][c] = sum_b dlog[b][k] gap[b][c]; dbl[k] = sum_b dlog[b][k]; loss = mean_b loss_b.
// One warp per output: lanes take a fixed strided subset of the samples, then a
// fixed shuffle tree (deterministic).
__global__ void head_param_grad_kernel(const float* __restrict__ gap, const float* __restrict__ dlog,
                                       const float* __restrict__ loss_b, float* __restrict__ dwl,
                                       float* __restrict__ dbl, float* __restrict__ loss, int B, int C, int K) {
    const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
    const int nout = K * C + K + 1;
    if (w >= nout) return;
    float s = 0.f;
    if (w < K * C) {
        const int k = w / C, c = w - k * C;
        for (int b = lane; b < B; b += 32) s = fmaf(dlog[(int64_t)b * K + k], gap[(int64_t)b * C + c], s);
    } else if (w < K * C + K) {
        const int k = w - K * C;
        for (int b = lane; b < B; b += 32) s += dlog[(int64_t)b * K + k];
    } else {
        for (int b = lane; b < B; b += 32) s += loss_b[b];
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane != 0) return;
    if (w < K * C) dwl[w] = s;
    else if (w < K * C + K) dbl[w - K * C] = s;
    else *loss = s / (float)B;
}

// dg[b][c] = (sum_k dlog[b][k] wl[k][c]) / HW: the gradient of every feature pixel of sample b
__global__ void head_dg_kernel(const float* __restrict__ dlog, const float* __restrict__ wl, float* __restrict__ dg,
                               int B, int C, int K, float inv_hw) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= B * C) return;
    const int b = i / C, c = i - b * C;
    float s = 0.f;
    for (int k = 0; k < K; ++k) s = fmaf(dlog[(int64_t)b * K + k], wl[(int64_t)k * C + c], s);
    dg[i] = s * inv_hw;
}

// dfeat[b][hw][c] = dg[b][c] * (feat > 0)   (8 channels per thread; ReLU backward of the last conv)
__global__ void head_dfeat_kernel(const uint4* __restrict__ feat, const float* __restrict__ dg,
                                  uint4* __restrict__ dfeat, int B, int HW, int C8) {
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)B * HW * C8;
    if (idx >= total) return;
    const int c8 = (int)(idx % C8);
    const int b = (int)(idx / ((int64_t)HW * C8));
    const uint4 f4 = feat[idx];
    const uint32_t fw[4] = {f4.x, f4.y, f4.z, f4.w};
    const float4* g4 = reinterpret_cast<const float4*>(dg + ((int64_t)b * C8 + c8) * 8);
    const float4 ga = __ldg(g4), gb = __ldg(g4 + 1);
    const float g[8] = {ga.x, ga.y, ga.z, ga.w, gb.x, gb.y, gb.z, gb.w};
    uint32_t o[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const float f0 = __uint_as_float(fw[j] << 16), f1 = __uint_as_float(fw[j] & 0xffff0000u);
        __nv_bfloat162 h = __floats2bfloat162_rn(f0 > 0.f ? g[2 * j] : 0.f, f1 > 0.f ? g[2 * j + 1] : 0.f);
        o[j] = *reinterpret_cast<uint32_t*>(&h);
    }
    dfeat[idx] = make_uint4(o[0], o[1], o[2], o[3]);
}

size_t head_ws_bytes(int B, int K, int C) {
    return (size_t)(B * C + B * K + B + B * C) * sizeof(float) + 16;
}

hex_status_t head_fwd_bwd(int B, int HW, int C, int K, const void* feat, const float* wl, const float* bl,
                          const int32_t* labels, float* loss, void* dfeat, float* dwl, float* dbl, void* ws,
                          cudaStream_t st) {
    float* gap = (float*)ws;
    float* dlog = gap + (size_t)B * C;
    float* loss_b = dlog + (size_t)B * K;
    float* dg = loss_b + B;
    if (((uintptr_t)dg & 15) != 0) dg = (float*)(((uintptr_t)dg + 15) & ~(uintptr_t)15);
    const int C8 = C / 8;
    const int slices = HEAD_THREADS / C8 > 0 ? HEAD_THREADS / C8 : 1;
    const size_t smem = ((size_t)slices * C + 16) * sizeof(float);
    if (smem > 48 * 1024) return HEX_ERR_UNSUPPORTED;
    head_sample_kernel<<<B, HEAD_THREADS, smem, st>>>((const uint4*)feat, wl, bl, labels, gap, dlog, loss_b, B, HW,
                                                      C, K);
    head_param_grad_kernel<<<ceil_div((int64_t)(K * C + K + 1) * 32, 256), 256, 0, st>>>(gap, dlog, loss_b, dwl, dbl,
                                                                                        loss, B, C, K);
    head_dg_kernel<<<ceil_div((int64_t)B * C, 256), 256, 0, st>>>(dlog, wl, dg, B, C, K, 1.f / (float)HW);
    const int64_t total = (int64_t)B * HW * C8;
    head_dfeat_kernel<<<ceil_div(total, 256), 256, 0, st>>>((const uint4*)feat, dg, (uint4*)dfeat, B, HW, C8);
    count_launch(4);
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

// the same update, four parameters per thread (16-byte loads / stores; 8-byte bf16 stores)
__global__ void sgd4_kernel(int64_t n4, float4* __restrict__ p, const float4* __restrict__ g, float4* __restrict__ m,
                            float lr, float mu, float gs, uint2* __restrict__ pb) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n4) return;
    const float4 gi = g[i], mi0 = m[i], pi0 = p[i];
    float4 mi, pi;
    mi.x = fmaf(mu, mi0.x, gi.x * gs); mi.y = fmaf(mu, mi0.y, gi.y * gs);
    mi.z = fmaf(mu, mi0.z, gi.z * gs); mi.w = fmaf(mu, mi0.w, gi.w * gs);
    pi.x = pi0.x - lr * mi.x; pi.y = pi0.y - lr * mi.y; pi.z = pi0.z - lr * mi.z; pi.w = pi0.w - lr * mi.w;
    m[i] = mi;
    p[i] = pi;
    if (pb) {
        __nv_bfloat162 a = __floats2bfloat162_rn(pi.x, pi.y), b = __floats2bfloat162_rn(pi.z, pi.w);
        pb[i] = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
    }
}

hex_status_t sgd_momentum(int64_t n, float* p, const float* g, float* m, float lr, float mu, float gs, void* pb,
                          cudaStream_t st) {
    if (n == 0) return HEX_OK;
    if (n % 4 == 0 && ((((uintptr_t)p | (uintptr_t)g | (uintptr_t)m) & 15) == 0) && (((uintptr_t)pb & 7) == 0)) {
        sgd4_kernel<<<ceil_div(n / 4, 256), 256, 0, st>>>(n / 4, (float4*)p, (const float4*)g, (float4*)m, lr, mu, gs,
                                                          (uint2*)pb);
        count_launch();
        return last_launch_status();
    }
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

// dx = dy * (y > 0): the ReLU backward for callers whose next op has no fused mask (the autograd
// wrapper's weight gradient needs the masked dy as an operand).  y is the post-ReLU output.
template <typename T>
__global__ void relu_bwd_kernel(int64_t n, const T* __restrict__ dy, const T* __restrict__ y, T* __restrict__ dx) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) dx[i] = (float)y[i] > 0.f ? dy[i] : T(0.f);
}

__global__ void relu_bwd_f32x4_kernel(int64_t n4, const float4* __restrict__ dy, const float4* __restrict__ y,
                                      float4* __restrict__ dx) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
        const float4 g = __ldg(dy + i), v = __ldg(y + i);
        dx[i] = make_float4(v.x > 0.f ? g.x : 0.f, v.y > 0.f ? g.y : 0.f, v.z > 0.f ? g.z : 0.f, v.w > 0.f ? g.w : 0.f);
    }
}

hex_status_t relu_bwd(int64_t n, int dtype, const void* dy, const void* y, void* dx, cudaStream_t st) {
    if (n == 0) return HEX_OK;
    if (dtype == HEX_F32 && (n & 3) == 0 && (((uintptr_t)dy | (uintptr_t)y | (uintptr_t)dx) & 15) == 0) {
        const int64_t n4 = n >> 2;
        int blocks = ceil_div(n4, 256);
        if (blocks > num_sms() * 8) blocks = num_sms() * 8;
        relu_bwd_f32x4_kernel<<<blocks, 256, 0, st>>>(n4, (const float4*)dy, (const float4*)y, (float4*)dx);
    } else if (dtype == HEX_F32)
        relu_bwd_kernel<float><<<ceil_div(n, 256), 256, 0, st>>>(n, (const float*)dy, (const float*)y, (float*)dx);
    else
        relu_bwd_kernel<__nv_bfloat16><<<ceil_div(n, 256), 256, 0, st>>>(
            n, (const __nv_bfloat16*)dy, (const __nv_bfloat16*)y, (__nv_bfloat16*)dx);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
