// conv3d.cu -- 3-D hexagonal convolution (Sec. 2 "Software
// Functionalities") through the 2-D entry points.
//
// The kd depth taps of output slice zo read input slices z = sd*zo + kz - (kd-1)/2.
// Unfolding them into channels -- x'[b*Do + zo][(kz, ci)] = x[b][ci][z] (zero
// outside [0, D)) -- turns the 3-D convolution into ONE 2-D hex convolution over
// B*Do images with Cin' = kd*Cin input channels and weights
// w'[co][(kz, ci)][t] = w[co][ci][kz][t]:
//   fwd:       y  = conv2d(x', w')                               (+ bias, ReLU)
//   bwd-data:  dx = fold(conv2d_bwd_data(dy, w'))   (depth col2im, kz ascending)
//   bwd-weight: dw[co][ci][kz][t] = conv2d_bwd_weight(x', dy)[co][(kz, ci)][t]
// so the tcgen05 tap-reuse kernels serve bf16 NDHWC volumes whose Cin'/Cout are
// multiples of 64, and the CUDA-core kernels everything else.  The unfold and
// fold are HBM-bound gathers (16-byte vectors for NDHWC when Cin % 8 == 0).
#include <cstdint>
#include <cstdlib>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {
namespace {

struct C3 {
    int B, Ci, Co, D, H, W, kd, sd, Do, pd;
};

// x (NCDHW) -> x' (NCHW over B*Do images, kd*Ci channels), one element per thread
template <typename T>
__global__ void unfold_ncdhw_kernel(const T* __restrict__ x, T* __restrict__ xu, C3 g) {
    const int64_t HW = (int64_t)g.H * g.W;
    const int64_t total = (int64_t)g.B * g.Do * g.kd * g.Ci * HW;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t p = i % HW;
        int64_t q = i / HW;
        const int c = (int)(q % (g.kd * g.Ci));
        const int64_t img = q / (g.kd * g.Ci);
        const int kz = c / g.Ci, ci = c - kz * g.Ci;
        const int zo = (int)(img % g.Do), b = (int)(img / g.Do);
        const int z = g.sd * zo + kz - g.pd;
        xu[i] = (z >= 0 && z < g.D) ? x[(((int64_t)b * g.Ci + ci) * g.D + z) * HW + p] : T(0.f);
    }
}

// x (NDHWC) -> x' (NHWC, channels (kz, ci)); V-element vectors (V = 8 bf16 / 4 f32 = 16 bytes, or 1)
template <typename T, int V>
__global__ void unfold_ndhwc_kernel(const T* __restrict__ x, T* __restrict__ xu, C3 g) {
    const int CV = g.Ci / V;
    const int64_t HW = (int64_t)g.H * g.W;
    const int64_t total = (int64_t)g.B * g.Do * HW * g.kd * CV;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int cv = (int)(i % CV);
        int64_t q = i / CV;
        const int kz = (int)(q % g.kd);
        q /= g.kd;
        const int64_t p = q % HW;
        const int64_t img = q / HW;
        const int zo = (int)(img % g.Do), b = (int)(img / g.Do);
        const int z = g.sd * zo + kz - g.pd;
        T* dst = xu + ((img * HW + p) * g.kd + kz) * g.Ci + (int64_t)cv * V;
        if constexpr (V * sizeof(T) == 16) {
            uint4 v = make_uint4(0u, 0u, 0u, 0u);
            if (z >= 0 && z < g.D)
                v = *reinterpret_cast<const uint4*>(x + ((((int64_t)b * g.D + z) * HW + p) * g.Ci) + (int64_t)cv * V);
            *reinterpret_cast<uint4*>(dst) = v;
        } else {
            const T* src = x + ((((int64_t)b * g.D + z) * HW + p) * g.Ci) + (int64_t)cv * V;
#pragma unroll
            for (int k = 0; k < V; ++k) dst[k] = (z >= 0 && z < g.D) ? src[k] : T(0.f);
        }
    }
}

// dx'[B*Do images][(kz, ci)] -> dx[b][ci][z] (both layouts, `cl` = channels-last):
// dx = sum over the (kz, zo) with sd*zo + kz - pd = z, kz ascending, fp32
template <typename T>
__global__ void fold_kernel(const T* __restrict__ dxu, T* __restrict__ dx, C3 g, int cl) {
    const int64_t HW = (int64_t)g.H * g.W;
    const int64_t total = (int64_t)g.B * g.Ci * g.D * HW;
    const int Ciu = g.kd * g.Ci;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        int ci, z, b;
        int64_t p;
        if (cl) {  // i = ((b*D + z)*HW + p)*Ci + ci
            ci = (int)(i % g.Ci);
            int64_t q = i / g.Ci;
            p = q % HW;
            q /= HW;
            z = (int)(q % g.D);
            b = (int)(q / g.D);
        } else {  // i = ((b*Ci + ci)*D + z)*HW + p
            p = i % HW;
            int64_t q = i / HW;
            z = (int)(q % g.D);
            q /= g.D;
            ci = (int)(q % g.Ci);
            b = (int)(q / g.Ci);
        }
        float acc = 0.f;
        for (int kz = 0; kz < g.kd; ++kz) {
            const int zz = z - kz + g.pd;  // = sd * zo
            if (zz < 0 || zz % g.sd) continue;
            const int zo = zz / g.sd;
            if (zo >= g.Do) continue;
            const int64_t img = (int64_t)b * g.Do + zo;
            const int c = kz * g.Ci + ci;
            acc += to_f32(cl ? dxu[(img * HW + p) * Ciu + c] : dxu[(img * Ciu + c) * HW + p]);
        }
        dx[i] = from_f32<T>(acc);
    }
}

// w[co][ci][kz][t] -> w'[co][kz*Ci + ci][t]
template <typename T>
__global__ void wperm_kernel(const T* __restrict__ w, T* __restrict__ wu, int Co, int Ci, int kd, int Tn) {
    const int64_t total = (int64_t)Co * Ci * kd * Tn;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(i % Tn);
        int64_t q = i / Tn;
        const int kz = (int)(q % kd);
        q /= kd;
        const int ci = (int)(q % Ci);
        const int co = (int)(q / Ci);
        wu[(((int64_t)co * kd + kz) * Ci + ci) * Tn + t] = w[i];
    }
}

// dw[co][ci][kz][t] (+)= dw'[co][kz*Ci + ci][t]; dbias (+)= dbias' when both given
__global__ void dwperm_kernel(const float* __restrict__ dwu, float* __restrict__ dw, int Co, int Ci, int kd, int Tn,
                              int accumulate, const float* __restrict__ dbu, float* __restrict__ db) {
    const int64_t total = (int64_t)Co * Ci * kd * Tn;
    if (db && dbu) {
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < Co; i += (int64_t)gridDim.x * blockDim.x)
            db[i] = accumulate ? db[i] + dbu[i] : dbu[i];
    }
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(i % Tn);
        int64_t q = i / Tn;
        const int kz = (int)(q % kd);
        q /= kd;
        const int ci = (int)(q % Ci);
        const int co = (int)(q / Ci);
        const float v = dwu[(((int64_t)co * kd + kz) * Ci + ci) * Tn + t];
        dw[i] = accumulate ? dw[i] + v : v;
    }
}

// [B][P][Q][HW] -> [B][Q][P][HW] (NCDHW <-> per-slice NCHW of the B*Do images: P, Q = Do, Co or Co, Do)
template <typename T>
__global__ void swap_mid_kernel(const T* __restrict__ src, T* __restrict__ dst, int B, int P, int Q, int64_t HW) {
    const int64_t total = (int64_t)B * P * Q * HW;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t h = i % HW;
        int64_t r = i / HW;
        const int q = (int)(r % Q);
        r /= Q;
        const int pp = (int)(r % P);
        const int b = (int)(r / P);
        dst[(((int64_t)b * Q + q) * P + pp) * HW + h] = src[i];
    }
}

// tcgen05 path weights: tr = 0: wp[kz*T + t][co][ci] = w[co][ci][kz][t];
// tr = 1 (bwd-data as a forward): wp[kz*T + t][ci][co] = w[co][ci][kd-1-kz][T-1-t]
__global__ void pack3d_kernel(const __nv_bfloat16* __restrict__ w, __nv_bfloat16* __restrict__ wp, int Co, int Ci,
                              int kd, int Tn, int tr) {
    const int64_t total = (int64_t)Co * Ci * kd * Tn;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int t = (int)(i % Tn);
        int64_t q = i / Tn;
        const int kz = (int)(q % kd);
        q /= kd;
        const int ci = (int)(q % Ci);
        const int co = (int)(q / Ci);
        if (!tr) wp[(((int64_t)kz * Tn + t) * Co + co) * Ci + ci] = w[i];
        else wp[(((int64_t)(kd - 1 - kz) * Tn + (Tn - 1 - t)) * Ci + ci) * Co + co] = w[i];
    }
}

inline int grid_for(int64_t total) {
    const int64_t b = (total + 255) / 256;
    return (int)(b < 148 * 16 ? (b < 1 ? 1 : b) : 148 * 16);
}

size_t elt(int dtype) { return dtype == HEX_F32 ? 4 : 2; }
size_t up1k(size_t b) { return (b + 1023) & ~(size_t)1023; }

hex_status_t c3_check(const hex_conv3d_desc_t* d, C3* g, hex_conv2d_desc_t* d2) {
    if (!d) return HEX_ERR_INVALID_ARG;
    if (d->kernel_depth < 1 || (d->kernel_depth & 1) == 0 || d->depth_stride < 1) return HEX_ERR_INVALID_ARG;
    if (d->depth < 1 || d->batch < 1) return HEX_ERR_SHAPE;
    g->B = d->batch; g->Ci = d->in_channels; g->Co = d->out_channels;
    g->D = d->depth; g->H = d->height; g->W = d->width;
    g->kd = d->kernel_depth; g->sd = d->depth_stride; g->pd = (d->kernel_depth - 1) / 2;
    g->Do = (d->depth - 1) / d->depth_stride + 1;
    const int64_t imgs = (int64_t)d->batch * g->Do;
    const int64_t ciu = (int64_t)d->in_channels * d->kernel_depth;
    if (imgs > INT32_MAX || ciu > INT32_MAX) return HEX_ERR_SHAPE;
    d2->batch = (int32_t)imgs;
    d2->in_channels = (int32_t)ciu;
    d2->out_channels = d->out_channels;
    d2->height = d->height; d2->width = d->width;
    d2->kernel_size = d->kernel_size; d2->stride = d->stride; d2->parity = d->parity;
    d2->dtype = d->dtype; d2->layout = d->layout;
    int32_t Ho, Wo, po;
    return hex_output_shape(d->height, d->width, d->stride, d->parity, &Ho, &Wo, &po);
}

template <typename T>
void launch_unfold(const void* x, void* xu, const C3& g, int layout, cudaStream_t st) {
    if (layout == HEX_NHWC) {
        constexpr int V16 = 16 / sizeof(T);
        const bool vec = g.Ci % V16 == 0 && ((uintptr_t)x & 15) == 0 && ((uintptr_t)xu & 15) == 0;
        const int64_t total = (int64_t)g.B * g.Do * g.H * g.W * g.kd * (g.Ci / (vec ? V16 : 1));
        if (vec) unfold_ndhwc_kernel<T, V16><<<grid_for(total), 256, 0, st>>>((const T*)x, (T*)xu, g);
        else unfold_ndhwc_kernel<T, 1><<<grid_for(total), 256, 0, st>>>((const T*)x, (T*)xu, g);
    } else {
        const int64_t total = (int64_t)g.B * g.Do * g.kd * g.Ci * g.H * g.W;
        unfold_ncdhw_kernel<T><<<grid_for(total), 256, 0, st>>>((const T*)x, (T*)xu, g);
    }
    count_launch();
}

hex_status_t unfold(const void* x, void* xu, const C3& g, int dtype, int layout, cudaStream_t st) {
    if (dtype == HEX_F32) launch_unfold<float>(x, xu, g, layout, st);
    else launch_unfold<__nv_bfloat16>(x, xu, g, layout, st);
    return last_launch_status();
}

hex_status_t swap_mid(const void* src, void* dst, int B, int P, int Q, int64_t HW, int dtype, cudaStream_t st) {
    const int64_t total = (int64_t)B * P * Q * HW;
    if (dtype == HEX_F32)
        swap_mid_kernel<float><<<grid_for(total), 256, 0, st>>>((const float*)src, (float*)dst, B, P, Q, HW);
    else
        swap_mid_kernel<__nv_bfloat16><<<grid_for(total), 256, 0, st>>>((const __nv_bfloat16*)src,
                                                                         (__nv_bfloat16*)dst, B, P, Q, HW);
    count_launch();
    return last_launch_status();
}

// bytes of the output volume (B*Do*Co*Ho*Wo) -- staged in the workspace for NCDHW, whose
// [b][co][zo] order differs from the 2-D call's [b*Do + zo][co]
size_t out_vol_bytes(const hex_conv3d_desc_t* d, const C3& g) {
    int32_t Ho, Wo, po;
    if (hex_output_shape(d->height, d->width, d->stride, d->parity, &Ho, &Wo, &po) != HEX_OK) return 0;
    return (size_t)g.B * g.Do * g.Co * Ho * Wo * elt(d->dtype);
}

// the depth-in-K-loop tcgen05 path: bf16 NDHWC, in-plane stride 1, channels multiples of 64
bool c3_tc_ok(const hex_conv3d_desc_t* d, int Cin, int Cout, int Dout, Geom* g) {
    if (d->dtype != HEX_BF16 || d->layout != HEX_NHWC || d->stride != 1 || Cin % 64 || Cout % 64) return false;
    g->B = d->batch; g->H = d->height; g->W = d->width;
    g->n = d->kernel_size; g->s = 1; g->parity = d->parity; g->T = hex_num_taps(d->kernel_size);
    int32_t po;
    if (hex_output_shape(g->H, g->W, 1, g->parity, &g->Ho, &g->Wo, &po) != HEX_OK) return false;
    return tc_conv3d_supported(*g, Cin, Cout, Dout);
}

bool a16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

hex_status_t wperm(const void* w, void* wu, const C3& g, int Tn, int dtype, cudaStream_t st) {
    const int64_t total = (int64_t)g.Co * g.Ci * g.kd * Tn;
    if (dtype == HEX_F32)
        wperm_kernel<float><<<grid_for(total), 256, 0, st>>>((const float*)w, (float*)wu, g.Co, g.Ci, g.kd, Tn);
    else
        wperm_kernel<__nv_bfloat16><<<grid_for(total), 256, 0, st>>>((const __nv_bfloat16*)w, (__nv_bfloat16*)wu,
                                                                      g.Co, g.Ci, g.kd, Tn);
    count_launch();
    return last_launch_status();
}

}  // namespace
}  // namespace hexconv

using namespace hexconv;

hex_status_t hex_conv3d_output_shape(const hex_conv3d_desc_t* d, int32_t* Do, int32_t* Ho, int32_t* Wo) {
    if (!Do || !Ho || !Wo) return HEX_ERR_INVALID_ARG;
    C3 g;
    hex_conv2d_desc_t d2;
    hex_status_t st = c3_check(d, &g, &d2);
    if (st != HEX_OK) return st;
    int32_t po;
    st = hex_output_shape(d->height, d->width, d->stride, d->parity, Ho, Wo, &po);
    *Do = g.Do;
    return st;
}

hex_status_t hex_conv3d_workspace_size(const hex_conv3d_desc_t* d, int32_t pass, size_t* bytes) {
    if (!bytes) return HEX_ERR_INVALID_ARG;
    C3 g;
    hex_conv2d_desc_t d2;
    hex_status_t st = c3_check(d, &g, &d2);
    if (st != HEX_OK) return st;
    size_t ws2 = 0;
    st = hex_conv2d_workspace_size(&d2, pass, &ws2);
    if (st != HEX_OK) return st;
    const int Tn = hex_num_taps(d->kernel_size);
    const size_t vol = (size_t)d2.batch * d2.in_channels * d->height * d->width * elt(d->dtype);  // x' / dx'
    const size_t wb = (size_t)g.Co * g.Ci * g.kd * Tn * (pass == 2 ? sizeof(float) : elt(d->dtype));
    const size_t dbb = pass == 2 ? up1k((size_t)g.Co * sizeof(float)) : 0;
    const size_t stage = d->layout == HEX_NHWC ? 0 : up1k(out_vol_bytes(d, g));  // NCDHW y / dy reorder
    *bytes = up1k(vol) + up1k(wb) + dbb + stage + ws2 + 2048;
    return HEX_OK;
}

hex_status_t hex_conv3d_fwd(const hex_conv3d_desc_t* d, const void* x, const void* w, const float* bias,
                            int32_t fuse_relu, void* y, void* ws, size_t ws_bytes, hex_stream_t stream) {
    C3 g;
    hex_conv2d_desc_t d2;
    hex_status_t st = c3_check(d, &g, &d2);
    if (st != HEX_OK) return st;
    if (!x || !w || !y) return HEX_ERR_INVALID_ARG;
    size_t need = 0;
    if ((st = hex_conv3d_workspace_size(d, 0, &need)) != HEX_OK) return st;
    if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const int Tn = hex_num_taps(d->kernel_size);
    uint8_t* p = (uint8_t*)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    Geom tg;
    if (c3_tc_ok(d, g.Ci, g.Co, g.Do, &tg) && a16(x) && a16(y) && a16(w) && (!bias || a16(bias)) &&
        !sw_on("HEXCONV_CONV3D_UNFOLD")) {
        // depth taps in the K loop of the tcgen05 tap-reuse kernel: no unfolded copy
        const int64_t total = (int64_t)g.Co * g.Ci * g.kd * Tn;
        pack3d_kernel<<<grid_for(total), 256, 0, s>>>((const __nv_bfloat16*)w, (__nv_bfloat16*)p, g.Co, g.Ci, g.kd,
                                                       Tn, 0);
        count_launch();
        if ((st = last_launch_status()) != HEX_OK) return st;
        TcConvArgs a{};
        a.g = tg; a.Cin = g.Ci; a.Cout = g.Co;
        a.x = x; a.wpack = p; a.bias = bias; a.y = y; a.relu_y = nullptr; a.relu = fuse_relu;
        return tc_conv3d_fwd(a, g.D, g.Do, g.sd, g.kd, s);
    }
    void* xu = p;
    p += up1k((size_t)d2.batch * d2.in_channels * d->height * d->width * elt(d->dtype));
    void* wu = p;
    p += up1k((size_t)g.Co * g.Ci * g.kd * Tn * elt(d->dtype));
    void* y2 = y;  // NCDHW: the 2-D call writes [b*Do + zo][co] planes, reordered to [b][co][zo] below
    if (d->layout != HEX_NHWC) {
        y2 = p;
        p += up1k(out_vol_bytes(d, g));
    }
    if ((st = unfold(x, xu, g, d->dtype, d->layout, s)) != HEX_OK) return st;
    if ((st = wperm(w, wu, g, Tn, d->dtype, s)) != HEX_OK) return st;
    st = hex_conv2d_fwd(&d2, xu, wu, bias, fuse_relu, y2, p, ws_bytes - (size_t)(p - (uint8_t*)ws), stream);
    if (st != HEX_OK || d->layout == HEX_NHWC) return st;
    const int64_t HWo = (int64_t)(out_vol_bytes(d, g) / elt(d->dtype)) / ((int64_t)g.B * g.Do * g.Co);
    return swap_mid(y2, y, g.B, g.Do, g.Co, HWo, d->dtype, s);
}

hex_status_t hex_conv3d_bwd_data(const hex_conv3d_desc_t* d, const void* dy, const void* w, void* dx, void* ws,
                                 size_t ws_bytes, hex_stream_t stream) {
    C3 g;
    hex_conv2d_desc_t d2;
    hex_status_t st = c3_check(d, &g, &d2);
    if (st != HEX_OK) return st;
    if (!dy || !w || !dx) return HEX_ERR_INVALID_ARG;
    size_t need = 0;
    if ((st = hex_conv3d_workspace_size(d, 1, &need)) != HEX_OK) return st;
    if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const int Tn = hex_num_taps(d->kernel_size);
    uint8_t* p = (uint8_t*)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    Geom tg;
    if (g.sd == 1 && c3_tc_ok(d, g.Co, g.Ci, g.D, &tg) && a16(dy) && a16(dx) && a16(w) &&
        !sw_on("HEXCONV_CONV3D_UNFOLD")) {
        // stride 1: dx = the forward of dy with depth- and tap-reversed, channel-transposed weights
        // (the 3-D form of DESIGN.md P18), depth taps in the K loop
        const int64_t total = (int64_t)g.Co * g.Ci * g.kd * Tn;
        pack3d_kernel<<<grid_for(total), 256, 0, s>>>((const __nv_bfloat16*)w, (__nv_bfloat16*)p, g.Co, g.Ci, g.kd,
                                                       Tn, 1);
        count_launch();
        if ((st = last_launch_status()) != HEX_OK) return st;
        TcConvArgs a{};
        a.g = tg; a.Cin = g.Co; a.Cout = g.Ci;
        a.x = dy; a.wpack = p; a.bias = nullptr; a.y = dx; a.relu_y = nullptr; a.relu = 0;
        return tc_conv3d_fwd(a, g.D, g.D, 1, g.kd, s);
    }
    void* dxu = p;
    p += up1k((size_t)d2.batch * d2.in_channels * d->height * d->width * elt(d->dtype));
    void* wu = p;
    p += up1k((size_t)g.Co * g.Ci * g.kd * Tn * elt(d->dtype));
    const void* dy2 = dy;  // NCDHW: reorder dy [b][co][zo] -> [b*Do + zo][co] planes for the 2-D call
    if (d->layout != HEX_NHWC) {
        const int64_t HWo = (int64_t)(out_vol_bytes(d, g) / elt(d->dtype)) / ((int64_t)g.B * g.Do * g.Co);
        if ((st = swap_mid(dy, p, g.B, g.Co, g.Do, HWo, d->dtype, s)) != HEX_OK) return st;
        dy2 = p;
        p += up1k(out_vol_bytes(d, g));
    }
    if ((st = wperm(w, wu, g, Tn, d->dtype, s)) != HEX_OK) return st;
    st = hex_conv2d_bwd_data(&d2, dy2, wu, nullptr, dxu, p, ws_bytes - (size_t)(p - (uint8_t*)ws), stream);
    if (st != HEX_OK) return st;
    const int64_t total = (int64_t)g.B * g.Ci * g.D * g.H * g.W;
    const int cl = d->layout == HEX_NHWC;
    if (d->dtype == HEX_F32)
        fold_kernel<float><<<grid_for(total), 256, 0, s>>>((const float*)dxu, (float*)dx, g, cl);
    else
        fold_kernel<__nv_bfloat16><<<grid_for(total), 256, 0, s>>>((const __nv_bfloat16*)dxu, (__nv_bfloat16*)dx, g,
                                                                    cl);
    count_launch();
    return last_launch_status();
}

hex_status_t hex_conv3d_bwd_weight(const hex_conv3d_desc_t* d, const void* x, const void* dy, float* dw, float* dbias,
                                   int32_t accumulate, void* ws, size_t ws_bytes, hex_stream_t stream) {
    C3 g;
    hex_conv2d_desc_t d2;
    hex_status_t st = c3_check(d, &g, &d2);
    if (st != HEX_OK) return st;
    if (!x || !dy || !dw) return HEX_ERR_INVALID_ARG;
    size_t need = 0;
    if ((st = hex_conv3d_workspace_size(d, 2, &need)) != HEX_OK) return st;
    if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    const int Tn = hex_num_taps(d->kernel_size);
    uint8_t* p = (uint8_t*)(((uintptr_t)ws + 1023) & ~(uintptr_t)1023);
    void* xu = p;
    p += up1k((size_t)d2.batch * d2.in_channels * d->height * d->width * elt(d->dtype));
    float* dwu = (float*)p;
    p += up1k((size_t)g.Co * g.Ci * g.kd * Tn * sizeof(float));
    float* dbu = (float*)p;  // fresh dbias, added by dwperm_kernel when accumulating
    p += up1k((size_t)g.Co * sizeof(float));
    Geom tg;
    if (c3_tc_ok(d, g.Ci, g.Co, g.Do, &tg) && g.Co % 128 == 0 && a16(x) && a16(dy) &&
        !sw_on("HEXCONV_CONV3D_UNFOLD")) {
        tg.B = g.B * g.Do;  // output slices
        if (tc_wgrad_tr_supported(tg, g.Ci * g.kd, g.Co)) {
            // depth taps in the units of the tcgen05 tap-reuse weight gradient: no unfolded copy of x; the
            // partials come out in the unfolded (kz, ci) channel order, permuted by dwperm below
            TcWgradArgs a{};
            a.g = tg; a.Cin = g.Ci; a.Cout = g.Co; a.x = x; a.dy = dy; a.dw = dwu; a.dbias = dbias ? dbu : nullptr;
            a.accumulate = 0;
            const TrDepth dz{g.kd, g.D, g.Do, g.sd};
            st = tc_conv3d_wgrad(a, dz, p, ws_bytes - (size_t)(p - (uint8_t*)ws), s);
            if (st != HEX_OK) return st;
            const int64_t total = (int64_t)g.Co * g.Ci * g.kd * Tn;
            dwperm_kernel<<<grid_for(total), 256, 0, s>>>(dwu, dw, g.Co, g.Ci, g.kd, Tn, accumulate, dbu, dbias);
            count_launch();
            return last_launch_status();
        }
    }
    const void* dy2 = dy;
    if (d->layout != HEX_NHWC) {
        const int64_t HWo = (int64_t)(out_vol_bytes(d, g) / elt(d->dtype)) / ((int64_t)g.B * g.Do * g.Co);
        if ((st = swap_mid(dy, p, g.B, g.Co, g.Do, HWo, d->dtype, s)) != HEX_OK) return st;
        dy2 = p;
        p += up1k(out_vol_bytes(d, g));
    }
    if ((st = unfold(x, xu, g, d->dtype, d->layout, s)) != HEX_OK) return st;
    st = hex_conv2d_bwd_weight(&d2, xu, dy2, dwu, dbias ? dbu : nullptr, 0, p,
                               ws_bytes - (size_t)(p - (uint8_t*)ws), stream);
    if (st != HEX_OK) return st;
    const int64_t total = (int64_t)g.Co * g.Ci * g.kd * Tn;
    dwperm_kernel<<<grid_for(total), 256, 0, s>>>(dwu, dw, g.Co, g.Ci, g.kd, Tn, accumulate, dbu, dbias);
    count_launch();
    return last_launch_status();
}
