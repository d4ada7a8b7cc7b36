// kernels.h -- internal launcher interfaces between the C ABI (abi.cu) and the
// kernel translation units.  Not installed; not part of the public ABI.
#pragma once
#include "common.cuh"
#include "geometry.cuh"

namespace hexconv {

struct DirectConvArgs {
    Geom g;
    int Cin, Cout, dtype;
    Strides4 sx, sy;  // sx: x / dx (input grid), sy: y / dy (output grid)
    const void* x;
    const void* w;
    const float* bias;
    void* y;
    const void* dy;
    const void* relu_y;
    void* dx;
    float* dw;
    float* dbias;
    int relu, accumulate;
};

hex_status_t direct_conv_fwd(const DirectConvArgs& a, cudaStream_t st);
hex_status_t direct_conv_bwd_data(const DirectConvArgs& a, cudaStream_t st);
hex_status_t direct_conv_bwd_weight(const DirectConvArgs& a, void* ws, cudaStream_t st);
size_t direct_wgrad_ws_bytes(const Geom& g, int Cin, int Cout);
hex_status_t launch_gather_map(int32_t* map, const Geom& g, cudaStream_t st);

struct PoolArgs {
    Geom g;
    int C, dtype, layout, mode;
    Strides4 sx, sy;
    const void* x;
    void* y;
    uint8_t* argmax;
    const void* dy;
    const uint8_t* argmax_in;
    void* dx;
};
hex_status_t pool_fwd(const PoolArgs& a, cudaStream_t st);
// bf16 NHWC max pool n = 1, s = 2, C % 64 == 0: TMA-staged bands (pool_tma.cu)
bool pool_tma_fwd_supported(const PoolArgs& a);
hex_status_t pool_tma_fwd(const PoolArgs& a, cudaStream_t st);
// NCHW plane-staged pools (plane_kernels.cu); return false when the shape is not covered
bool pool_plane_fwd(const PoolArgs& a, cudaStream_t st);
bool pool_plane_bwd(const PoolArgs& a, cudaStream_t st);
hex_status_t pool_bwd(const PoolArgs& a, cudaStream_t st);
// NCHW n = 1, stride 2 max / avg pool forward (pool_nchw.cu)
bool pool_n1s2_nchw_supported(const PoolArgs& a);
hex_status_t pool_n1s2_nchw_fwd(const PoolArgs& a, cudaStream_t st);
// NCHW n = 1, stride 2 backward with the ReLU backward fused (dx *= relu_y > 0; relu_y may be null);
// false when the shape is not covered (plane_kernels.cu)
bool pool_plane_bwd_n1s2(const PoolArgs& a, const void* relu_y, cudaStream_t st);

// tcgen05 implicit-GEMM path (bf16 NHWC, stride 1).
struct TcConvArgs {
    Geom g;
    int Cin, Cout;
    const void* x;      // bf16 NHWC [B][H][W][Cin]
    const void* wpack;  // bf16 [T][Cout][Cin] (tap-major, K-major rows)
    const float* bias;
    void* y;            // bf16 NHWC [B][H][W][Cout]
    const void* relu_y; // optional bf16 NHWC [B][H][W][Cout] mask source
    int relu;
};
bool tc_conv_supported(const Geom& g, int Cin, int Cout);
bool tc_conv_fwd_supported(const Geom& g, int Cin, int Cout);  // also stride 2
// strided.cu: dy of a stride-s layer scattered onto the full grid (bf16 NHWC, C % 8 == 0)
hex_status_t lattice_upsample(const void* dy, void* up, const Geom& g, int C, cudaStream_t st);
bool tc_fwd_tr_supported(const Geom& g, int Cin, int Cout);  // tap-reuse forward (tc_fwd_tr.cu)
hex_status_t tc_fwd_tr(const TcConvArgs& a, cudaStream_t st);
// fused maxpool_{n=1,s=2}(relu(conv(x) + bias)) (tc_fwd_tr.cu); the conv output is not materialised
// strided bf16 NHWC backward-data by phase classes on the tensor cores (lat_dgrad.cu)
bool lat_dgrad_supported(const Geom& g, int Cin, int Cout);
size_t lat_dgrad_ws_bytes(const Geom& g, int Cin, int Cout);
hex_status_t lat_dgrad(const Geom& g, int Cin, int Cout, const void* dy, const void* w, const void* relu_y, void* dx,
                       void* ws, size_t ws_bytes, cudaStream_t st);
bool tc_conv_pool_supported(const Geom& g, int Cin, int Cout, int mode);  // fused conv + ReLU + pool (max / avg)
bool tc_conv3d_supported(const Geom& g, int Cin, int Cout, int Do);
hex_status_t tc_conv3d_fwd(const TcConvArgs& a, int D, int Do, int sd, int kd, cudaStream_t st);
hex_status_t tc_conv_pool(const TcConvArgs& a, int mode, void* y_pool, uint8_t* argmax, cudaStream_t st);
hex_status_t tc_conv_fwd(const TcConvArgs& a, cudaStream_t st);
hex_status_t tc_pack_weights(const void* w, void* wpack, int Cout, int Cin, int T, int transpose_reverse,
                             cudaStream_t st);
struct PackSeg {  // one layer / pass of a batched weight packing
    int64_t row0;  // first block (row) of this segment: rows are co (forward layout) or ci (transposed)
    int Cout, Cin, T, tr;
    const void* w;
    void* wpack;
};
constexpr int HEX_PACK_MAX = 16;
struct PackSegs {
    int count;
    PackSeg seg[HEX_PACK_MAX];
};
hex_status_t tc_pack_weights_multi(const PackSegs& segs, cudaStream_t st);

struct TcWgradArgs {
    Geom g;
    int Cin, Cout;
    const void* x;   // bf16 NHWC input
    const void* dy;  // bf16 NHWC output gradient
    float* dw;       // fp32 [Cout][Cin][T]
    float* dbias;    // fp32 [Cout] or NULL
    int accumulate;
};
bool tc_wgrad_supported(const Geom& g, int Cin, int Cout);
size_t tc_wgrad_ws_bytes(const Geom& g, int Cin, int Cout);
hex_status_t tc_conv_wgrad(const TcWgradArgs& a, void* ws, size_t ws_bytes, cudaStream_t st);  // s = 1, or 2 (lattice)
bool tc_wgrad_lat_supported(const Geom& g, int Cin, int Cout);
size_t tc_wgrad_lat_ws_bytes(const Geom& g, int Cin, int Cout);
// tap-reuse variant (tc_wgrad_tr.cu); writes split-K partials, reduced by tc_conv_wgrad
bool tc_wgrad_tr_supported(const Geom& g, int Cin, int Cout);
struct TrDepth {  // 3-D weight gradient: depth taps folded into the units' channel chunks
    int kd, D, Do, sd;
};
size_t tc_wgrad_tr_ws_bytes(const Geom& g, int Cin, int Cout, int kd = 1);
hex_status_t tc_wgrad_tr(const TcWgradArgs& a, void* ws, size_t ws_bytes, int* chunks_out, float** db_part_out,
                         cudaStream_t st, const TrDepth* dz = nullptr);
// 3-D (conv3d.cu): x bf16 NDHWC [B*D][H][W][Cin], dy [B*Do][H][W][Cout] (a.g.B = B * Do), dw fp32
// [Cout][kd * Cin][T] in (kz, ci) channel order (permuted by the caller), dbias fresh
hex_status_t tc_conv3d_wgrad(const TcWgradArgs& a, const TrDepth& dz, void* ws, size_t ws_bytes, cudaStream_t st);

// single-input-channel bf16 NHWC stencil (config 5 layer 1)
bool smallc_supported(const Geom& g, int Cin, int Cout);
size_t smallc_wgrad_ws_bytes(const Geom& g, int Cout);
hex_status_t smallc_fwd(const void* x, const void* w, const float* bias, void* y, const Geom& g, int Cout, int relu,
                        cudaStream_t st);
hex_status_t smallc_wgrad(const void* x, const void* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                          int Cout, void* ws, cudaStream_t st);

// the same layer on the warp-level tensor cores (stride 1)
bool smallc_mma_supported(const Geom& g, int Cin, int Cout);
size_t smallc_mma_wgrad_ws_bytes(const Geom& g, int Cout);
hex_status_t smallc_mma_fwd(const void* x, const void* w, const float* bias, void* y, const Geom& g, int Cout,
                            int relu, cudaStream_t st);
hex_status_t smallc_mma_wgrad(const void* x, const void* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                              int Cout, void* ws, cudaStream_t st);

// single-input-channel fp32 NCHW stride-1 conv (plane_kernels.cu)
bool c1_conv_supported(const Geom& g, int Cin, int Cout, int dtype, int layout);
size_t c1_wgrad_ws_bytes(const Geom& g, int Cout);
hex_status_t c1_conv_fwd(const float* x, const float* w, const float* bias, float* y, const Geom& g, int Cout,
                         int relu, cudaStream_t st);
hex_status_t c1_conv_wgrad(const float* x, const float* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                           int Cout, void* ws, cudaStream_t st);

// fp32 NCHW weight gradient, column-walking sliding windows (f32_wgrad.cu)
bool f32_wgrad_supported(const Geom& g, int Cin, int Cout, int dtype, int layout);
size_t f32_wgrad_ws_bytes(const Geom& g, int Cin, int Cout);
hex_status_t f32_wgrad(const float* x, const float* dy, float* dw, float* dbias, int accumulate, const Geom& g,
                       int Cin, int Cout, void* ws, cudaStream_t st);

// register-blocked fp32 NCHW stride-1 conv (forward / transposed backward-data)
bool tiled_supported(const Geom& g, int dtype, int layout);
hex_status_t tiled_conv(const float* x, const float* w, const float* bias, const float* relu_y, float* y,
                        const Geom& g, int Cin, int Cout, int relu, int transpose, cudaStream_t st);

// fp32 NCHW convolution on the tcgen05 tensor cores in 3xTF32 (tf32_conv.cu).  Cx = channels of the
// gathered tensor (fwd: Cin, bwd-data: Cout), Nout = output channels (fwd: Cout, bwd-data: Cin).
bool tf32_conv_supported(const Geom& g, int Cx, int Nout, int dtype, int layout);
size_t tf32_conv_ws_bytes(const Geom& g, int Cx, int Nout);
hex_status_t tf32_conv(const Geom& g, int Cin, int Cout, int mode, const float* in, const float* w,
                       const float* bias, const float* relu_y, int relu, float* out, void* ws, size_t ws_bytes,
                       cudaStream_t st);
bool tf32_wgrad_supported(const Geom& g, int Cin, int Cout, int dtype, int layout);
size_t tf32_wgrad_ws_bytes(const Geom& g, int Cin, int Cout);
hex_status_t tf32_wgrad(const Geom& g, int Cin, int Cout, const float* x, const float* dy, float* dw, float* dbias,
                        int accumulate, void* ws, size_t ws_bytes, cudaStream_t st, int dbg = 0);

}  // namespace hexconv
