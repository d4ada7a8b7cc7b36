/*
 * hexconv.h -- C ABI of the B200-native hexagonal convolution / pooling
 * library (libhexconv.so), after HexagDLy (Steppa & Holch, arXiv 1903.01814).
 *
 * Data model (Sec. 2.1 "Input Format"): a hexagonally
 * sampled image is stored in a square tensor by "shifting every second column
 * upwards by half the distance between neighbouring pixels"; rows are counted
 * top->bottom and columns left->right.  `parity` selects which columns were
 * shifted: HEX_PARITY_ODD_LOW (0, the paper's default reading, A1)
 * means odd tensor columns are physically half a pitch lower.  Cells without a
 * hexagonal pixel hold arbitrary values and are treated as ordinary data.
 *
 * Kernel of size n (Sec. 2.2): all pixels within n layers
 * of neighbours of the centre, T(n) = 3n(n+1)+1 taps.  Weights are indexed
 * [Cout][Cin][T] with taps in canonical order: column-major left->right,
 * top->bottom (A2).
 *
 * Stride s: kernel centres form the lattice
 * anchored at pixel (0,0) with s equal steps along the three hex axes; output
 * column C is input column s*C, its rows are rho(C)+s*R with
 * rho(C) = floor((s*C+parity)/2) mod s, and every column is truncated to the
 * shortest one ("steps that would lead to an output with columns of unequal
 * length are neglected", A6).  Wo = floor((W-1)/s)+1,
 * Ho = min_C floor((H-1-rho(C))/s)+1.
 *
 * Conventions (all entry points):
 *  - Every tensor pointer is a caller-owned CUDA DEVICE pointer unless the
 *    argument says "host".  Tensors are dense and contiguous in the declared
 *    layout: HEX_NCHW = [B][C][H][W], HEX_NHWC = [B][H][W][C].
 *  - Argument validation is synchronous; on error nothing is launched and a
 *    status other than HEX_OK is returned.  Kernels run asynchronously on
 *    `stream` (a cudaStream_t; NULL = legacy default stream).  A launch
 *    failure returns HEX_ERR_CUDA; device faults surface at the caller's next
 *    synchronisation.
 *  - No device memory is allocated inside a call (except the NVLS setup
 *    calls hex_nvls_open / hex_nvls_map): scratch space is passed in `ws`
 *    (device) of `ws_bytes`, sized by hex_conv2d_workspace_size().
 *  - Thread-safe and re-entrant.  Results are deterministic (no floating
 *    point atomics): the same inputs give bitwise identical outputs.
 *  - HEX_BF16 tensors use round-to-nearest-even from fp32 accumulators.
 *    Weight/bias gradients are always fp32.  Bias is always fp32.
 *  - There is no CPU path: every entry point that touches tensor data runs
 *    CUDA kernels for sm_100a.
 */
#ifndef HEXCONV_H_
#define HEXCONV_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#define HEX_API __attribute__((visibility("default")))
#else
#define HEX_API
#endif

/* Same type as cudaStream_t (driver_types.h: typedef struct CUstream_st* cudaStream_t). */
typedef struct CUstream_st* hex_stream_t;

typedef enum {
    HEX_OK = 0,
    HEX_ERR_INVALID_ARG = 1,   /* null pointer, n < 0, stride < 1, bad enum, ... */
    HEX_ERR_SHAPE = 2,         /* non-positive dimension, channel mismatch        */
    HEX_ERR_EMPTY_LATTICE = 3, /* Ho or Wo would be 0 (A7)              */
    HEX_ERR_DTYPE = 4,
    HEX_ERR_LAYOUT = 5,
    HEX_ERR_ALIGNMENT = 6,     /* pointer not 16-byte aligned where required      */
    HEX_ERR_WORKSPACE = 7,     /* ws too small or NULL when required              */
    HEX_ERR_UNSUPPORTED = 8,   /* valid but unsupported (e.g. n > HEX_MAX_N)      */
    HEX_ERR_CUDA = 9           /* a CUDA runtime call failed                      */
} hex_status_t;

typedef enum { HEX_F32 = 0, HEX_BF16 = 1 } hex_dtype_t;
typedef enum { HEX_NCHW = 0, HEX_NHWC = 1 } hex_layout_t;
typedef enum { HEX_PARITY_ODD_LOW = 0, HEX_PARITY_EVEN_LOW = 1 } hex_parity_t;
typedef enum { HEX_POOL_MAX = 0, HEX_POOL_AVG = 1, HEX_POOL_AVG_PAD = 2 } hex_pool_mode_t;

#define HEX_MAX_N 7   /* largest supported kernel size (T = 169) */

typedef struct {
    int32_t batch, in_channels, out_channels, height, width;
    int32_t kernel_size; /* n >= 0; T(n) = 3n(n+1)+1 taps                          */
    int32_t stride;      /* s >= 1                                                 */
    int32_t parity;      /* hex_parity_t of the input grid                         */
    int32_t dtype;       /* hex_dtype_t of x, y, w, dy, dx                         */
    int32_t layout;      /* hex_layout_t of x, y, dy, dx                           */
} hex_conv2d_desc_t;

typedef struct {
    int32_t batch, channels, height, width;
    int32_t kernel_size; /* n >= 1 */
    int32_t stride;      /* s >= 1 */
    int32_t parity, dtype, layout;
    int32_t mode;        /* hex_pool_mode_t */
} hex_pool2d_desc_t;

/* ---------------------------------------------------------------- geometry */

/* T(n) = 3n(n+1)+1, or -1 if n < 0. */
HEX_API int32_t hex_num_taps(int32_t n);

/* Output grid of the stride lattice.  Ho, Wo,
 * parity_out are host pointers.  parity_out is the parity convention of the
 * output grid (pitch s): which output columns are physically lower.
 * Errors: HEX_ERR_INVALID_ARG (s < 1, bad parity, NULL), HEX_ERR_SHAPE
 * (H or W < 1), HEX_ERR_EMPTY_LATTICE (Ho == 0). */
HEX_API hex_status_t hex_output_shape(int32_t H, int32_t W, int32_t stride, int32_t parity,
                              int32_t* Ho, int32_t* Wo, int32_t* parity_out);

/* Test hook: the offset displacement of every tap for a centre whose column
 * has parity p = (col + parity) mod 2.  dc_dr (host, 2*T int32) receives
 * (dc, drow) pairs in canonical order.  (A2) */
HEX_API hex_status_t hex_tap_offsets(int32_t n, int32_t centre_col_parity, int32_t* dc_dr);

/* The T(n) taps as axial displacements (dq, dr) in canonical order, i.e. the
 * element order of a user-defined kernel ("structure detecting kernels",
 * PAPER.md:207-210; A2: lexicographic (dq, dr) over
 * |dq|+|dr|+|dq+dr| <= 2n = column-major left->right, top->bottom).
 * dq_dr: host, 2*T int32.  Errors: HEX_ERR_INVALID_ARG (n < 0, NULL),
 * HEX_ERR_UNSUPPORTED (n > HEX_MAX_N). */
HEX_API hex_status_t hex_tap_axial(int32_t n, int32_t* dq_dr);

/* Test hook: device int32 map [Ho][Wo][T], entry = r*W + c of tap t of
 * output (R,C), or -1 when that neighbour lies outside the grid.  Uses
 * desc->height/width/kernel_size/stride/parity only. */
HEX_API hex_status_t hex_conv2d_gather_map(const hex_conv2d_desc_t* desc, int32_t* map, hex_stream_t stream);

/* ---------------------------------------------------------------- convolution */

/* Workspace bytes needed by pass 0 = fwd, 1 = bwd_data, 2 = bwd_weight.
 * bytes is a host pointer.  0 means ws may be NULL. */
HEX_API hex_status_t hex_conv2d_workspace_size(const hex_conv2d_desc_t* desc, int32_t pass, size_t* bytes);

/* Forward (A3 cross-correlation,
 * A4 zero contribution of off-grid neighbours):
 *   y[b,co,R,C] = bias[co] + sum_ci sum_t w[co,ci,t] * x[b,ci, centre(R,C)+off_t]
 * then y = max(y, 0) if fuse_relu.
 * x: [B,Cin,H,W] in desc layout/dtype.  w: [Cout][Cin][T] in desc dtype (NULL on
 * the tensor-core path: weights prepacked in ws by hex_conv2d_pack_weights).
 * bias: fp32 [Cout] or NULL.  y: [B,Cout,Ho,Wo] in desc layout/dtype.
 *
 * Kernel selection (internal, channel-count driven; hex_conv2d_algo reports it):
 *  - tcgen05 tensor cores (bf16, NHWC, n <= 3, W >= 2):
 *      fwd       s = 1, 2 or 3, Cin % 64 == 0, Cout % 64 == 0 (s > 1:
 *                element-stride-s input boxes per output column class);
 *      bwd_data  s = 1: Cin % 64 == 0, Cout % 64 == 0 (the forward kernel on dy
 *                with reversed taps / transposed channels);  s = 2, 3 with
 *                Cin % 64 == 0, Cout % 64 == 0: phase classes (only the
 *                lattice taps, TMA boxes of dy); other s > 1: the s = 1
 *                kernel on dy scattered onto the stride-1 grid (Cout % 64 == 0);
 *      bwd_weight Cin % 64 == 0, Cout % 128 == 0 (s = 2, 3: on the lattice,
 *                x boxes with element stride s; other s > 1: via the
 *                scattered dy).
 *  - Cin == 1, bf16 NHWC, Cout % 64 == 0, n <= 2: warp-level mma.sync
 *    stencil kernels (s = 1) or FFMA stencils (s > 1).
 *  - fp32 NCHW, n <= 3, gathered channels >= 8 (fwd: Cin, bwd_data: Cout),
 *    output channels <= 64 (fwd: Cout, bwd_data: Cin), any stride: tcgen05
 *    in 3xTF32 (x = hi + lo, hi = tf32(x); D += hi.hi + hi.lo + lo.hi; ~fp32
 *    accuracy, A13), the hexagonal gather built in tensor memory.
 *  - everything else (small or odd channel counts, NHWC fp32, n <= 7, any
 *    stride): CUDA-core FFMA kernels, exact fp32 products. */
HEX_API hex_status_t hex_conv2d_fwd(const hex_conv2d_desc_t* desc, const void* x, const void* w,
                            const float* bias, int32_t fuse_relu, void* y,
                            void* ws, size_t ws_bytes, hex_stream_t stream);

/* Backward w.r.t. the input: the adjoint of the forward map,
 *   dx[b,ci,p] = sum_co sum_{(o,t): centre(o)+off_t = p} w[co,ci,t] * dy[b,co,o].
 * dy: [B,Cout,Ho,Wo]; dx: [B,Cin,H,W] (overwritten).
 * relu_y (optional, may be NULL): a tensor shaped like dx (the ReLU output
 * that was this layer's input); when given, dx is multiplied by (relu_y > 0)
 * -- the fused ReLU backward of the previous layer.  w as for the forward
 * (NULL: prepacked, pass 1, on the stride-1 tensor-core path). */
HEX_API hex_status_t hex_conv2d_bwd_data(const hex_conv2d_desc_t* desc, const void* dy, const void* w,
                                 const void* relu_y, void* dx,
                                 void* ws, size_t ws_bytes, hex_stream_t stream);

/* Backward w.r.t. weights and bias:
 *   dw[co,ci,t] = sum_{b,o} dy[b,co,o] * x[b,ci,centre(o)+off_t]   (off-grid -> 0)
 *   dbias[co]   = sum_{b,o} dy[b,co,o]
 * dw: fp32 [Cout][Cin][T]; dbias fp32 [Cout] or NULL.  accumulate != 0 adds
 * into dw/dbias instead of overwriting.  Deterministic two-stage reduction. */
HEX_API hex_status_t hex_conv2d_bwd_weight(const hex_conv2d_desc_t* desc, const void* x, const void* dy,
                                   float* dw, float* dbias, int32_t accumulate,
                                   void* ws, size_t ws_bytes, hex_stream_t stream);

/* Fused forward + ReLU + max pool (PAPER.md:144-151 then 202-205):
 *   y_pool = maxpool_{n=1, stride 2}( relu?( conv(x, w) + bias ) )
 * with the pool's lattice, window, tie-break and argmax exactly as hex_pool2d_fwd
 * (desc->parity, A8/A9) on the conv output grid, bit-identical to
 * hex_conv2d_fwd followed by hex_pool2d_fwd, but the conv output is never
 * written to memory.  desc: stride 1, bf16, NHWC.  y_pool: bf16 NHWC
 * [B][Ho][Wo][Cout], argmax_tap: uint8 [B][Ho][Wo][Cout] (not NULL), with
 * (Ho, Wo) = hex_output_shape(H, W, 2, parity).  ws as for pass 0.
 * HEX_ERR_UNSUPPORTED when no fused kernel covers the shape (the caller then
 * runs the two passes); hex_conv2d_fwd_maxpool_supported answers up front. */
HEX_API int32_t hex_conv2d_fwd_maxpool_supported(const hex_conv2d_desc_t* desc);
/* The same fused kernel for either pooling mode ("hex max/avg pool in one epilogue"):
 * mode HEX_POOL_MAX as hex_conv2d_fwd_maxpool, HEX_POOL_AVG the in-grid average (A8) of the bf16
 * conv outputs -- fp32 sum in canonical tap order times 1/count, RNE, bit-identical to hex_conv2d_fwd
 * followed by hex_pool2d_fwd(HEX_POOL_AVG) -- with argmax_tap ignored (may be NULL).
 * HEX_POOL_AVG_PAD has no fused kernel: HEX_ERR_UNSUPPORTED (as for unsupported shapes). */
HEX_API int32_t hex_conv2d_fwd_pool_supported(const hex_conv2d_desc_t* desc, int32_t mode);
HEX_API hex_status_t hex_conv2d_fwd_pool(const hex_conv2d_desc_t* desc, int32_t mode, const void* x,
                                         const void* w, const float* bias, int32_t fuse_relu, void* y_pool,
                                         uint8_t* argmax_tap, void* ws, size_t ws_bytes, hex_stream_t stream);
HEX_API hex_status_t hex_conv2d_fwd_maxpool(const hex_conv2d_desc_t* desc, const void* x, const void* w,
                                            const float* bias, int32_t fuse_relu, void* y_pool,
                                            uint8_t* argmax_tap, void* ws, size_t ws_bytes,
                                            hex_stream_t stream);

/* Weight packing hoisted out of the calls (the config-5 training step: the
 * weights change once per step, and each layer's fwd and bwd_data would pack
 * them again).  The bf16 tensor-core paths read the weights as per-tap K-major
 * tiles that hex_conv2d_fwd / hex_conv2d_fwd_maxpool / hex_conv2d_bwd_data
 * otherwise write into the front of their workspace on every call.  This call
 * does that packing for `count` (<= 16) layers in ONE kernel launch: for layer i,
 * descs[i] (host array), passes[i] = 0 (fwd and fwd_maxpool layout) or 1
 * (bwd_data, stride 1: transposed channels, reversed taps), w[i] the device
 * weights [Cout][Cin][T] (bf16, 16-byte aligned), ws[i] / ws_bytes[i] that
 * pass's workspace (hex_conv2d_workspace_size); w, ws, ws_bytes are host arrays
 * of device pointers / sizes.  A later fwd / fwd_maxpool / bwd_data call with
 * w == NULL and the same workspace uses the packed weights as they stand (the
 * caller repacks after changing w).  w == NULL is accepted on those tensor-core
 * paths only; elsewhere it is HEX_ERR_INVALID_ARG.
 * Errors: HEX_ERR_INVALID_ARG (count outside 0..16, NULL arrays / entries, pass
 * not 0/1), HEX_ERR_UNSUPPORTED (a descriptor whose pass does not take the
 * tensor-core path: check hex_conv2d_algo), HEX_ERR_WORKSPACE, HEX_ERR_ALIGNMENT,
 * descriptor errors as hex_conv2d_fwd. */
HEX_API hex_status_t hex_conv2d_pack_weights(int32_t count, const hex_conv2d_desc_t* descs,
                                             const int32_t* passes, const void* const* w, void* const* ws,
                                             const size_t* ws_bytes, hex_stream_t stream);

/* Which kernel family a call with this descriptor runs: *algo (host) = 0 for
 * the CUDA-core stencil path, 1 for the bf16 tcgen05 tensor-core path, 2 for
 * the fp32 3xTF32 tcgen05 path.  pass: 0 fwd, 1 bwd_data, 2 bwd_weight. */
HEX_API hex_status_t hex_conv2d_algo(const hex_conv2d_desc_t* desc, int32_t pass, int32_t* algo);

/* ---------------------------------------------------------------- 3-D convolution */

/* 3-D hexagonal convolution (Sec. 2 "Software Functionalities":
 * "the input data is expected to have a hexagonal layout in the x-y-plane while
 * data points along the z-axis are assumed to be equidistant").
 * Kernel: the hexagonal kernel of size n in each of kd (odd) depth slices with
 * independent weights w[Cout][Cin][kd][T(n)] (canonical taps, A2),
 * centred in depth; zero padding in depth; output depth slices are the centres
 * 0, sd, 2sd, ... (Do = (D-1)/sd + 1); the in-plane lattice is the 2-D one.
 *   y[b][co][zo][R][C] = bias[co] + sum_ci sum_kz sum_t w[co][ci][kz][t] *
 *                        x[b][ci][sd*zo + kz - (kd-1)/2][centre(R,C) + off_t]
 * layout HEX_NCHW means NCDHW, HEX_NHWC means NDHWC (channels innermost).
 * Implementation: bf16 NDHWC with in-plane s = 1 and Cin, Cout multiples of
 * 64 runs fwd (and bwd_data when sd = 1) on the tcgen05 tap-reuse kernel with
 * the depth taps inside its K loop (out-of-volume slices are TMA zero fill),
 * and bwd_weight (Cout a multiple of 128, well-filled tiles) on the tcgen05
 * tap-reuse weight gradient with the depth taps as its channel-chunk units.
 * Everything else unfolds the kd depth taps into input channels of one 2-D
 * convolution over B*Do images (x' = depth-unfolded input, Cin' = kd*Cin,
 * ordered (kz, ci)), so every 2-D path applies.  The workspace holds x' (or
 * dx'), the reordered weights and the 2-D call's own workspace.
 * Errors: as the 2-D calls, plus HEX_ERR_INVALID_ARG for even / non-positive
 * kernel_depth or depth_stride < 1, HEX_ERR_SHAPE for depth < 1. */
typedef struct {
    int32_t batch, in_channels, out_channels, depth, height, width;
    int32_t kernel_size;  /* in-plane n >= 0                       */
    int32_t kernel_depth; /* kd >= 1, odd                          */
    int32_t stride;       /* in-plane s >= 1                       */
    int32_t depth_stride; /* sd >= 1                               */
    int32_t parity, dtype, layout;
} hex_conv3d_desc_t;

/* *Do, *Ho, *Wo (host) of the output volume. */
HEX_API hex_status_t hex_conv3d_output_shape(const hex_conv3d_desc_t* desc, int32_t* Do, int32_t* Ho, int32_t* Wo);
/* Workspace bytes of pass 0 = fwd, 1 = bwd_data, 2 = bwd_weight. */
HEX_API hex_status_t hex_conv3d_workspace_size(const hex_conv3d_desc_t* desc, int32_t pass, size_t* bytes);
/* y [B,Cout,Do,Ho,Wo] (desc layout) = conv3d(x) (+ bias, optional fused ReLU). */
HEX_API hex_status_t hex_conv3d_fwd(const hex_conv3d_desc_t* desc, const void* x, const void* w, const float* bias,
                                    int32_t fuse_relu, void* y, void* ws, size_t ws_bytes, hex_stream_t stream);
/* dx [B,Cin,D,H,W] = adjoint of the forward applied to dy (overwritten; depth taps
 * summed in ascending kz, deterministic). */
HEX_API hex_status_t hex_conv3d_bwd_data(const hex_conv3d_desc_t* desc, const void* dy, const void* w, void* dx,
                                         void* ws, size_t ws_bytes, hex_stream_t stream);
/* dw (fp32 [Cout][Cin][kd][T]) and dbias (fp32 [Cout], NULL ok); accumulate != 0
 * adds to them. */
HEX_API hex_status_t hex_conv3d_bwd_weight(const hex_conv3d_desc_t* desc, const void* x, const void* dy, float* dw,
                                           float* dbias, int32_t accumulate, void* ws, size_t ws_bytes,
                                           hex_stream_t stream);

/* ---------------------------------------------------------------- pooling */

/* Pooling (the sub-convolutions are replaced by pooling
 * and "combined with aggregation functions", same padding/striding scheme).
 * HEX_POOL_MAX: y = x at the first strict maximum over the in-grid
 * neighbourhood in canonical tap order (A8, A9); argmax_tap
 * (uint8 [B,C,Ho,Wo] in desc layout, may be NULL) receives that tap index.
 * HEX_POOL_AVG: y = in-grid sum / in-grid count (A8).
 * HEX_POOL_AVG_PAD: y = in-grid sum / T(n) -- off-grid cells count as zeros (the
 *   include-pad alternative to A8; torch's count_include_pad analogue).
 *   Backward spreads dy / T(n) over the in-grid cells. */
HEX_API hex_status_t hex_pool2d_fwd(const hex_pool2d_desc_t* desc, const void* x, void* y,
                            uint8_t* argmax_tap, hex_stream_t stream);

/* Pool backward (gather form, no atomics).  MAX: dx[p] = sum of dy[o] over
 * outputs whose argmax tap points at p (argmax_tap required).  AVG:
 * dx[p] = sum_{o: p in N(o)} dy[o] / count(o).  dx is overwritten. */
HEX_API hex_status_t hex_pool2d_bwd(const hex_pool2d_desc_t* desc, const void* dy,
                            const uint8_t* argmax_tap, void* dx, hex_stream_t stream);

/* ---------------------------------------------------------------- training helpers
 * Used by the data-parallel training step (BASELINE config 5).  Not part of
 * the paper's method; plain elementwise / reduction kernels. */

/* Pool backward with the ReLU backward of the pooled layer fused:
 *   dx = hex_pool2d_bwd(dy, argmax) * (relu_y > 0)
 * relu_y: the pool's forward input (the post-ReLU activation), shaped like dx.
 * Same arguments, layouts and errors as hex_pool2d_bwd; relu_y must not be
 * NULL.  NCHW n = 1, stride 2 runs one kernel; other shapes run the pool
 * backward and then the elementwise mask (hex_relu_bwd). */
HEX_API hex_status_t hex_pool2d_bwd_relu(const hex_pool2d_desc_t* desc, const void* dy, const uint8_t* argmax_tap,
                                         const void* relu_y, void* dx, hex_stream_t stream);

/* Head of the C5 network, forward + backward in one launch:
 * feat bf16 NHWC [B][HW][C] (ReLU output) -> global average pool -> logits
 * [B][K] = gap @ wl^T + bl (wl fp32 [K][C], bl fp32 [K]) -> mean softmax
 * cross-entropy against labels (int32 [B]).  Writes loss (fp32 scalar),
 * dfeat (bf16 NHWC, = d loss / d feat masked by feat > 0), dwl, dbl (fp32).
 * ws must hold hex_head_workspace_size(B, K, C) bytes. */
HEX_API size_t hex_head_workspace_size(int32_t B, int32_t K, int32_t C);
HEX_API hex_status_t hex_head_fwd_bwd(int32_t B, int32_t HW, int32_t C, int32_t K,
                              const void* feat, const float* wl, const float* bl,
                              const int32_t* labels, float* loss, void* dfeat,
                              float* dwl, float* dbl, void* ws, size_t ws_bytes,
                              hex_stream_t stream);

/* SGD with momentum over a flat fp32 parameter vector:
 *   g = grad * grad_scale;  mom = mu * mom + g;  param -= lr * mom;
 * and, if param_bf16 != NULL, param_bf16 = bf16(param). */
HEX_API hex_status_t hex_sgd_momentum(int64_t count, float* param, const float* grad, float* mom,
                              float lr, float mu, float grad_scale, void* param_bf16,
                              hex_stream_t stream);

/* Elementwise fp32 -> bf16 (RNE) conversion of count values. */
/* ReLU backward for callers without a fused mask: dx[i] = y[i] > 0 ? dy[i] : 0
 * over `count` elements of `dtype` (y = the post-ReLU forward output; dy, y,
 * dx device, same dtype; dx may alias dy).  Errors: HEX_ERR_SHAPE (count < 0),
 * HEX_ERR_DTYPE, HEX_ERR_INVALID_ARG (NULL with count > 0). */
HEX_API hex_status_t hex_relu_bwd(int64_t count, int32_t dtype, const void* dy, const void* y, void* dx,
                                  hex_stream_t stream);

HEX_API hex_status_t hex_cast_f32_bf16(int64_t count, const float* src, void* dst, hex_stream_t stream);

/* ---------------------------------------------------------------- NVLS gradient sum
 * The data-parallel exchange of the method's training step -- the sum over
 * ranks of the flat fp32 gradient vector (every rank trains on its own share
 * of the batch) -- performed inside the NVSwitch: the
 * gradient vector lives in device memory bound to a CUDA multicast object
 * spanning one GPU per rank.  Ranks write their local gradients through the
 * unicast pointer; hex_nvls_allreduce_f32 then replaces a bucket of it, on
 * every rank, by the sum over ranks (multimem.ld_reduce of a 1/world slice
 * per rank + multimem.st to all replicas, ordered by multicast counters; see
 * csrc/nvls.cu).  Every rank ends with bitwise identical sums.
 *
 * Setup (collective: every rank calls each step, in order, with a barrier
 * between the steps; the only calls that allocate device memory):
 *   1. hex_nvls_open: rank 0 creates the multicast object and, for world > 1,
 *      exports it as a POSIX file descriptor (*fd_out, host; the caller passes
 *      it to the other ranks, e.g. SCM_RIGHTS, and closes it); ranks > 0
 *      import it from fd_in (host; the caller may close it afterwards).  Every
 *      rank attaches `device`.  data_bytes: the region the caller needs.
 *   2. barrier (all devices attached)
 *   3. hex_nvls_map: backs the object with `device` memory, maps it, zeroes
 *      it; *uc = local pointer, *mc = multicast pointer (device), *map_bytes =
 *      usable bytes (data_bytes rounded up to 256).
 *   4. barrier (all counters zero)
 * hex_nvls_allreduce_f32(h, offset, count, slot, stream): sums elements
 * [offset, offset+count) of the fp32 region across the ranks, asynchronously
 * on `stream` after the work already enqueued there; offset % 4 == 0
 * (HEX_ERR_ALIGNMENT), the bucket must lie in the region (HEX_ERR_SHAPE).
 * `slot` (0 .. HEX_NVLS_SLOTS-1) names the call site: every rank must issue
 * the same sequence of (slot, offset, count) calls; concurrent calls must use
 * different slots.  Graph-capturable (its epoch counters live in device
 * memory).  A rank that does not arrive within 10 s makes the others trap (a
 * launch failure at their next synchronisation) instead of hanging.
 * hex_nvls_open_local(device, data_bytes, out): a single-rank region in plain
 * device memory (no multicast object; then hex_nvls_map as above): the same
 * kernel protocol with ordinary loads / stores / atomics in place of the
 * multimem ones -- the gradient "sum" of one rank, for single-GPU use and for
 * exercising the protocol on GPUs without multicast support.
 * hex_nvls_supported: *supported = 1 if `device` exists, reports multicast
 * support and a one-device multicast object can actually be created (a GPU
 * leased without its NVSwitch fabric reports the attribute but cannot).  hex_nvls_close: synchronises the device, unmaps, frees.
 * hex_nvls_plan (host only, no GPU needed): the element range [*begin, *end)
 * that (rank, cta) reduces for a bucket of `count` elements, and the grid
 * size *grid (cta = -1: grid only).
 * Errors: HEX_ERR_UNSUPPORTED (no multicast support), HEX_ERR_CUDA (a driver
 * call failed; the message is printed to stderr), HEX_ERR_INVALID_ARG. */
#define HEX_NVLS_SLOTS 64
#define HEX_NVLS_MAX_CTAS 148
typedef struct hex_nvls hex_nvls_t;
HEX_API hex_status_t hex_nvls_supported(int32_t device, int32_t* supported);
HEX_API hex_status_t hex_nvls_open(int32_t world, int32_t rank, int32_t device, size_t data_bytes,
                                   int32_t fd_in, int32_t* fd_out, hex_nvls_t** out);
HEX_API hex_status_t hex_nvls_open_local(int32_t device, size_t data_bytes, hex_nvls_t** out);
HEX_API hex_status_t hex_nvls_map(hex_nvls_t* h, void** uc, void** mc, size_t* map_bytes);
HEX_API hex_status_t hex_nvls_allreduce_f32(hex_nvls_t* h, int64_t offset, int64_t count, int32_t slot,
                                            hex_stream_t stream);
HEX_API hex_status_t hex_nvls_close(hex_nvls_t* h);
HEX_API hex_status_t hex_nvls_plan(int64_t count, int32_t world, int32_t rank, int32_t cta, int32_t* grid,
                                   int64_t* begin, int64_t* end);

/* ---------------------------------------------------------------- misc */
HEX_API const char* hex_status_string(hex_status_t status);
/* Library version, e.g. 0x000100 for 0.1.0. */
HEX_API int32_t hex_version(void);

/* Test hook for A/B tests of kernel selection: the HEXCONV_* switches
 * (DESIGN.md appendix) are read from the environment once, when the library
 * is loaded; this overrides one of them (value NULL = unset).  Every switch
 * selects between kernels that compute the same result.  Not synchronised
 * with concurrent calls: set switches between calls only.
 * Errors: HEX_ERR_INVALID_ARG (NULL or unknown name). */
HEX_API hex_status_t hex_debug_set_switch(const char* name, const char* value);
/* Number of kernels this library has launched since load (host counter,
 * used by bench.py to report gpu_launches). */
HEX_API int64_t hex_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HEXCONV_H_ */
