// abi.cu -- the C ABI of libhexconv (include/hexconv.h): argument validation,
// path selection (tcgen05 implicit GEMM vs CUDA-core stencil) and launch.
// Validation is synchronous and never launches on error.  There is no CPU
// fallback: every data-touching call runs CUDA kernels.
#include <mutex>
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include <algorithm>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {
std::atomic<int64_t> g_launches{0};
size_t head_ws_bytes(int B, int K, int C);
hex_status_t head_fwd_bwd(int B, int HW, int C, int K, const void* feat, const float* wl, const float* bl,
                          const int32_t* labels, float* loss, void* dfeat, float* dwl, float* dbl, void* ws,
                          cudaStream_t st);
hex_status_t sgd_momentum(int64_t n, float* p, const float* g, float* m, float lr, float mu, float gs, void* pb,
                          cudaStream_t st);
hex_status_t cast_f32_bf16(int64_t n, const float* s, void* d, cudaStream_t st);
hex_status_t relu_bwd(int64_t n, int dtype, const void* dy, const void* y, void* dx, cudaStream_t st);
}  // namespace hexconv


// ------------------------------------------------------------------ kernel-selection switches
// Read from the environment once, when the shared library is loaded (a constructor), so the dispatch path
// never calls getenv and a CUDA graph captures the same kernel selection as every later call.
namespace {
struct SwitchEntry {
    const char* name;
    bool set;
    char text[32];
};
SwitchEntry g_switches[] = {
    {"HEXCONV_CONV3D_UNFOLD", false, ""},
    {"HEXCONV_DEBUG", false, ""},
    {"HEXCONV_DISABLE_TC", false, ""},
    {"HEXCONV_FORCE_2SM", false, ""},
    {"HEXCONV_FP_DEBUG", false, ""},
    {"HEXCONV_FP_NREG", false, ""},
    {"HEXCONV_FT_DEBUG", false, ""},
    {"HEXCONV_FUSED_POOL_REGIONS", false, ""},
    {"HEXCONV_FWD_TR_NORES", false, ""},
    {"HEXCONV_NO_2SM", false, ""},
    {"HEXCONV_NO_CONV3D_TC", false, ""},
    {"HEXCONV_NO_F32_WGRAD", false, ""},
    {"HEXCONV_NO_FUSED_POOL", false, ""},
    {"HEXCONV_NO_FWD_TR", false, ""},
    {"HEXCONV_NO_FWD_TR_PAIR", false, ""},
    {"HEXCONV_NO_FWD_VPAIR", false, ""},
    {"HEXCONV_NO_LAT_DGRAD", false, ""},
    {"HEXCONV_NO_PLANE", false, ""},
    {"HEXCONV_NO_POOL_TMA", false, ""},
    {"HEXCONV_NO_TC_STRIDED_FWD", false, ""},
    {"HEXCONV_NO_TC_STRIDED_BWD", false, ""},
    {"HEXCONV_NO_TC_WGRAD_LAT", false, ""},
    {"HEXCONV_NO_TF32", false, ""},
    {"HEXCONV_NO_TILED", false, ""},
    {"HEXCONV_NO_WG_TR", false, ""},
    {"HEXCONV_POOL_BWD_V2", false, ""},
    {"HEXCONV_POOL_GENERIC", false, ""},
    {"HEXCONV_POOL_PIXEL_BWD", false, ""},
    {"HEXCONV_POOL_TMA_MIN_W", false, ""},
    {"HEXCONV_POOL_V", false, ""},
    {"HEXCONV_POOL_WIDE_BWD", false, ""},
    {"HEXCONV_SMALLC_FFMA", false, ""},
    {"HEXCONV_WG_DEBUG", false, ""},
    {"HEXCONV_WG_TR_MINFILL", false, ""},
    {"HEXCONV_WG_TR_RB", false, ""}
};
constexpr int kNumSwitches = (int)(sizeof(g_switches) / sizeof(g_switches[0]));

void load_switch(SwitchEntry& e, const char* v) {
    e.set = v != nullptr;
    snprintf(e.text, sizeof(e.text), "%s", v ? v : "");
}

__attribute__((constructor)) void read_switches_at_load() {
    for (int i = 0; i < kNumSwitches; ++i) load_switch(g_switches[i], getenv(g_switches[i].name));
}

const SwitchEntry* find_switch(const char* name) {
    for (int i = 0; i < kNumSwitches; ++i)
        if (strcmp(g_switches[i].name, name) == 0) return &g_switches[i];
    return nullptr;
}
}  // namespace

namespace hexconv {
bool sw_on(const char* name) {
    const SwitchEntry* e = find_switch(name);
    return e && e->set;
}
int sw_int(const char* name, int dflt) {
    const SwitchEntry* e = find_switch(name);
    return e && e->set ? atoi(e->text) : dflt;
}
double sw_double(const char* name, double dflt) {
    const SwitchEntry* e = find_switch(name);
    return e && e->set ? atof(e->text) : dflt;
}
}  // namespace hexconv

using namespace hexconv;

namespace {

inline bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

hex_status_t check_common(int B, int C, int H, int W, int n, int s, int parity, int dtype, int layout) {
    if (n < 0 || s < 1) return HEX_ERR_INVALID_ARG;
    if (parity != 0 && parity != 1) return HEX_ERR_INVALID_ARG;
    if (B < 1 || C < 1 || H < 1 || W < 1) return HEX_ERR_SHAPE;
    if (dtype != HEX_F32 && dtype != HEX_BF16) return HEX_ERR_DTYPE;
    if (layout != HEX_NCHW && layout != HEX_NHWC) return HEX_ERR_LAYOUT;
    if (n > HEX_MAX_N) return HEX_ERR_UNSUPPORTED;
    return HEX_OK;
}

hex_status_t conv_geom(const hex_conv2d_desc_t* d, Geom* g) {
    if (!d) return HEX_ERR_INVALID_ARG;
    hex_status_t st = check_common(d->batch, d->in_channels, d->height, d->width, d->kernel_size, d->stride,
                                   d->parity, d->dtype, d->layout);
    if (st != HEX_OK) return st;
    if (d->out_channels < 1) return HEX_ERR_SHAPE;
    g->B = d->batch; g->H = d->height; g->W = d->width;
    g->n = d->kernel_size; g->s = d->stride; g->parity = d->parity; g->T = hex_taps(d->kernel_size);
    if (!out_shape(g->H, g->W, g->s, g->parity, &g->Ho, &g->Wo, nullptr)) return HEX_ERR_EMPTY_LATTICE;
    return HEX_OK;
}

// The tensor-core path: bf16, NHWC, stride 1 and channel counts that tile.
bool use_tc_fwd(const hex_conv2d_desc_t* d, const Geom& g) {
    return d->dtype == HEX_BF16 && d->layout == HEX_NHWC && tc_conv_fwd_supported(g, d->in_channels, d->out_channels);
}
bool use_tc_bwd_data(const hex_conv2d_desc_t* d, const Geom& g) {
    return d->dtype == HEX_BF16 && d->layout == HEX_NHWC && tc_conv_supported(g, d->out_channels, d->in_channels);
}
bool use_smallc(const hex_conv2d_desc_t* d, const Geom& g) {
    return d->dtype == HEX_BF16 && d->layout == HEX_NHWC && smallc_supported(g, d->in_channels, d->out_channels);
}
bool use_f32wg(const hex_conv2d_desc_t* d, const Geom& g) {
    return f32_wgrad_supported(g, d->in_channels, d->out_channels, d->dtype, d->layout);
}
bool use_c1(const hex_conv2d_desc_t* d, const Geom& g) {
    return c1_conv_supported(g, d->in_channels, d->out_channels, d->dtype, d->layout);
}
bool use_tf32_fwd(const hex_conv2d_desc_t* d, const Geom& g) {
    return tf32_conv_supported(g, d->in_channels, d->out_channels, d->dtype, d->layout);
}
bool use_tf32_bwd_data(const hex_conv2d_desc_t* d, const Geom& g) {
    return tf32_conv_supported(g, d->out_channels, d->in_channels, d->dtype, d->layout);
}
bool use_tf32_wgrad(const hex_conv2d_desc_t* d, const Geom& g) {
    return tf32_wgrad_supported(g, d->in_channels, d->out_channels, d->dtype, d->layout);
}
bool use_tc_wgrad(const hex_conv2d_desc_t* d, const Geom& g) {
    return d->dtype == HEX_BF16 && d->layout == HEX_NHWC && tc_wgrad_supported(g, d->in_channels, d->out_channels);
}

// strided layers: the backward passes run the stride-1 tensor-core kernels on dy scattered onto the
// full grid (strided.cu)
Geom stride1(const Geom& g) {
    Geom g1 = g;
    g1.s = 1;
    g1.Ho = g.H;
    g1.Wo = g.W;
    return g1;
}
bool strided_tc_ok(const hex_conv2d_desc_t* d, const Geom& g) {
    return g.s > 1 && d->dtype == HEX_BF16 && d->layout == HEX_NHWC && d->out_channels % 8 == 0 &&
           !sw_on("HEXCONV_NO_TC_STRIDED_BWD");
}
bool use_lat_dgrad(const hex_conv2d_desc_t* d, const Geom& g) {  // strided bf16 bwd-data by phase classes
    return g.s > 1 && d->dtype == HEX_BF16 && d->layout == HEX_NHWC && !sw_on("HEXCONV_NO_TC_STRIDED_BWD") &&
           lat_dgrad_supported(g, d->in_channels, d->out_channels);
}
bool use_tc_bwd_data_up(const hex_conv2d_desc_t* d, const Geom& g) {
    return strided_tc_ok(d, g) && tc_conv_supported(stride1(g), d->out_channels, d->in_channels);
}
bool use_tc_wgrad_lat(const hex_conv2d_desc_t* d, const Geom& g) {  // strided (s = 2, 3) weight gradient on the lattice
    return strided_tc_ok(d, g) && tc_wgrad_lat_supported(g, d->in_channels, d->out_channels);
}
bool use_tc_wgrad_up(const hex_conv2d_desc_t* d, const Geom& g) {
    return strided_tc_ok(d, g) && tc_wgrad_supported(stride1(g), d->in_channels, d->out_channels);
}
size_t up_bytes(const hex_conv2d_desc_t* d, const Geom& g) {  // + slack for aligning it and what follows
    return (size_t)g.B * g.H * g.W * d->out_channels * 2 + 2048;
}

size_t packed_weight_bytes(const hex_conv2d_desc_t* d, const Geom& g) {
    return (size_t)g.T * d->out_channels * d->in_channels * 2 + 1024;
}

DirectConvArgs make_direct(const hex_conv2d_desc_t* d, const Geom& g) {
    DirectConvArgs a{};
    a.g = g;
    a.Cin = d->in_channels;
    a.Cout = d->out_channels;
    a.dtype = d->dtype;
    a.sx = make_strides(d->layout, d->in_channels, g.H, g.W);
    a.sy = make_strides(d->layout, d->out_channels, g.Ho, g.Wo);
    return a;
}

void* align_up(void* p, size_t a) { return (void*)(((uintptr_t)p + a - 1) & ~(uintptr_t)(a - 1)); }

}  // namespace

extern "C" {

int32_t hex_num_taps(int32_t n) { return n < 0 ? -1 : hex_taps(n); }

int32_t hex_version(void) { return 0x000200; }

hex_status_t hex_debug_set_switch(const char* name, const char* value) {
    if (!name) return HEX_ERR_INVALID_ARG;
    for (int i = 0; i < kNumSwitches; ++i)
        if (strcmp(g_switches[i].name, name) == 0) {
            load_switch(g_switches[i], value);
            return HEX_OK;
        }
    return HEX_ERR_INVALID_ARG;
}

int64_t hex_launch_count(void) { return g_launches.load(); }

const char* hex_status_string(hex_status_t s) {
    switch (s) {
        case HEX_OK: return "ok";
        case HEX_ERR_INVALID_ARG: return "invalid argument";
        case HEX_ERR_SHAPE: return "shape mismatch";
        case HEX_ERR_EMPTY_LATTICE: return "empty lattice";
        case HEX_ERR_DTYPE: return "unsupported dtype";
        case HEX_ERR_LAYOUT: return "unsupported layout";
        case HEX_ERR_ALIGNMENT: return "misaligned pointer";
        case HEX_ERR_WORKSPACE: return "workspace too small";
        case HEX_ERR_UNSUPPORTED: return "unsupported configuration";
        case HEX_ERR_CUDA: return "CUDA error";
    }
    return "unknown status";
}

hex_status_t hex_output_shape(int32_t H, int32_t W, int32_t stride, int32_t parity, int32_t* Ho, int32_t* Wo,
                              int32_t* parity_out) {
    if (!Ho || !Wo || !parity_out) return HEX_ERR_INVALID_ARG;
    if (stride < 1 || (parity != 0 && parity != 1)) return HEX_ERR_INVALID_ARG;
    if (H < 1 || W < 1) return HEX_ERR_SHAPE;
    int ho, wo, po;
    bool ok = out_shape(H, W, stride, parity, &ho, &wo, &po);
    *Ho = ho < 0 ? 0 : ho;
    *Wo = wo;
    *parity_out = po;
    return ok ? HEX_OK : HEX_ERR_EMPTY_LATTICE;
}

hex_status_t hex_tap_offsets(int32_t n, int32_t p, int32_t* dc_dr) {
    if (n < 0 || (p != 0 && p != 1) || !dc_dr) return HEX_ERR_INVALID_ARG;
    if (n > HEX_MAX_N) return HEX_ERR_UNSUPPORTED;
    const int T = hex_taps(n);
    for (int t = 0; t < T; ++t) tap_offset(n, p, t, &dc_dr[2 * t], &dc_dr[2 * t + 1]);
    return HEX_OK;
}

hex_status_t hex_tap_axial(int32_t n, int32_t* dq_dr) {
    if (n < 0 || !dq_dr) return HEX_ERR_INVALID_ARG;
    if (n > HEX_MAX_N) return HEX_ERR_UNSUPPORTED;
    int t = 0;  // lexicographic (dq, dr) over the hexagonal disc |dq| + |dr| + |dq + dr| <= 2n
    for (int dq = -n; dq <= n; ++dq)
        for (int dr = -n; dr <= n; ++dr)
            if (abs(dq) + abs(dr) + abs(dq + dr) <= 2 * n) {
                dq_dr[2 * t] = dq;
                dq_dr[2 * t + 1] = dr;
                ++t;
            }
    return HEX_OK;
}

hex_status_t hex_conv2d_gather_map(const hex_conv2d_desc_t* d, int32_t* map, hex_stream_t stream) {
    if (!d || !map) return HEX_ERR_INVALID_ARG;
    if (d->kernel_size < 0 || d->stride < 1 || (d->parity != 0 && d->parity != 1)) return HEX_ERR_INVALID_ARG;
    if (d->height < 1 || d->width < 1) return HEX_ERR_SHAPE;
    if (d->kernel_size > HEX_MAX_N) return HEX_ERR_UNSUPPORTED;
    Geom g{};
    g.B = 1; g.H = d->height; g.W = d->width; g.n = d->kernel_size; g.s = d->stride; g.parity = d->parity;
    g.T = hex_taps(g.n);
    if (!out_shape(g.H, g.W, g.s, g.parity, &g.Ho, &g.Wo, nullptr)) return HEX_ERR_EMPTY_LATTICE;
    return launch_gather_map(map, g, (cudaStream_t)stream);
}

hex_status_t hex_conv2d_workspace_size(const hex_conv2d_desc_t* d, int32_t pass, size_t* bytes) {
    if (!bytes) return HEX_ERR_INVALID_ARG;
    Geom g;
    hex_status_t st = conv_geom(d, &g);
    if (st != HEX_OK) return st;
    switch (pass) {
        case 0:
            *bytes = use_tc_fwd(d, g)     ? packed_weight_bytes(d, g)
                     : use_tf32_fwd(d, g) ? tf32_conv_ws_bytes(g, d->in_channels, d->out_channels)
                                          : 0;
            return HEX_OK;
        case 1:
            *bytes = use_tc_bwd_data(d, g)      ? packed_weight_bytes(d, g)
                     : use_tc_bwd_data_up(d, g)
                         ? std::max(up_bytes(d, g) + packed_weight_bytes(d, g),
                                    use_lat_dgrad(d, g) ? lat_dgrad_ws_bytes(g, d->in_channels, d->out_channels) : 0)
                     : use_lat_dgrad(d, g)      ? lat_dgrad_ws_bytes(g, d->in_channels, d->out_channels)
                     : use_tf32_bwd_data(d, g)  ? tf32_conv_ws_bytes(g, d->out_channels, d->in_channels)
                                                : 0;
            return HEX_OK;
        case 2:
            *bytes = use_tc_wgrad(d, g)      ? tc_wgrad_ws_bytes(g, d->in_channels, d->out_channels)
                     : use_tc_wgrad_lat(d, g) ? tc_wgrad_lat_ws_bytes(g, d->in_channels, d->out_channels)
                     : use_tc_wgrad_up(d, g) ? up_bytes(d, g) + tc_wgrad_ws_bytes(stride1(g), d->in_channels,
                                                                                   d->out_channels)
                     : use_tf32_wgrad(d, g)  ? tf32_wgrad_ws_bytes(g, d->in_channels, d->out_channels)
                     : use_smallc(d, g) ? smallc_wgrad_ws_bytes(g, d->out_channels)
                     : use_c1(d, g)     ? c1_wgrad_ws_bytes(g, d->out_channels)
                     : use_f32wg(d, g)  ? f32_wgrad_ws_bytes(g, d->in_channels, d->out_channels)
                                        : direct_wgrad_ws_bytes(g, d->in_channels, d->out_channels);
            return HEX_OK;
        default: return HEX_ERR_INVALID_ARG;
    }
}

hex_status_t hex_conv2d_algo(const hex_conv2d_desc_t* d, int32_t pass, int32_t* algo) {
    if (!algo) return HEX_ERR_INVALID_ARG;
    Geom g;
    hex_status_t st = conv_geom(d, &g);
    if (st != HEX_OK) return st;
    switch (pass) {
        case 0: *algo = use_tc_fwd(d, g) ? 1 : use_tf32_fwd(d, g) ? 2 : 0; return HEX_OK;
        case 1:
            *algo = use_tc_bwd_data(d, g) || use_lat_dgrad(d, g) || use_tc_bwd_data_up(d, g) ? 1
                    : use_tf32_bwd_data(d, g)                                              ? 2
                                                                                           : 0;
            return HEX_OK;
        case 2:
            *algo = use_tc_wgrad(d, g) || use_tc_wgrad_lat(d, g) || use_tc_wgrad_up(d, g) ? 1
                    : use_tf32_wgrad(d, g)                                             ? 2
                                                                                       : 0;
            return HEX_OK;
        default: return HEX_ERR_INVALID_ARG;
    }
}

hex_status_t hex_conv2d_fwd(const hex_conv2d_desc_t* d, const void* x, const void* w, const float* bias,
                            int32_t fuse_relu, void* y, void* ws, size_t ws_bytes, hex_stream_t stream) {
    Geom g;
    hex_status_t st = conv_geom(d, &g);
    if (st != HEX_OK) return st;
    if (!x || !y) return HEX_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (use_tc_fwd(d, g)) {
        if (!aligned16(x) || !aligned16(y) || (w && !aligned16(w)) || (bias && !aligned16(bias)))
            return HEX_ERR_ALIGNMENT;
        const size_t need = packed_weight_bytes(d, g);
        if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
        void* wp = align_up(ws, 1024);
        if (w && (st = tc_pack_weights(w, wp, d->out_channels, d->in_channels, g.T, 0, s)) != HEX_OK) return st;
        TcConvArgs a{};
        a.g = g; a.Cin = d->in_channels; a.Cout = d->out_channels;
        a.x = x; a.wpack = wp; a.bias = bias; a.y = y; a.relu_y = nullptr; a.relu = fuse_relu;
        return tc_conv_fwd(a, s);
    }
    if (!w) return HEX_ERR_INVALID_ARG;  // w == NULL (prepacked) only on the tensor-core path
    if (use_smallc(d, g)) {
        if (((uintptr_t)y & 3) != 0) return HEX_ERR_ALIGNMENT;
        return smallc_fwd(x, w, bias, y, g, d->out_channels, fuse_relu, s);
    }
    if (use_tf32_fwd(d, g))
        return tf32_conv(g, d->in_channels, d->out_channels, 0, (const float*)x, (const float*)w, bias, nullptr,
                         fuse_relu, (float*)y, ws, ws_bytes, s);
    if (use_c1(d, g)) return c1_conv_fwd((const float*)x, (const float*)w, bias, (float*)y, g, d->out_channels,
                                         fuse_relu, s);
    if (tiled_supported(g, d->dtype, d->layout))
        return tiled_conv((const float*)x, (const float*)w, bias, nullptr, (float*)y, g, d->in_channels,
                          d->out_channels, fuse_relu, 0, s);
    DirectConvArgs a = make_direct(d, g);
    a.x = x; a.w = w; a.bias = bias; a.y = y; a.relu = fuse_relu;
    return direct_conv_fwd(a, s);
}

int32_t hex_conv2d_fwd_pool_supported(const hex_conv2d_desc_t* d, int32_t mode) {
    Geom g;
    if (conv_geom(d, &g) != HEX_OK) return 0;
    return use_tc_fwd(d, g) && tc_conv_pool_supported(g, d->in_channels, d->out_channels, mode) ? 1 : 0;
}

hex_status_t hex_conv2d_fwd_pool(const hex_conv2d_desc_t* d, int32_t mode, const void* x, const void* w,
                                 const float* bias, int32_t fuse_relu, void* y_pool, uint8_t* argmax, void* ws,
                                 size_t ws_bytes, hex_stream_t stream) {
    Geom g;
    hex_status_t st = conv_geom(d, &g);
    if (st != HEX_OK) return st;
    if (mode != HEX_POOL_MAX && mode != HEX_POOL_AVG && mode != HEX_POOL_AVG_PAD) return HEX_ERR_INVALID_ARG;
    if (!x || !y_pool || (mode == HEX_POOL_MAX && !argmax)) return HEX_ERR_INVALID_ARG;
    if (!use_tc_fwd(d, g) || !tc_conv_pool_supported(g, d->in_channels, d->out_channels, mode))
        return HEX_ERR_UNSUPPORTED;
    if (!aligned16(x) || !aligned16(y_pool) || (w && !aligned16(w)) ||
        (mode == HEX_POOL_MAX && ((uintptr_t)argmax & 7)) || (bias && !aligned16(bias)))
        return HEX_ERR_ALIGNMENT;
    const size_t need = packed_weight_bytes(d, g);
    if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
    cudaStream_t s = (cudaStream_t)stream;
    void* wp = align_up(ws, 1024);
    if (w && (st = tc_pack_weights(w, wp, d->out_channels, d->in_channels, g.T, 0, s)) != HEX_OK) return st;
    TcConvArgs a{};
    a.g = g; a.Cin = d->in_channels; a.Cout = d->out_channels;
    a.x = x; a.wpack = wp; a.bias = bias; a.y = nullptr; a.relu_y = nullptr; a.relu = fuse_relu;
    return tc_conv_pool(a, mode, y_pool, mode == HEX_POOL_MAX ? argmax : nullptr, s);
}

int32_t hex_conv2d_fwd_maxpool_supported(const hex_conv2d_desc_t* d) {
    return hex_conv2d_fwd_pool_supported(d, HEX_POOL_MAX);
}

hex_status_t hex_conv2d_fwd_maxpool(const hex_conv2d_desc_t* d, const void* x, const void* w, const float* bias,
                                    int32_t fuse_relu, void* y_pool, uint8_t* argmax, void* ws, size_t ws_bytes,
                                    hex_stream_t stream) {
    return hex_conv2d_fwd_pool(d, HEX_POOL_MAX, x, w, bias, fuse_relu, y_pool, argmax, ws, ws_bytes, stream);
}

hex_status_t hex_conv2d_bwd_data(const hex_conv2d_desc_t* d, const void* dy, const void* w, const void* relu_y,
                                 void* dx, void* ws, size_t ws_bytes, hex_stream_t stream) {
    Geom g;
    hex_status_t st = conv_geom(d, &g);
    if (st != HEX_OK) return st;
    if (!dy || !dx) return HEX_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (use_tc_bwd_data(d, g)) {
        if (!aligned16(dy) || !aligned16(dx) || (w && !aligned16(w)) || (relu_y && !aligned16(relu_y)))
            return HEX_ERR_ALIGNMENT;
        const size_t need = packed_weight_bytes(d, g);
        if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
        void* wp = align_up(ws, 1024);
        // stride 1: dx = fwd conv of dy with W'[ci][co][t] = W[co][ci][T-1-t] (P18)
        if (w && (st = tc_pack_weights(w, wp, d->out_channels, d->in_channels, g.T, 1, s)) != HEX_OK) return st;
        TcConvArgs a{};
        a.g = g; a.Cin = d->out_channels; a.Cout = d->in_channels;
        a.x = dy; a.wpack = wp; a.bias = nullptr; a.y = dx; a.relu_y = relu_y; a.relu = 0;
        return tc_conv_fwd(a, s);
    }
    if (!w) return HEX_ERR_INVALID_ARG;  // w == NULL (prepacked) only on the stride-1 tensor-core path
    if (use_lat_dgrad(d, g) && aligned16(dy) && aligned16(dx) && (!relu_y || aligned16(relu_y))) {
        // stride s: phase classes (lat_dgrad.cu); a class list or staging that does not fit falls through
        st = lat_dgrad(g, d->in_channels, d->out_channels, dy, w, relu_y, dx, ws, ws_bytes, s);
        if (st != HEX_ERR_UNSUPPORTED) return st;
    }
    if (use_tc_bwd_data_up(d, g)) {  // stride s: the stride-1 bwd-data of dy scattered onto the full grid
        if (!aligned16(dy) || !aligned16(dx) || !aligned16(w) || (relu_y && !aligned16(relu_y)))
            return HEX_ERR_ALIGNMENT;
        if (!ws || ws_bytes < up_bytes(d, g) + packed_weight_bytes(d, g)) return HEX_ERR_WORKSPACE;
        void* up = align_up(ws, 1024);
        void* wp = align_up((char*)up + (up_bytes(d, g) - 2048), 1024);
        if ((st = lattice_upsample(dy, up, g, d->out_channels, s)) != HEX_OK) return st;
        if ((st = tc_pack_weights(w, wp, d->out_channels, d->in_channels, g.T, 1, s)) != HEX_OK) return st;
        TcConvArgs a{};
        a.g = stride1(g); a.Cin = d->out_channels; a.Cout = d->in_channels;
        a.x = up; a.wpack = wp; a.bias = nullptr; a.y = dx; a.relu_y = relu_y; a.relu = 0;
        return tc_conv_fwd(a, s);
    }
    if (use_tf32_bwd_data(d, g))
        return tf32_conv(g, d->in_channels, d->out_channels, 1, (const float*)dy, (const float*)w, nullptr,
                         (const float*)relu_y, 0, (float*)dx, ws, ws_bytes, s);
    if (tiled_supported(g, d->dtype, d->layout))
        return tiled_conv((const float*)dy, (const float*)w, nullptr, (const float*)relu_y, (float*)dx, g,
                          d->out_channels, d->in_channels, 0, 1, s);
    DirectConvArgs a = make_direct(d, g);
    a.dy = dy; a.w = w; a.relu_y = relu_y; a.dx = dx;
    return direct_conv_bwd_data(a, s);
}

hex_status_t hex_conv2d_pack_weights(int32_t count, const hex_conv2d_desc_t* descs, const int32_t* passes,
                                     const void* const* w, void* const* ws, const size_t* ws_bytes,
                                     hex_stream_t stream) {
    if (count < 0 || count > HEX_PACK_MAX) return HEX_ERR_INVALID_ARG;
    if (count == 0) return HEX_OK;
    if (!descs || !passes || !w || !ws || !ws_bytes) return HEX_ERR_INVALID_ARG;
    PackSegs segs{};
    int64_t begin = 0;
    for (int i = 0; i < count; ++i) {
        const hex_conv2d_desc_t* d = &descs[i];
        Geom g;
        const hex_status_t st = conv_geom(d, &g);
        if (st != HEX_OK) return st;
        if (!w[i] || !ws[i]) return HEX_ERR_INVALID_ARG;
        if (passes[i] != 0 && passes[i] != 1) return HEX_ERR_INVALID_ARG;
        if (!(passes[i] == 0 ? use_tc_fwd(d, g) : use_tc_bwd_data(d, g))) return HEX_ERR_UNSUPPORTED;
        if (ws_bytes[i] < packed_weight_bytes(d, g)) return HEX_ERR_WORKSPACE;
        if (!aligned16(w[i])) return HEX_ERR_ALIGNMENT;
        PackSeg& sg = segs.seg[i];
        sg.row0 = begin;
        sg.Cout = d->out_channels; sg.Cin = d->in_channels; sg.T = g.T; sg.tr = passes[i];
        sg.w = w[i];
        sg.wpack = align_up(ws[i], 1024);
        begin += sg.tr ? sg.Cin : sg.Cout;
    }
    segs.count = count;
    return tc_pack_weights_multi(segs, (cudaStream_t)stream);
}

hex_status_t hex_conv2d_bwd_weight(const hex_conv2d_desc_t* d, const void* x, const void* dy, float* dw,
                                   float* dbias, int32_t accumulate, void* ws, size_t ws_bytes,
                                   hex_stream_t stream) {
    Geom g;
    hex_status_t st = conv_geom(d, &g);
    if (st != HEX_OK) return st;
    if (!x || !dy || !dw) return HEX_ERR_INVALID_ARG;
    cudaStream_t s = (cudaStream_t)stream;
    if (use_tc_wgrad(d, g)) {
        if (!aligned16(x) || !aligned16(dy)) return HEX_ERR_ALIGNMENT;
        const size_t need = tc_wgrad_ws_bytes(g, d->in_channels, d->out_channels);
        if (need && (!ws || ws_bytes < need)) return HEX_ERR_WORKSPACE;
        TcWgradArgs a{};
        a.g = g; a.Cin = d->in_channels; a.Cout = d->out_channels;
        a.x = x; a.dy = dy; a.dw = dw; a.dbias = dbias; a.accumulate = accumulate;
        return tc_conv_wgrad(a, ws, ws_bytes, s);
    }
    if (use_tc_wgrad_lat(d, g)) {  // s = 2, 3: the lattice walked directly, x boxes with element stride s
        if (!aligned16(x) || !aligned16(dy)) return HEX_ERR_ALIGNMENT;
        TcWgradArgs a{};
        a.g = g; a.Cin = d->in_channels; a.Cout = d->out_channels;
        a.x = x; a.dy = dy; a.dw = dw; a.dbias = dbias; a.accumulate = accumulate;
        return tc_conv_wgrad(a, ws, ws_bytes, s);
    }
    if (use_tc_wgrad_up(d, g)) {  // stride s: the stride-1 weight gradient against dy on the full grid
        if (!aligned16(x) || !aligned16(dy)) return HEX_ERR_ALIGNMENT;
        const Geom g1 = stride1(g);
        const size_t ub = up_bytes(d, g), need = tc_wgrad_ws_bytes(g1, d->in_channels, d->out_channels);
        if (!ws || ws_bytes < ub + need) return HEX_ERR_WORKSPACE;
        void* up = align_up(ws, 1024);
        char* rest = (char*)align_up((char*)up + (ub - 2048), 1024);
        if ((st = lattice_upsample(dy, up, g, d->out_channels, s)) != HEX_OK) return st;
        TcWgradArgs a{};
        a.g = g1; a.Cin = d->in_channels; a.Cout = d->out_channels;
        a.x = x; a.dy = up; a.dw = dw; a.dbias = dbias; a.accumulate = accumulate;
        return tc_conv_wgrad(a, rest, ws_bytes - (size_t)(rest - (char*)ws), s);
    }
    if (use_tf32_wgrad(d, g))
        return tf32_wgrad(g, d->in_channels, d->out_channels, (const float*)x, (const float*)dy, dw, dbias,
                          accumulate, ws, ws_bytes, s);
    if (use_smallc(d, g)) {
        const size_t need = smallc_wgrad_ws_bytes(g, d->out_channels);
        if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
        if (((uintptr_t)dy & 3) != 0) return HEX_ERR_ALIGNMENT;
        return smallc_wgrad(x, dy, dw, dbias, accumulate, g, d->out_channels, ws, s);
    }
    if (use_c1(d, g)) {
        if (!ws || ws_bytes < c1_wgrad_ws_bytes(g, d->out_channels)) return HEX_ERR_WORKSPACE;
        return c1_conv_wgrad((const float*)x, (const float*)dy, dw, dbias, accumulate, g, d->out_channels, ws, s);
    }
    if (use_f32wg(d, g)) {
        if (!ws || ws_bytes < f32_wgrad_ws_bytes(g, d->in_channels, d->out_channels)) return HEX_ERR_WORKSPACE;
        return f32_wgrad((const float*)x, (const float*)dy, dw, dbias, accumulate, g, d->in_channels,
                         d->out_channels, ws, s);
    }
    const size_t need = direct_wgrad_ws_bytes(g, d->in_channels, d->out_channels);
    if (!ws || ws_bytes < need) return HEX_ERR_WORKSPACE;
    DirectConvArgs a = make_direct(d, g);
    a.x = x; a.dy = dy; a.dw = dw; a.dbias = dbias; a.accumulate = accumulate;
    return direct_conv_bwd_weight(a, ws, s);
}

static hex_status_t pool_geom(const hex_pool2d_desc_t* d, Geom* g) {
    if (!d) return HEX_ERR_INVALID_ARG;
    hex_status_t st = check_common(d->batch, d->channels, d->height, d->width, d->kernel_size, d->stride,
                                   d->parity, d->dtype, d->layout);
    if (st != HEX_OK) return st;
    if (d->kernel_size < 1) return HEX_ERR_INVALID_ARG;
    if (d->mode != HEX_POOL_MAX && d->mode != HEX_POOL_AVG && d->mode != HEX_POOL_AVG_PAD) return HEX_ERR_INVALID_ARG;
    g->B = d->batch; g->H = d->height; g->W = d->width;
    g->n = d->kernel_size; g->s = d->stride; g->parity = d->parity; g->T = hex_taps(d->kernel_size);
    if (g->T > 255) return HEX_ERR_UNSUPPORTED;  // argmax is a uint8 tap index
    if (!out_shape(g->H, g->W, g->s, g->parity, &g->Ho, &g->Wo, nullptr)) return HEX_ERR_EMPTY_LATTICE;
    return HEX_OK;
}

static PoolArgs make_pool(const hex_pool2d_desc_t* d, const Geom& g) {
    PoolArgs a{};
    a.g = g;
    a.C = d->channels; a.dtype = d->dtype; a.layout = d->layout; a.mode = d->mode;
    a.sx = make_strides(d->layout, d->channels, g.H, g.W);
    a.sy = make_strides(d->layout, d->channels, g.Ho, g.Wo);
    return a;
}

hex_status_t hex_pool2d_fwd(const hex_pool2d_desc_t* d, const void* x, void* y, uint8_t* argmax_tap,
                            hex_stream_t stream) {
    Geom g;
    hex_status_t st = pool_geom(d, &g);
    if (st != HEX_OK) return st;
    if (!x || !y) return HEX_ERR_INVALID_ARG;
    PoolArgs a = make_pool(d, g);
    if (d->dtype == HEX_BF16 && d->layout == HEX_NHWC && d->channels % 8 == 0) {
        if (!aligned16(x) || !aligned16(y) || (argmax_tap && ((uintptr_t)argmax_tap & 7))) return HEX_ERR_ALIGNMENT;
    }
    a.x = x; a.y = y; a.argmax = argmax_tap;
    return pool_fwd(a, (cudaStream_t)stream);
}

hex_status_t hex_pool2d_bwd(const hex_pool2d_desc_t* d, const void* dy, const uint8_t* argmax_tap, void* dx,
                            hex_stream_t stream) {
    Geom g;
    hex_status_t st = pool_geom(d, &g);
    if (st != HEX_OK) return st;
    if (!dy || !dx) return HEX_ERR_INVALID_ARG;
    if (d->mode == HEX_POOL_MAX && !argmax_tap) return HEX_ERR_INVALID_ARG;
    PoolArgs a = make_pool(d, g);
    if (d->dtype == HEX_BF16 && d->layout == HEX_NHWC && d->channels % 8 == 0) {
        if (!aligned16(dy) || !aligned16(dx) || (argmax_tap && ((uintptr_t)argmax_tap & 7))) return HEX_ERR_ALIGNMENT;
    }
    a.dy = dy; a.argmax_in = argmax_tap; a.dx = dx;
    return pool_bwd(a, (cudaStream_t)stream);
}

hex_status_t hex_pool2d_bwd_relu(const hex_pool2d_desc_t* d, const void* dy, const uint8_t* argmax_tap,
                                 const void* relu_y, void* dx, hex_stream_t stream) {
    Geom g;
    hex_status_t st = pool_geom(d, &g);
    if (st != HEX_OK) return st;
    if (!dy || !dx || !relu_y) return HEX_ERR_INVALID_ARG;
    if (d->mode == HEX_POOL_MAX && !argmax_tap) return HEX_ERR_INVALID_ARG;
    PoolArgs a = make_pool(d, g);
    if (d->dtype == HEX_BF16 && d->layout == HEX_NHWC && d->channels % 8 == 0) {
        if (!aligned16(dy) || !aligned16(dx) || (argmax_tap && ((uintptr_t)argmax_tap & 7))) return HEX_ERR_ALIGNMENT;
    }
    a.dy = dy; a.argmax_in = argmax_tap; a.dx = dx;
    cudaStream_t s = (cudaStream_t)stream;
    if (pool_plane_bwd_n1s2(a, relu_y, s)) {  // mask fused
        count_launch();
        return last_launch_status();
    }
    if ((st = pool_bwd(a, s)) != HEX_OK) return st;
    return relu_bwd((int64_t)g.B * d->channels * g.H * g.W, d->dtype, dx, relu_y, dx, s);
}

size_t hex_head_workspace_size(int32_t B, int32_t K, int32_t C) {
    if (B < 1 || K < 1 || C < 1) return 0;
    return head_ws_bytes(B, K, C);
}

hex_status_t hex_head_fwd_bwd(int32_t B, int32_t HW, int32_t C, int32_t K, const void* feat, const float* wl,
                              const float* bl, const int32_t* labels, float* loss, void* dfeat, float* dwl,
                              float* dbl, void* ws, size_t ws_bytes, hex_stream_t stream) {
    if (B < 1 || HW < 1 || C < 1 || K < 1) return HEX_ERR_SHAPE;
    if (K > 8 || C % 8 != 0) return HEX_ERR_UNSUPPORTED;
    if (!feat || !wl || !bl || !labels || !loss || !dfeat || !dwl || !dbl) return HEX_ERR_INVALID_ARG;
    if (!aligned16(feat) || !aligned16(dfeat)) return HEX_ERR_ALIGNMENT;
    if (!ws || ws_bytes < head_ws_bytes(B, K, C)) return HEX_ERR_WORKSPACE;
    return head_fwd_bwd(B, HW, C, K, feat, wl, bl, labels, loss, dfeat, dwl, dbl, ws, (cudaStream_t)stream);
}

hex_status_t hex_sgd_momentum(int64_t count, float* param, const float* grad, float* mom, float lr, float mu,
                              float grad_scale, void* param_bf16, hex_stream_t stream) {
    if (count < 0) return HEX_ERR_SHAPE;
    if (count > 0 && (!param || !grad || !mom)) return HEX_ERR_INVALID_ARG;
    return sgd_momentum(count, param, grad, mom, lr, mu, grad_scale, param_bf16, (cudaStream_t)stream);
}

hex_status_t hex_relu_bwd(int64_t count, int32_t dtype, const void* dy, const void* y, void* dx,
                          hex_stream_t stream) {
    if (count < 0) return HEX_ERR_SHAPE;
    if (dtype != HEX_F32 && dtype != HEX_BF16) return HEX_ERR_DTYPE;
    if (count > 0 && (!dy || !y || !dx)) return HEX_ERR_INVALID_ARG;
    return relu_bwd(count, dtype, dy, y, dx, (cudaStream_t)stream);
}

hex_status_t hex_cast_f32_bf16(int64_t count, const float* src, void* dst, hex_stream_t stream) {
    if (count < 0) return HEX_ERR_SHAPE;
    if (count > 0 && (!src || !dst)) return HEX_ERR_INVALID_ARG;
    return cast_f32_bf16(count, src, dst, (cudaStream_t)stream);
}

}  // extern "C"
