// tc_conv.cu -- tcgen05 implicit-GEMM hexagonal convolution (placeholder: the
// tensor-core path is being brought up; until then every shape takes the
// CUDA-core stencil path).
#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {

bool tc_conv_supported(const Geom&, int, int) { return false; }
bool tc_wgrad_supported(const Geom&, int, int) { return false; }
size_t tc_wgrad_ws_bytes(const Geom&, int, int) { return 0; }
hex_status_t tc_conv_fwd(const TcConvArgs&, cudaStream_t) { return HEX_ERR_UNSUPPORTED; }
hex_status_t tc_conv_wgrad(const TcWgradArgs&, void*, size_t, cudaStream_t) { return HEX_ERR_UNSUPPORTED; }
hex_status_t tc_pack_weights(const void*, void*, int, int, int, int, cudaStream_t) { return HEX_ERR_UNSUPPORTED; }

}  // namespace hexconv
