// strided.cu -- backward passes of strided hexagonal convolutions on the tensor cores.
//
// A stride-s convolution is the stride-1 convolution sampled at the lattice centres
// (rho(C) + sR, sC) (A5; pin P10).  Its adjoints are therefore the stride-1
// adjoints applied to dy scattered back onto the full grid (zeros between lattice points):
//   dx = bwd_data_s1(up(dy)),  dw = bwd_weight_s1(x, up(dy)).
// This kernel builds up(dy) (bf16 NHWC, 16-byte vectors); the stride-1 tcgen05 kernels do the rest.
// It spends s^2 times the MMA work of a phase decomposition, but runs the strided backward on the
// tensor cores instead of the CUDA-core gather kernels.
#include <cstdint>

#include "common.cuh"
#include "geometry.cuh"
#include "kernels.h"

namespace hexconv {

__global__ void lattice_upsample_kernel(const uint4* __restrict__ dy, uint4* __restrict__ up, Geom g, int C8) {
    const int64_t total = (int64_t)g.B * g.H * g.W * C8;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
        const int c8 = (int)(i % C8);
        int64_t q = i / C8;
        const int c = (int)(q % g.W);
        q /= g.W;
        const int r = (int)(q % g.H);
        const int b = (int)(q / g.H);
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (c % g.s == 0) {
            const int C = c / g.s;
            const int d = r - hex_rho(C, g.s, g.parity);
            if (C < g.Wo && d >= 0 && d % g.s == 0 && d / g.s < g.Ho)
                v = dy[(((int64_t)b * g.Ho + d / g.s) * g.Wo + C) * C8 + c8];
        }
        up[i] = v;
    }
}

hex_status_t lattice_upsample(const void* dy, void* up, const Geom& g, int C, cudaStream_t st) {
    const int64_t total = (int64_t)g.B * g.H * g.W * (C / 8);
    const int64_t blocks = (total + 255) / 256;
    lattice_upsample_kernel<<<(int)(blocks < 148 * 16 ? blocks : 148 * 16), 256, 0, st>>>((const uint4*)dy, (uint4*)up,
                                                                                          g, C / 8);
    count_launch();
    return last_launch_status();
}

}  // namespace hexconv
