// zero_probe.cu -- development check: signed-zero behaviour of fmaxf, cvt.rn.relu.bf16x2.f32 and
// __hmax2 on this GPU (decides whether the fused pool may take the window maximum's bits directly).
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__global__ void k(const float* in, uint32_t* out) {
    const float a = in[0], z = in[1];  // -0.0f, +0.0f (loaded so nothing folds)
    out[0] = __float_as_uint(fmaxf(a, z));
    out[1] = __float_as_uint(fmaxf(z, a));
    uint32_t r;
    asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(a), "f"(in[2]));
    out[2] = r;
    __nv_bfloat162 x = __floats2bfloat162_rn(a, z), y = __floats2bfloat162_rn(z, a);
    __nv_bfloat162 m = __hmax2(x, y);
    out[3] = *reinterpret_cast<uint32_t*>(&m);
    m = __hmax2(y, x);
    out[4] = *reinterpret_cast<uint32_t*>(&m);
    out[5] = __heq2_mask(x, y);
}
int main() {
    float h[3] = {-0.0f, 0.0f, -1.5f};
    float* d; uint32_t* o; uint32_t ho[6];
    cudaMalloc(&d, sizeof(h)); cudaMalloc(&o, sizeof(ho));
    cudaMemcpy(d, h, sizeof(h), cudaMemcpyHostToDevice);
    k<<<1, 1>>>(d, o);
    cudaMemcpy(ho, o, sizeof(ho), cudaMemcpyDeviceToHost);
    printf("fmaxf(-0,+0)=%08x fmaxf(+0,-0)=%08x cvt.relu(-0,-1.5)=%08x hmax2=%08x %08x heq2(-0,+0)=%08x\n",
           ho[0], ho[1], ho[2], ho[3], ho[4], ho[5]);
    return 0;
}
