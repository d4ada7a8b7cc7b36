// tf32_prof.cu -- development timing probe of the 3xTF32 conv kernel: builds csrc/tf32_conv.cu with
// -DTF_PROF=1 (clock64 accumulators in CTA 0) and runs the config-3 layer-2 forward / bwd-data shapes
// (argument "c2": the config-2 stride-2 layer).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include \
//        -DTF_PROF=1 -o tools/tf32_prof.bin tools/tf32_prof.cu -lcuda
#include <cstdio>
#include <cstring>
#include <vector>
#include "../paper_1903_01814_b200/csrc/tf32_conv.cu"

namespace hexconv {
std::atomic<int64_t> g_launches{0};
bool sw_on(const char*) { return false; }
int sw_int(const char*, int d) { return d; }
double sw_double(const char*, double d) { return d; }
}  // namespace hexconv

int main(int argc, char** argv) {
    using namespace hexconv;
    const int mode = argc > 1 ? atoi(argv[1]) : 0;
    const bool c2 = argc > 2 && !strcmp(argv[2], "c2");  // config 2: 32 x 16 -> 32, 48 x 48, n = 2, stride 2
    const int B = c2 ? 32 : 256, H = c2 ? 48 : 40, W = c2 ? 48 : 40, Cin = 16, Cout = 32, n = 2;
    Geom g{};
    g.B = B; g.H = H; g.W = W; g.n = n; g.s = c2 ? 2 : 1; g.parity = 0; g.T = hex_taps(n);
    g.Ho = c2 ? 24 : H; g.Wo = c2 ? 24 : W;
    float *x, *w, *y, *ws;
    cudaMalloc(&x, (size_t)B * 32 * H * W * 4);
    cudaMalloc(&y, (size_t)B * 32 * H * W * 4);
    cudaMalloc(&w, Cout * Cin * g.T * 4);
    cudaMalloc(&ws, 1 << 20);
    cudaMemset(x, 0, (size_t)B * 32 * H * W * 4);
    cudaMemset(w, 0, Cout * Cin * g.T * 4);
    for (int it = 0; it < 3; ++it)
        tf32_conv(g, Cin, Cout, mode, x, w, nullptr, nullptr, 0, y, ws, 1 << 20, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    hex_status_t st = tf32_conv(g, Cin, Cout, mode, x, w, nullptr, nullptr, 0, y, ws, 1 << 20, 0);
    cudaEventRecord(e1);
    cudaDeviceSynchronize();
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[32];
    cudaMemcpyFromSymbol(h, g_tf_prof, sizeof(h));
    printf("mode %d status %d err %s  %.1f us\n", mode, (int)st, cudaGetErrorString(cudaGetLastError()), ms * 1e3);
    const char* names[16] = {"mma wait full", "mma issue", "", "", "bld gather", "bld split", "bld wait empty",
                             "bld st+signal", "", "", "epi wait tfull", "epi work", "", "", "", ""};
    for (int i = 0; i < 16; ++i)
        if (names[i][0]) printf("  %-16s %12lld cycles\n", names[i], h[i]);
    return 0;
}
