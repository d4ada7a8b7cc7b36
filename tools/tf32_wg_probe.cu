// tf32_wg_probe.cu -- development harness for the 3xTF32 weight-gradient kernel: runs it on a small shape
// with parts switched off (bit 0 MMA, 1 tcgen05.st, 2 TMA, 3 tcgen05.ld) and reports the CUDA status, to
// locate a faulting instruction; then times the config-3 layer-2 / layer-4 shapes.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 --expt-relaxed-constexpr -I include \
//        -DTF_PROF=1 -o tools/tf32_wg_probe.bin tools/tf32_wg_probe.cu -lcuda
#include <cstdio>
#include <cstdlib>
#include "../paper_1903_01814_b200/csrc/tf32_conv.cu"

namespace hexconv {
std::atomic<int64_t> g_launches{0};
bool sw_on(const char*) { return false; }
int sw_int(const char*, int d) { return d; }
double sw_double(const char*, double d) { return d; }
}  // namespace hexconv

using namespace hexconv;

static float run(int B, int Cin, int Cout, int H, int W, int n, int s, int dbg, int reps) {
    Geom g{};
    g.B = B; g.H = H; g.W = W; g.n = n; g.s = s; g.parity = 0; g.T = hex_taps(n);
    out_shape(H, W, s, 0, &g.Ho, &g.Wo, nullptr);
    float *x, *dy, *dw, *db, *ws;
    const size_t wsb = tf32_wgrad_ws_bytes(g, Cin, Cout);
    cudaMalloc(&x, (size_t)B * Cin * H * W * 4);
    cudaMalloc(&dy, (size_t)B * Cout * g.Ho * g.Wo * 4);
    cudaMalloc(&dw, (size_t)Cout * Cin * g.T * 4);
    cudaMalloc(&db, Cout * 4);
    cudaMalloc(&ws, wsb + 1024);
    cudaMemset(x, 0, (size_t)B * Cin * H * W * 4);
    cudaMemset(dy, 0, (size_t)B * Cout * g.Ho * g.Wo * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    hex_status_t st = tf32_wgrad(g, Cin, Cout, x, dy, dw, db, 0, ws, wsb + 1024, 0, dbg);
    cudaError_t e = cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int i = 0; i < reps && e == cudaSuccess; ++i) tf32_wgrad(g, Cin, Cout, x, dy, dw, db, 0, ws, wsb + 1024, 0, dbg);
    cudaEventRecord(e1);
    e = e == cudaSuccess ? cudaDeviceSynchronize() : e;
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("B%d %d->%d %dx%d n%d s%d dbg%d: status %d cuda %s  %.1f us\n", B, Cin, Cout, H, W, n, s, dbg, (int)st,
           cudaGetErrorString(e), reps ? ms * 1e3 / reps : 0.f);
    long long h[32];
    cudaMemcpyFromSymbol(h, g_tf_prof, sizeof(h));
    const char* nm[16] = {"mma wait full", "mma issue", "B wait empty", "B split+store", "B load issue",
                          "-", "A wait xfull", "A gather", "A wait empty", "A st+signal", "", "", "", "", "", ""};
    for (int i = 0; i < 10; ++i) printf("    %-16s %10lld\n", nm[i], h[16 + i]);
    cudaMemset(h, 0, 0);
    cudaFree(x); cudaFree(dy); cudaFree(dw); cudaFree(db); cudaFree(ws);
    return ms;
}

int main(int argc, char** argv) {
    const int dbg = argc > 1 ? atoi(argv[1]) : 0;
    if (argc > 2) {
        run(256, 16, 32, 40, 40, 2, 1, dbg, 10);
        run(256, 32, 64, 20, 20, 1, 1, dbg, 10);
        run(32, 16, 32, 48, 48, 2, 2, dbg, 10);
        return 0;
    }
    run(2, 16, 32, 11, 12, 2, 1, dbg, 0);
    return 0;
}
