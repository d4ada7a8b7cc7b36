// geometry.cuh -- offset-column hexagonal grid geometry for the CUDA path.
//
// Independent of the oracle (oracle/hexoracle.c derives the same facts by
// enumerating axial coordinates; this file uses closed forms):
//
//  * Taps of a size-n kernel (Sec. 2.2): for a centre in a
//    column of parity p = (col + parity) & 1, column offset dc in [-n, n]
//    holds 2n+1-|dc| taps at row offsets top(dc,p) .. top(dc,p)+2n-|dc| with
//    top(dc,p) = -n + floor((|dc| + p) / 2)   (SPEC.md:98 closed form).
//    Canonical tap order (A2): dc ascending, then row ascending.
//  * Stride lattice: output column C is input
//    column s*C, output row R is input row rho(C) + s*R with
//    rho(C) = floor((s*C + parity)/2) mod s; Wo = floor((W-1)/s)+1,
//    Ho = min over C of floor((H-1-rho(C))/s)+1 (rho has period 2 in C).
//  * Output parity: v(C) = 2*rho(C) + ((s*C + parity) & 1) is twice the
//    physical depth of the top centre of output column C; column 1 deeper
//    than column 0 => odd output columns are lower => parity_out = 0.
#pragma once
#include <stdint.h>

namespace hexconv {

__host__ __device__ __forceinline__ int hex_taps(int n) { return 3 * n * (n + 1) + 1; }

__host__ __device__ __forceinline__ int hex_rho(int C, int s, int parity) {
    return ((s * C + parity) >> 1) % s;
}

__host__ __device__ __forceinline__ int tap_top(int n, int dc, int p) {
    int a = dc < 0 ? -dc : dc;
    return -n + ((a + p) >> 1);
}

// Host: output shape; returns false if the lattice is empty.
inline bool out_shape(int H, int W, int s, int parity, int* Ho, int* Wo, int* parity_out) {
    int wo = (W - 1) / s + 1;
    int ho = 1 << 30;
    for (int C = 0; C < (wo < 2 ? wo : 2); ++C) {
        int r = hex_rho(C, s, parity);
        int h = (H - 1 - r) >= 0 ? (H - 1 - r) / s + 1 : 0;
        if (h < ho) ho = h;
    }
    *Wo = wo;
    *Ho = ho;
    int v0 = 2 * hex_rho(0, s, parity) + (parity & 1);
    int v1 = 2 * hex_rho(1, s, parity) + ((s + parity) & 1);
    if (parity_out) *parity_out = (v1 > v0) ? 0 : 1;
    return ho > 0 && wo > 0;
}

// Tap t -> (dc, dr) for centre parity p (host and device; O(n) walk).
__host__ __device__ __forceinline__ void tap_offset(int n, int p, int t, int* dc, int* dr) {
    for (int c = -n; c <= n; ++c) {
        int len = 2 * n + 1 - (c < 0 ? -c : c);
        if (t < len) {
            *dc = c;
            *dr = tap_top(n, c, p) + t;
            return;
        }
        t -= len;
    }
    *dc = 0;
    *dr = 0;
}

// Problem geometry passed by value to kernels.
struct Geom {
    int B, H, W, Ho, Wo;
    int n, s, parity, T;
};

}  // namespace hexconv
