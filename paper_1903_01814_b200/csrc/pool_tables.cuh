// pool_tables.cuh -- compile-time candidate tables of the hexagonal max/avg
// pool backward for kernel size n = 1, stride 2 (the configuration of
// BASELINE configs 2, 3 and 5), shared by the NHWC (pool.cu) and NCHW
// (plane_kernels.cu) kernels.
//
// Lattice (A5): output column C sits on input
// column 2C with centre parity P = parity and rho(C) = C & 1.  The input block
// rows {2R', 2R'+1} x columns {2C, 2C+1} is reached only by windows in columns
// C, C+1 and rows R'-1..R'+1; which (window, tap) reaches which pixel depends
// only on (P, rho), listed here (at most two windows per pixel).
#pragma once

namespace hexconv {

struct Cand {
    int dC, dR, tap;  // window (C + dC, R' + dR), tap index; tap < 0: none
};
// candidate k (0/1) of pixel (row 2R' + pr, column 2C + pc) for centre parity P, rho(C) = RHO
__host__ __device__ constexpr Cand blk_cand(int P, int RHO, int pc, int pr, int k) {
    if (pc == 0) {  // column 2C: the window column's own taps 2, 3, 4 (dr = -1, 0, +1)
        if (RHO == 0) {
            if (pr == 0) return k == 0 ? Cand{0, 0, 3} : Cand{0, 0, -1};
            return k == 0 ? Cand{0, 0, 4} : Cand{0, 1, 2};
        }
        if (pr == 0) return k == 0 ? Cand{0, -1, 4} : Cand{0, 0, 2};
        return k == 0 ? Cand{0, 0, 3} : Cand{0, 0, -1};
    }
    // column 2C+1: k = 0 from window column C (dc = +1, taps 5, 6), k = 1 from C+1 (dc = -1, taps 0, 1)
    if (P == 0) {
        if (RHO == 0) {
            if (pr == 0) return k == 0 ? Cand{0, 0, 6} : Cand{1, 0, 0};
            return k == 0 ? Cand{0, 1, 5} : Cand{1, 0, 1};
        }
        if (pr == 0) return k == 0 ? Cand{0, 0, 5} : Cand{1, 0, 1};
        return k == 0 ? Cand{0, 0, 6} : Cand{1, 1, 0};
    }
    if (RHO == 0) {
        if (pr == 0) return k == 0 ? Cand{0, 0, 5} : Cand{1, -1, 1};
        return k == 0 ? Cand{0, 0, 6} : Cand{1, 0, 0};
    }
    if (pr == 0) return k == 0 ? Cand{0, -1, 6} : Cand{1, 0, 0};
    return k == 0 ? Cand{0, 0, 5} : Cand{1, 0, 1};
}
__host__ __device__ constexpr bool blk_uses(int P, int RHO, int dC, int dR) {
    for (int pc = 0; pc < 2; ++pc)
        for (int pr = 0; pr < 2; ++pr)
            for (int k = 0; k < 2; ++k) {
                const Cand c = blk_cand(P, RHO, pc, pr, k);
                if (c.tap >= 0 && c.dC == dC && c.dR == dR) return true;
            }
    return false;
}

}  // namespace hexconv
