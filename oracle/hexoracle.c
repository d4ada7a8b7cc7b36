/*
 * hexoracle.c -- fp64 CPU oracle for hexagonal convolution and pooling on
 * offset-column data (HexagDLy, arXiv 1903.01814).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * It shares no code, header, table or constant generator with the CUDA
 * library under paper_1903_01814_b200/csrc (and neither includes the other).
 *
 * It computes the plain DEFINITION the paper's sub-kernel construction
 * reaches ("the results of the sub-convolutions are then merged and added to
 * receive the convolved hexagonal data", Sec. 2.3): a
 * cross-correlation over the hexagonal neighbourhood of each kernel centre,
 * with neighbours enumerated in AXIAL coordinates and converted back to the
 * offset (tensor) index.  No blocking, fusion or reordering.
 *
 * Readings of the paper that this file freezes are listed in DESIGN.md
 * section "Readings" (A1..A20); the ones used here are cited inline.
 *
 * Layout: every tensor is dense NCHW float64, row-major:
 *   x[b][c][r][col], weights w[co][ci][t] with t in canonical tap order.
 * Parity pi (A1): pi=0 -> odd tensor columns are physically half a pitch
 * LOWER (they were "shifted upwards" into alignment);
 * pi=1 is the mirror.
 *
 * Parity pinned: every function below is pinned by tests/test_oracle_pins.py
 * (see DESIGN.md "Oracle pins").  Parity unpinned: none, except the two
 * readings A6 (omitted steps = truncate) and A8 (avg divisor = in-grid count)
 * which cannot be checked against the original library.
 *
 * Build: gcc -O2 -fopenmp -shared -fPIC -o liboracle.so hexoracle.c -lm
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <math.h>

/* ------------------------------------------------------------------ */
/* Coordinates (Sec. 2.1)             */
/* ------------------------------------------------------------------ */

static int64_t floordiv(int64_t a, int64_t b) {
    int64_t q = a / b;
    if ((a % b != 0) && ((a < 0) != (b < 0))) q -= 1;
    return q;
}
static int64_t posmod(int64_t a, int64_t b) {
    int64_t m = a % b;
    return m < 0 ? m + b : m;
}

/* offset (row, col) -> axial (q, ra).  q = col; ra = row - floor((col+pi)/2).
 * Moving down a column is +ra; stepping to column col+1 at the physically
 * lower-right neighbour is (+1, 0). */
void oracle_offset_to_axial(int64_t row, int64_t col, int pi, int64_t* q, int64_t* ra) {
    *q = col;
    *ra = row - floordiv(col + pi, 2);
}

void oracle_axial_to_offset(int64_t q, int64_t ra, int pi, int64_t* row, int64_t* col) {
    *col = q;
    *row = ra + floordiv(q + pi, 2);
}

/* Physical pixel centre (Fig.1 caption, 114-118): columns are
 * sqrt(3)/2 pitch apart; rows 1 pitch apart; the physically lower columns
 * ((col+pi) odd) sit half a pitch further down. y grows upward. */
void oracle_pixel_center(int64_t row, int64_t col, int pi, double pitch, double* x, double* y) {
    *x = (double)col * (sqrt(3.0) / 2.0) * pitch;
    *y = -((double)row + 0.5 * (double)posmod(col + pi, 2)) * pitch;
}

/* Hexagonal graph distance between two axial coordinates. */
int64_t oracle_hex_distance(int64_t q1, int64_t r1, int64_t q2, int64_t r2) {
    int64_t dq = q1 - q2, dr = r1 - r2, ds = dq + dr;
    return (llabs(dq) + llabs(dr) + llabs(ds)) / 2;
}

/* ------------------------------------------------------------------ */
/* Kernel taps (Sec. 2.2): a hexagonal kernel of size n  */
/* covers every pixel within n "layers of neighbouring elements", i.e.   */
/* hex distance <= n.  Canonical element order (A2): column-major        */
/* left->right, top->bottom = lexicographic order of axial (dq, dr).     */
/* ------------------------------------------------------------------ */

/* Fills dq[], dr[] (capacity cap) and returns the number of taps, or -1. */
int oracle_tap_list(int n, int cap, int* dq, int* dr) {
    if (n < 0) return -1;
    int count = 0;
    for (int a = -n; a <= n; ++a)          /* columns left -> right */
        for (int b = -n; b <= n; ++b) {    /* top -> bottom within the column */
            if (oracle_hex_distance(a, b, 0, 0) <= n) {
                if (count < cap) { dq[count] = a; dr[count] = b; }
                ++count;
            }
        }
    return count;
}

int oracle_num_taps(int n) {
    return oracle_tap_list(n, 0, NULL, NULL);
}

/* Offset displacement (dc, drow) of every tap for a centre in a column of
 * parity p = (col + pi) mod 2, by converting through axial coordinates.
 * Test hook for the bit-exact tap-table check. */
int oracle_tap_offsets(int n, int p, int cap, int* dc, int* drow) {
    int T = oracle_num_taps(n);
    if (T < 0 || T > cap) return -1;
    int* dq = (int*)malloc(sizeof(int) * T);
    int* dr = (int*)malloc(sizeof(int) * T);
    oracle_tap_list(n, T, dq, dr);
    /* centre at offset (row 0, col p) with pi = 0: its column parity is p */
    int64_t q0, r0;
    oracle_offset_to_axial(0, p, 0, &q0, &r0);
    for (int t = 0; t < T; ++t) {
        int64_t rr, cc;
        oracle_axial_to_offset(q0 + dq[t], r0 + dr[t], 0, &rr, &cc);
        dc[t] = (int)(cc - p);
        drow[t] = (int)rr;
    }
    free(dq); free(dr);
    return T;
}

/* ------------------------------------------------------------------ */
/* Stride lattice ("symmetric strides in equally sized   */
/* steps along the three symmetry axes ... starting from the top left    */
/* cell"; "centred on a pixel that is part of the actual */
/* input tensor"; "steps that would lead to an output with columns of    */
/* unequal length are neglected").                                        */
/*                                                                        */
/* Lattice = anchor pixel (0,0) + s * (integer combinations of the axial */
/* unit steps (1,0) and (0,1)).  Output column C is input column s*C;    */
/* its lattice rows are enumerated literally; all columns are truncated  */
/* to the shortest one (reading A6).                                      */
/* ------------------------------------------------------------------ */

/* Lattice rows (ascending, only rows inside [0,H)) of input column s*C:
 * the cells of that column whose axial coordinate differs from the anchor's
 * by s times an integer vector.  Returns their count; writes up to cap. */
static int lattice_rows(int H, int s, int pi, int C, int cap, int* rows) {
    int64_t qa, ra_anchor;
    oracle_offset_to_axial(0, 0, pi, &qa, &ra_anchor);
    int64_t q = (int64_t)s * C;           /* (q - qa) = s*C is a multiple of s */
    int count = 0;
    for (int64_t rr = 0; rr < H; ++rr) {
        int64_t qq, ra;
        oracle_offset_to_axial(rr, q, pi, &qq, &ra);
        if (posmod(ra - ra_anchor, s) == 0) {
            if (count < cap) rows[count] = (int)rr;
            ++count;
        }
    }
    return count;
}

/* Output shape.  Returns 0 on success, 1 if the lattice is empty (A7),
 * 2 for invalid arguments. pi_out: parity convention of the output grid
 * (which output columns are physically lower). */
int oracle_out_shape(int H, int W, int s, int pi, int* Ho, int* Wo, int* pi_out) {
    if (H < 1 || W < 1 || s < 1 || (pi != 0 && pi != 1)) return 2;
    int wo = 0;
    for (int c = 0; c < W; c += s) ++wo;   /* input columns s*C inside the grid */
    int ho = -1;
    for (int C = 0; C < wo; ++C) {
        int cnt = lattice_rows(H, s, pi, C, 0, NULL);
        if (ho < 0 || cnt < ho) ho = cnt;
    }
    *Wo = wo;
    *Ho = ho < 0 ? 0 : ho;
    /* physical height of the top lattice centre of output columns 0 and 1
     * (on a grid tall enough that both exist) */
    int top0 = 0, top1 = 0;
    lattice_rows(2 * s + 2, s, pi, 0, 1, &top0);
    lattice_rows(2 * s + 2, s, pi, 1, 1, &top1);
    double x0, y0, x1, y1;
    oracle_pixel_center(top0, 0, pi, 1.0, &x0, &y0);
    oracle_pixel_center(top1, s, pi, 1.0, &x1, &y1);
    /* output column 1 physically lower than column 0 -> odd columns lower -> 0 */
    *pi_out = (y1 < y0) ? 0 : 1;
    return (*Ho <= 0 || *Wo <= 0) ? 1 : 0;
}

/* Centre (row, col) in the input grid of output element (R, C). */
static void lattice_centre(int H, int s, int pi, int R, int C, int* row, int* col) {
    int* rows = (int*)malloc(sizeof(int) * (size_t)(H + 1));
    lattice_rows(H, s, pi, C, H + 1, rows);
    *row = rows[R];
    *col = s * C;
    free(rows);
}

/* Gather map (test hook): map[(R*Wo + C)*T + t] = r*W + c of tap t of output
 * (R,C), or -1 when that neighbour lies outside the grid. */
int oracle_gather_map(int H, int W, int n, int s, int pi, int32_t* map) {
    int Ho, Wo, po;
    int st = oracle_out_shape(H, W, s, pi, &Ho, &Wo, &po);
    if (st) return st;
    int T = oracle_num_taps(n);
    int* dq = (int*)malloc(sizeof(int) * T);
    int* dr = (int*)malloc(sizeof(int) * T);
    oracle_tap_list(n, T, dq, dr);
    for (int R = 0; R < Ho; ++R)
        for (int C = 0; C < Wo; ++C) {
            int r, c;
            lattice_centre(H, s, pi, R, C, &r, &c);
            int64_t q0, a0;
            oracle_offset_to_axial(r, c, pi, &q0, &a0);
            for (int t = 0; t < T; ++t) {
                int64_t rr, cc;
                oracle_axial_to_offset(q0 + dq[t], a0 + dr[t], pi, &rr, &cc);
                int32_t v = -1;
                if (rr >= 0 && rr < H && cc >= 0 && cc < W) v = (int32_t)(rr * W + cc);
                map[((int64_t)R * Wo + C) * T + t] = v;
            }
        }
    free(dq); free(dr);
    return 0;
}

/* Shared helper: the gather map of a problem, allocated. */
static int32_t* build_map(int H, int W, int n, int s, int pi, int* Ho, int* Wo, int* T) {
    int po;
    if (oracle_out_shape(H, W, s, pi, Ho, Wo, &po)) return NULL;
    *T = oracle_num_taps(n);
    int32_t* map = (int32_t*)malloc(sizeof(int32_t) * (size_t)(*Ho) * (*Wo) * (*T));
    oracle_gather_map(H, W, n, s, pi, map);
    return map;
}

/* ------------------------------------------------------------------ */
/* Convolution (A3 cross-correlation, A4 zero */
/* contribution from out-of-grid neighbours, A12 optional bias).         */
/* y[b][co][R][C] = bias[co] + sum_ci sum_t w[co][ci][t] * x[b][ci][nb_t] */
/* ------------------------------------------------------------------ */
int oracle_conv2d_fwd(int B, int Ci, int Co, int H, int W, int n, int s, int pi,
                      const double* x, const double* w, const double* bias, double* y) {
    int Ho, Wo, T;
    int32_t* map = build_map(H, W, n, s, pi, &Ho, &Wo, &T);
    if (!map) return 1;
    const int64_t HW = (int64_t)H * W, HWo = (int64_t)Ho * Wo;
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int co = 0; co < Co; ++co)
            for (int64_t o = 0; o < HWo; ++o) {
                double acc = 0.0;
                for (int ci = 0; ci < Ci; ++ci)
                    for (int t = 0; t < T; ++t) {
                        int32_t m = map[o * T + t];
                        if (m >= 0)
                            acc += w[((int64_t)co * Ci + ci) * T + t] *
                                   x[((int64_t)b * Ci + ci) * HW + m];
                    }
                y[((int64_t)b * Co + co) * HWo + o] = (bias ? bias[co] : 0.0) + acc;
            }
    free(map);
    return 0;
}

/* Backward of the convolution: the literal adjoint of the forward map,
 * written as a scatter over every (output, tap) pair that touched an in-grid
 * input cell.  Any output pointer may be NULL to skip that gradient. */
int oracle_conv2d_bwd(int B, int Ci, int Co, int H, int W, int n, int s, int pi,
                      const double* x, const double* w, const double* dy,
                      double* dx, double* dw, double* dbias) {
    int Ho, Wo, T;
    int32_t* map = build_map(H, W, n, s, pi, &Ho, &Wo, &T);
    if (!map) return 1;
    const int64_t HW = (int64_t)H * W, HWo = (int64_t)Ho * Wo;
    if (dx) {
        #pragma omp parallel for collapse(2) schedule(static)
        for (int b = 0; b < B; ++b)
            for (int ci = 0; ci < Ci; ++ci) {
                double* dxp = dx + ((int64_t)b * Ci + ci) * HW;
                for (int64_t i = 0; i < HW; ++i) dxp[i] = 0.0;
                for (int co = 0; co < Co; ++co)
                    for (int64_t o = 0; o < HWo; ++o) {
                        double g = dy[((int64_t)b * Co + co) * HWo + o];
                        for (int t = 0; t < T; ++t) {
                            int32_t m = map[o * T + t];
                            if (m >= 0) dxp[m] += w[((int64_t)co * Ci + ci) * T + t] * g;
                        }
                    }
            }
    }
    if (dw) {
        #pragma omp parallel for collapse(2) schedule(static)
        for (int co = 0; co < Co; ++co)
            for (int ci = 0; ci < Ci; ++ci) {
                double* dwp = dw + ((int64_t)co * Ci + ci) * T;
                for (int t = 0; t < T; ++t) dwp[t] = 0.0;
                for (int b = 0; b < B; ++b)
                    for (int64_t o = 0; o < HWo; ++o) {
                        double g = dy[((int64_t)b * Co + co) * HWo + o];
                        for (int t = 0; t < T; ++t) {
                            int32_t m = map[o * T + t];
                            if (m >= 0) dwp[t] += g * x[((int64_t)b * Ci + ci) * HW + m];
                        }
                    }
            }
    }
    if (dbias) {
        for (int co = 0; co < Co; ++co) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b)
                for (int64_t o = 0; o < HWo; ++o) acc += dy[((int64_t)b * Co + co) * HWo + o];
            dbias[co] = acc;
        }
    }
    free(map);
    return 0;
}

/* ------------------------------------------------------------------ */
/* Pooling (sub-convolutions replaced by pooling and    */
/* combined with aggregation functions, same padding/striding scheme).    */
/* mode 0 = max: max over in-grid neighbours (A8), ties -> first in       */
/* canonical order (A9); argmax is the tap index.                          */
/* mode 1 = avg: in-grid sum / in-grid count (A8).                         */
/* mode 2 = include-pad avg: in-grid sum / T(n), i.e. off-grid cells are   */
/*          zeros in the average (the alternative reading of A8, f4).      */
/* ------------------------------------------------------------------ */
int oracle_pool2d_fwd(int B, int Cc, int H, int W, int n, int s, int pi, int mode,
                      const double* x, double* y, uint8_t* argmax) {
    if (n < 1 || mode < 0 || mode > 2) return 2;
    int Ho, Wo, T;
    int32_t* map = build_map(H, W, n, s, pi, &Ho, &Wo, &T);
    if (!map) return 1;
    const int64_t HW = (int64_t)H * W, HWo = (int64_t)Ho * Wo;
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < Cc; ++c)
            for (int64_t o = 0; o < HWo; ++o) {
                const double* xp = x + ((int64_t)b * Cc + c) * HW;
                int64_t oi = ((int64_t)b * Cc + c) * HWo + o;
                if (mode == 0) {
                    int best = -1;
                    double bv = 0.0;
                    for (int t = 0; t < T; ++t) {
                        int32_t m = map[o * T + t];
                        if (m < 0) continue;
                        if (best < 0 || xp[m] > bv) { best = t; bv = xp[m]; }
                    }
                    y[oi] = bv;
                    if (argmax) argmax[oi] = (uint8_t)best;
                } else {
                    double acc = 0.0;
                    int cnt = 0;
                    for (int t = 0; t < T; ++t) {
                        int32_t m = map[o * T + t];
                        if (m < 0) continue;
                        acc += xp[m];
                        ++cnt;
                    }
                    y[oi] = acc / (double)(mode == 2 ? T : cnt);
                }
            }
    free(map);
    return 0;
}

/* Pool backward: max routes dy to the argmax cell; avg spreads dy/count
 * (include-pad: dy/T) over the in-grid neighbourhood (adjoint of the forward). */
int oracle_pool2d_bwd(int B, int Cc, int H, int W, int n, int s, int pi, int mode,
                      const double* dy, const uint8_t* argmax, double* dx) {
    if (n < 1 || mode < 0 || mode > 2) return 2;
    int Ho, Wo, T;
    int32_t* map = build_map(H, W, n, s, pi, &Ho, &Wo, &T);
    if (!map) return 1;
    const int64_t HW = (int64_t)H * W, HWo = (int64_t)Ho * Wo;
    if (mode == 0) {
        /* The argmax comes from the implementation under test: validate every entry before routing
         * (a tap index >= T or one that names an off-grid neighbour is an error, not a write). */
        if (!argmax) { free(map); return 2; }
        for (int64_t oi = 0; oi < (int64_t)B * Cc * HWo; ++oi) {
            const int a = argmax[oi];
            if (a >= T || map[(oi % HWo) * T + a] < 0) { free(map); return 3; }
        }
    }
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int c = 0; c < Cc; ++c) {
            double* dxp = dx + ((int64_t)b * Cc + c) * HW;
            for (int64_t i = 0; i < HW; ++i) dxp[i] = 0.0;
            for (int64_t o = 0; o < HWo; ++o) {
                int64_t oi = ((int64_t)b * Cc + c) * HWo + o;
                double g = dy[oi];
                if (mode == 0) {
                    int32_t m = map[o * T + argmax[oi]];
                    dxp[m] += g;
                } else {
                    int cnt = 0;
                    for (int t = 0; t < T; ++t) if (map[o * T + t] >= 0) ++cnt;
                    if (mode == 2) cnt = T;
                    for (int t = 0; t < T; ++t) {
                        int32_t m = map[o * T + t];
                        if (m >= 0) dxp[m] += g / (double)cnt;
                    }
                }
            }
        }
    free(map);
    return 0;
}

/* ------------------------------------------------------------------ */
/* 3-D hexagonal convolution (Sec. 2 "Software          */
/* Functionalities": "hexagonal layout in the x-y-plane while data points */
/* along the z-axis are assumed to be equidistant").     */
/* The kernel is a hexagonal kernel of size n in every one of kd depth    */
/* slices, with independent weights w[co][ci][kz][t] (t canonical, A2);   */
/* kd odd, the depth window centred on the output slice (kz = dz +        */
/* (kd-1)/2), zero padding in depth (A4 along z); depth stride sd takes   */
/* centres 0, sd, 2sd, ... (Do = (D-1)/sd + 1); in-plane lattice as the   */
/* 2-D convolution (A5, A6).  Layout x[b][ci][z][r][c].                   */
/* y[b][co][zo][R][C] = bias[co] + sum_ci sum_kz sum_t                    */
/*                      w[co][ci][kz][t] * x[b][ci][sd*zo+kz-(kd-1)/2][nb_t] */
/* ------------------------------------------------------------------ */
int oracle_conv3d_out_depth(int D, int kd, int sd) {
    if (D < 1 || kd < 1 || (kd & 1) == 0 || sd < 1) return -1;
    return (D - 1) / sd + 1;
}

int oracle_conv3d_fwd(int B, int Ci, int Co, int D, int H, int W, int n, int kd, int s, int sd, int pi,
                      const double* x, const double* w, const double* bias, double* y) {
    const int Do = oracle_conv3d_out_depth(D, kd, sd);
    if (Do < 0) return 2;
    int Ho, Wo, T;
    int32_t* map = build_map(H, W, n, s, pi, &Ho, &Wo, &T);
    if (!map) return 1;
    const int64_t HW = (int64_t)H * W, HWo = (int64_t)Ho * Wo;
    const int pd = (kd - 1) / 2;
    #pragma omp parallel for collapse(2) schedule(static)
    for (int b = 0; b < B; ++b)
        for (int co = 0; co < Co; ++co)
            for (int zo = 0; zo < Do; ++zo)
                for (int64_t o = 0; o < HWo; ++o) {
                    double acc = 0.0;
                    for (int ci = 0; ci < Ci; ++ci)
                        for (int kz = 0; kz < kd; ++kz) {
                            const int z = sd * zo + kz - pd;
                            if (z < 0 || z >= D) continue;
                            const double* xs = x + (((int64_t)b * Ci + ci) * D + z) * HW;
                            const double* ws = w + (((int64_t)co * Ci + ci) * kd + kz) * T;
                            for (int t = 0; t < T; ++t) {
                                const int32_t m = map[o * T + t];
                                if (m >= 0) acc += ws[t] * xs[m];
                            }
                        }
                    y[(((int64_t)b * Co + co) * Do + zo) * HWo + o] = (bias ? bias[co] : 0.0) + acc;
                }
    free(map);
    return 0;
}

/* Backward of the 3-D convolution: the literal adjoint (scatter over every
 * (output, depth tap, tap) that touched an in-grid, in-depth input cell). */
int oracle_conv3d_bwd(int B, int Ci, int Co, int D, int H, int W, int n, int kd, int s, int sd, int pi,
                      const double* x, const double* w, const double* dy,
                      double* dx, double* dw, double* dbias) {
    const int Do = oracle_conv3d_out_depth(D, kd, sd);
    if (Do < 0) return 2;
    int Ho, Wo, T;
    int32_t* map = build_map(H, W, n, s, pi, &Ho, &Wo, &T);
    if (!map) return 1;
    const int64_t HW = (int64_t)H * W, HWo = (int64_t)Ho * Wo;
    const int pd = (kd - 1) / 2;
    if (dx) {
        #pragma omp parallel for collapse(2) schedule(static)
        for (int b = 0; b < B; ++b)
            for (int ci = 0; ci < Ci; ++ci) {
                double* dxp = dx + ((int64_t)b * Ci + ci) * D * HW;
                for (int64_t i = 0; i < (int64_t)D * HW; ++i) dxp[i] = 0.0;
                for (int co = 0; co < Co; ++co)
                    for (int zo = 0; zo < Do; ++zo)
                        for (int kz = 0; kz < kd; ++kz) {
                            const int z = sd * zo + kz - pd;
                            if (z < 0 || z >= D) continue;
                            const double* ws = w + (((int64_t)co * Ci + ci) * kd + kz) * T;
                            for (int64_t o = 0; o < HWo; ++o) {
                                const double g = dy[(((int64_t)b * Co + co) * Do + zo) * HWo + o];
                                for (int t = 0; t < T; ++t) {
                                    const int32_t m = map[o * T + t];
                                    if (m >= 0) dxp[(int64_t)z * HW + m] += ws[t] * g;
                                }
                            }
                        }
            }
    }
    if (dw) {
        #pragma omp parallel for collapse(2) schedule(static)
        for (int co = 0; co < Co; ++co)
            for (int ci = 0; ci < Ci; ++ci)
                for (int kz = 0; kz < kd; ++kz) {
                    double* dwp = dw + (((int64_t)co * Ci + ci) * kd + kz) * T;
                    for (int t = 0; t < T; ++t) dwp[t] = 0.0;
                    for (int b = 0; b < B; ++b)
                        for (int zo = 0; zo < Do; ++zo) {
                            const int z = sd * zo + kz - pd;
                            if (z < 0 || z >= D) continue;
                            const double* xs = x + (((int64_t)b * Ci + ci) * D + z) * HW;
                            for (int64_t o = 0; o < HWo; ++o) {
                                const double g = dy[(((int64_t)b * Co + co) * Do + zo) * HWo + o];
                                for (int t = 0; t < T; ++t) {
                                    const int32_t m = map[o * T + t];
                                    if (m >= 0) dwp[t] += g * xs[m];
                                }
                            }
                        }
                }
    }
    if (dbias) {
        for (int co = 0; co < Co; ++co) {
            double acc = 0.0;
            for (int b = 0; b < B; ++b)
                for (int64_t i = 0; i < (int64_t)Do * HWo; ++i) acc += dy[((int64_t)b * Co + co) * Do * HWo + i];
            dbias[co] = acc;
        }
    }
    free(map);
    return 0;
}

/* Thread count of the OpenMP loops (timing the oracle single-threaded for bench.py's cpu_baseline). */
void oracle_set_threads(int n) {
#ifdef _OPENMP
    extern void omp_set_num_threads(int);
    if (n >= 1) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int oracle_max_threads(void) {
#ifdef _OPENMP
    extern int omp_get_max_threads(void);
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/* ------------------------------------------------------------------ */
/* Point evaluation of the weight gradient (same definition as          */
/* oracle_conv2d_bwd, evaluated only at listed (co, ci, t)) for full-   */
/* size checks where the dense fp64 oracle would not fit in memory.     */
/* x / dy are given in their storage format (fmt 0 = float32, 1 = bf16  */
/* bit patterns; both convert exactly to double) with element strides   */
/* (b, c, h, w).  pts = npts triples (co, ci, t); out[npts].             */
/* ------------------------------------------------------------------ */
static double load_any(const void* p, int fmt, int64_t i) {
    if (fmt == 0) return (double)((const float*)p)[i];
    uint32_t u = (uint32_t)((const uint16_t*)p)[i] << 16;
    float f;
    memcpy(&f, &u, 4);
    return (double)f;
}

int oracle_conv2d_bwd_weight_at(int B, int H, int W, int n, int s, int pi,
                                const void* x, int x_fmt, const int64_t* xs,
                                const void* dy, int dy_fmt, const int64_t* dys,
                                int npts, const int32_t* pts, double* out) {
    int Ho, Wo, T;
    int32_t* map = build_map(H, W, n, s, pi, &Ho, &Wo, &T);
    if (!map) return 1;
    #pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < npts; ++k) {
        const int co = pts[3 * k], ci = pts[3 * k + 1], t = pts[3 * k + 2];
        double acc = 0.0;
        for (int b = 0; b < B; ++b)
            for (int R = 0; R < Ho; ++R)
                for (int C = 0; C < Wo; ++C) {
                    int32_t m = map[((int64_t)R * Wo + C) * T + t];
                    if (m < 0) continue;
                    const int r = m / W, c = m % W;
                    double g = load_any(dy, dy_fmt, b * dys[0] + co * dys[1] + R * dys[2] + C * dys[3]);
                    acc += g * load_any(x, x_fmt, b * xs[0] + ci * xs[1] + r * xs[2] + c * xs[3]);
                }
        out[k] = acc;
    }
    free(map);
    return 0;
}
