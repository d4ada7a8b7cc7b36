"""Pins for the fp64 oracle (CPU only).

Each test fixes the oracle against something other than itself: the paper's
statements, SPEC.md's worked examples (tests/golden/spec_examples.json),
physical geometry computed here from the addressing description
(PAPER.md:100-107), closed forms, library reductions (torch fp64 conv2d /
unfold), invariants and finite differences.  Pin ids P1..P18 follow
SURVEY.md section 8(c) and DESIGN.md "Oracle pins".

The physical-geometry helpers below are written from the paper's description
of the addressing scheme and never call the oracle's coordinate code:
column c sits at x = c*sqrt(3)/2, row r at y = -r, and the physically lower
columns ((c+pi) odd) are half a pitch further down.
"""
import json
import math
import os

import numpy as np
import pytest
import torch
import torch.nn.functional as F

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
EPS = 1e-9


# ----------------------------------------------------------------- physical geometry (test-local)
def phys(r, c, pi=0):
    return (c * math.sqrt(3) / 2.0, -(r + 0.5 * ((c + pi) % 2)))


def phys_neigh(H, W, r, c, n, pi=0):
    """In-grid cells within Euclidean distance n (== hex distance <= n for n <= 6),
    ordered left->right (x), top->bottom (y descending)."""
    x0, y0 = phys(r, c, pi)
    cells = []
    for rr in range(H):
        for cc in range(W):
            x, y = phys(rr, cc, pi)
            if (x - x0) ** 2 + (y - y0) ** 2 <= n * n + EPS:
                cells.append((rr, cc))
    cells.sort(key=lambda rc: (rc[1], rc[0]))
    return cells


def phys_tap_offsets(n, p):
    """(dc, drow) offsets of the Euclidean disc of radius n around a centre in a
    column of parity p, sorted column-major left->right, top->bottom."""
    big = 4 * n + 4
    r0 = 2 * n + 2
    c0 = 2 * n + 2 + (p % 2)  # column parity p with pi = 0
    return [(cc - c0, rr - r0) for rr, cc in phys_neigh(2 * big, 2 * big, r0, c0, n)]


def phys_lattice(H, W, s, pi=0):
    """Kernel-centre lattice by brute force on physical positions: cells whose
    position relative to pixel (0,0) is i*s*e_diag + k*s*e_down (integers i,k),
    e_down = (0,-1), e_diag = (sqrt(3)/2, -1/2).  Columns truncated to the
    shortest (reading A6).  Returns rows[C] (list per output column)."""
    xa, ya = phys(0, 0, pi)
    cols = {}
    for cc in range(W):
        if abs(cc / s - round(cc / s)) < 1e-12:   # i integer <=> a lattice column
            cols[cc] = []
        for rr in range(H):
            x, y = phys(rr, cc, pi)
            i = (x - xa) / (s * math.sqrt(3) / 2)
            k = (-(y - ya) - i * s / 2) / s
            if abs(i - round(i)) < 1e-9 and abs(k - round(k)) < 1e-9:
                cols.setdefault(cc, []).append(rr)
    keys = sorted(cols)
    ho = min(len(cols[c]) for c in keys)
    return [(c, sorted(cols[c])[:ho]) for c in keys]


def rand(shape, seed):
    return np.random.default_rng(seed).standard_normal(shape)


# ----------------------------------------------------------------- P1 / P2: tap counts, column heights
def test_p1_tap_counts_closed_form(oracle):
    for n in range(0, 7):
        assert oracle.num_taps(n) == 3 * n * n + 3 * n + 1  # PAPER.md:124-127 (rings)
    assert [oracle.num_taps(n) for n in range(4)] == [1, 7, 19, 37]


def test_p1_column_heights(oracle):
    for n in range(0, 6):
        for p in (0, 1):
            offs = oracle.tap_offsets(n, p)
            for dc in range(-n, n + 1):
                col = [dr for (c, dr) in offs if c == dc]
                assert len(col) == 2 * n + 1 - abs(dc)
                assert col == list(range(col[0], col[0] + len(col)))  # contiguous column


def test_p2_subkernel_heights(oracle):
    # "The illustrated kernel of size 2 consists of three sub-kernels, each
    # representing a set of equal-length columns".
    for g in GOLD["subkernel_heights"]:
        n = g["n"]
        offs = oracle.tap_offsets(n, 0)
        heights = sorted({sum(1 for (c, _) in offs if c == dc) for dc in range(-n, n + 1)}, reverse=True)
        assert heights == g["heights"], g["cite"]


def test_p2_tap_order_is_physical_column_major(oracle):
    # canonical order (A2) = column-major left->right, top->bottom, pinned by
    # sorting the Euclidean disc on physical positions
    for n in range(0, 5):
        for p in (0, 1):
            assert oracle.tap_offsets(n, p) == phys_tap_offsets(n, p)


# ----------------------------------------------------------------- P3 / P4 / P5 / P6: coordinates
def test_p4_spec_coordinate_examples(oracle):
    for g in GOLD["offset_to_axial"]:
        assert oracle.offset_to_axial(*g["offset"]) == tuple(g["axial"]), g["cite"]
        assert oracle.axial_to_offset(*g["axial"]) == tuple(g["offset"]), g["cite"]
    for g in GOLD["pixel_center"]:
        x, y = oracle.pixel_center(*g["offset"])
        assert abs(x - g["xy"][0]) < 1e-12 and abs(y - g["xy"][1]) < 1e-12, g["cite"]
    for g in GOLD["hex_distance_offset"]:
        a = oracle.offset_to_axial(*g["a"])
        b = oracle.offset_to_axial(*g["b"])
        assert oracle.hex_distance(a, b) == g["d"], g["cite"]


def test_p4_round_trip_exhaustive(oracle):
    for pi in (0, 1):
        for r in range(0, 50, 3):
            for c in range(0, 51):
                assert oracle.axial_to_offset(*oracle.offset_to_axial(r, c, pi), pi) == (r, c)


def test_p5_distance_one_iff_unit_pitch(oracle):
    # hex distance 1 <=> Euclidean distance == pitch (10x11 exhaustive)
    for pi in (0, 1):
        cells = [(r, c) for r in range(10) for c in range(11)]
        for a in cells:
            qa = oracle.offset_to_axial(*a, pi)
            xa, ya = phys(*a, pi)
            xo, yo = oracle.pixel_center(*a, pi)
            assert abs(xa - xo) < 1e-12 and abs(ya - yo) < 1e-12
            for b in cells:
                d = oracle.hex_distance(qa, oracle.offset_to_axial(*b, pi))
                xb, yb = phys(*b, pi)
                e = math.hypot(xa - xb, ya - yb)
                assert (d == 1) == (abs(e - 1.0) < 1e-9)


def test_p3_spec_neighbourhoods(oracle):
    m = oracle.gather_map(8, 8, 1, 1, 0)
    for g in GOLD["neighborhood_n1"]:
        r, c = g["centre"]
        cells = {(int(v) // 8, int(v) % 8) for v in m[r, c] if v >= 0}
        assert cells == {tuple(x) for x in g["cells"]}, g["cite"]


def test_p6_brute_force_neighbourhoods(oracle):
    # gather map == Euclidean-disc filter over all cells, in physical column-major order
    for pi in (0, 1):
        for (H, W) in [(5, 6), (7, 4), (6, 9)]:
            for n in (0, 1, 2, 3):
                m = oracle.gather_map(H, W, n, 1, pi)
                for r in range(H):
                    for c in range(W):
                        got = [(int(v) // W, int(v) % W) for v in m[r, c] if v >= 0]
                        assert got == phys_neigh(H, W, r, c, n, pi)


def test_p6_bfs_distance(oracle):
    # hex distance == BFS distance on the physical unit-pitch neighbour graph
    H, W = 7, 8
    cells = [(r, c) for r in range(H) for c in range(W)]
    for pi in (0, 1):
        src = (3, 3)
        dist = {src: 0}
        frontier = [src]
        while frontier:
            nxt = []
            for a in frontier:
                xa, ya = phys(*a, pi)
                for b in cells:
                    if b not in dist:
                        xb, yb = phys(*b, pi)
                        if abs(math.hypot(xa - xb, ya - yb) - 1) < 1e-9:
                            dist[b] = dist[a] + 1
                            nxt.append(b)
            frontier = nxt
        qs = oracle.offset_to_axial(*src, pi)
        for b in cells:
            assert oracle.hex_distance(qs, oracle.offset_to_axial(*b, pi)) == dist[b]


# ----------------------------------------------------------------- P10 / P11 / P12: lattice & shapes
def test_p11_lattice_brute_force(oracle):
    for pi in (0, 1):
        for s in (1, 2, 3, 4):
            for H in range(1, 10):
                for W in range(1, 10):
                    lat = phys_lattice(H, W, s, pi)
                    ho = len(lat[0][1])
                    if ho == 0:
                        with pytest.raises(ValueError):
                            oracle.out_shape(H, W, s, pi)
                        continue
                    Ho, Wo, _ = oracle.out_shape(H, W, s, pi)
                    assert (Ho, Wo) == (ho, len(lat))
                    m = oracle.gather_map(H, W, 0, s, pi)  # n = 0: the centre itself
                    for C, (col, rows) in enumerate(lat):
                        assert col == s * C
                        assert [int(m[R, C, 0]) for R in range(Ho)] == [r * W + col for r in rows]


def test_p11_rho_spec_examples(oracle):
    for g in GOLD["rho"]:
        m = oracle.gather_map(g["H"], g["W"], 0, g["s"], 0)
        rho = [int(m[0, C, 0]) // g["W"] for C in range(m.shape[1])]
        assert rho == g["rho"], g["cite"]


def test_p10_rho_closed_form(oracle):
    # SPEC.md:157 closed form rho(C) = floor((sC+pi)/2) mod s, Ho = min_C floor((H-1-rho)/s)+1
    for pi in (0, 1):
        for s in (1, 2, 3, 4, 5):
            for H in range(2 * s, 14):
                for W in range(1, 14):
                    Ho, Wo, _ = oracle.out_shape(H, W, s, pi)
                    assert Wo == (W - 1) // s + 1
                    rho = [((s * C + pi) // 2) % s for C in range(Wo)]
                    assert Ho == min((H - 1 - r) // s + 1 for r in rho)
                    m = oracle.gather_map(H, W, 0, s, pi)
                    for C in range(Wo):
                        for R in range(Ho):
                            assert int(m[R, C, 0]) == (rho[C] + s * R) * W + s * C


def test_p12_output_shapes(oracle):
    assert oracle.out_shape(5, 5, 2)[:2] == (2, 3)      # omitted step: even columns lose a row
    assert oracle.out_shape(40, 40, 3)[:2] == (13, 14)
    assert oracle.out_shape(48, 48, 2)[:2] == (24, 24)
    assert oracle.out_shape(96, 96, 2)[:2] == (48, 48)
    for H, W in [(1, 1), (5, 7), (16, 16)]:
        assert oracle.out_shape(H, W, 1)[:2] == (H, W)   # stride 1: identity lattice
    # the output of pi=0 is again odd-low (pi_out = 0) for every stride
    for s in range(1, 8):
        assert oracle.out_shape(30, 30, s, 0)[2] == 0
    assert oracle.out_shape(30, 30, 1, 1)[2] == 1
    for s in range(2, 8):
        assert oracle.out_shape(30, 30, s, 1)[2] == 0


def test_p12_output_parity_physical(oracle):
    # output grid of pitch s is itself an offset grid: the centres of output
    # columns 0 and 1 differ in height by exactly s/2, with the sign pi_out says
    for pi in (0, 1):
        for s in range(1, 6):
            H = W = 4 * s + 3
            Ho, Wo, po = oracle.out_shape(H, W, s, pi)
            m = oracle.gather_map(H, W, 0, s, pi)
            r0, c0 = divmod(int(m[0, 0, 0]), W)
            r1, c1 = divmod(int(m[0, 1, 0]), W)
            dy = phys(r1, c1, pi)[1] - phys(r0, c0, pi)[1]
            assert abs(abs(dy) - s / 2) < 1e-12
            assert (dy < 0) == (po == 0)


def test_p10_stride_consistency(oracle):
    for pi in (0, 1):
        for n in (1, 2):
            for s in (2, 3):
                for (H, W) in [(12, 13), (11, 12), (9, 10)]:
                    x = rand((2, 3, H, W), 1)
                    w = rand((2, 3, oracle.num_taps(n)), 2)
                    y1 = oracle.conv2d_fwd(x, w, n=n, s=1, pi=pi)
                    ys = oracle.conv2d_fwd(x, w, n=n, s=s, pi=pi)
                    lat = phys_lattice(H, W, s, pi)
                    for C, (col, rows) in enumerate(lat):
                        for R, r in enumerate(rows):
                            np.testing.assert_allclose(ys[:, :, R, C], y1[:, :, r, col], rtol=0, atol=1e-12)


# ----------------------------------------------------------------- P7 / P9: impulses, n = 0
def test_p7_impulse_spec_example(oracle):
    g = GOLD["impulse_conv"]
    x = np.zeros((1, 1, g["H"], g["W"]))
    x[0, 0, g["impulse"][0], g["impulse"][1]] = 1
    y = oracle.conv2d_fwd(x, np.ones((1, 1, 7)), n=1)
    assert {tuple(v) for v in np.argwhere(y[0, 0] != 0).tolist()} == {tuple(v) for v in g["support"]}
    assert np.all(y[0, 0][y[0, 0] != 0] == 1.0)


def test_p7_impulse_reads_reversed_weights(oracle):
    # conv of an impulse at q with weights w: output at cell o is w[t] where o + off_t = q.
    # Reading the outputs around q in canonical order gives the reversed weight vector.
    for pi in (0, 1):
        for n in (1, 2, 3):
            T = oracle.num_taps(n)
            w = np.arange(1, T + 1, dtype=np.float64)
            for (r, c) in [(8, 8), (8, 9)]:
                x = np.zeros((1, 1, 17, 18))
                x[0, 0, r, c] = 1.0
                y = oracle.conv2d_fwd(x, w[None, None], n=n, pi=pi)[0, 0]
                assert np.count_nonzero(y) == T
                read = [y[rr, cc] for (rr, cc) in phys_neigh(17, 18, r, c, n, pi)]
                assert read == list(w[::-1])


def test_p9_n0_is_channel_matmul(oracle):
    for s in (1, 2, 3):
        x = rand((2, 3, 9, 10), 3)
        w = rand((4, 3, 1), 4)
        b = rand((4,), 5)
        y = oracle.conv2d_fwd(x, w, b, n=0, s=s)
        ref = np.einsum("oi,bihw->bohw", w[:, :, 0], x) + b[None, :, None, None]
        lat = phys_lattice(9, 10, s)
        for C, (col, rows) in enumerate(lat):
            for R, r in enumerate(rows):
                np.testing.assert_allclose(y[:, :, R, C], ref[:, :, r, col], atol=1e-12)


def test_spec_ones_conv(oracle):
    g = GOLD["ones_conv_5x5"]
    y = oracle.conv2d_fwd(np.ones((1, 1, 5, 5)), np.ones((1, 1, 7)), n=1)[0, 0]
    assert y[2, 2] == g["interior"] and y[0, 0] == g["corner_00"], g["cite"]


# ----------------------------------------------------------------- P8: library reduction (torch fp64)
def masked_box_weights(w, n, p):
    """Place canonical taps w[co,ci,T] into a (2n+1)^2 box for centre parity p
    using the physical disc (test-local geometry)."""
    Co, Ci, T = w.shape
    offs = phys_tap_offsets(n, p)
    assert len(offs) == T
    box = torch.zeros(Co, Ci, 2 * n + 1, 2 * n + 1, dtype=torch.float64)
    for t, (dc, dr) in enumerate(offs):
        box[:, :, dr + n, dc + n] = w[:, :, t]
    return box


def torch_hexconv(x, w, b, n, s, pi):
    """Hex conv as two parity-masked square conv2d (fp64) + lattice subsampling."""
    H, W = x.shape[-2:]
    ys = []
    for p in (0, 1):
        ys.append(F.conv2d(x, masked_box_weights(w, n, p), bias=b, padding=n))
    colpar = torch.tensor([(c + pi) % 2 for c in range(W)])
    full = torch.where(colpar.view(1, 1, 1, W) == 0, ys[0], ys[1])
    lat = phys_lattice(H, W, s, pi)
    rows = torch.tensor([r for (_, rs) in lat for r in rs]).view(len(lat), -1).T  # [Ho, Wo]
    cols = torch.tensor([c for (c, _) in lat]).view(1, -1).expand_as(rows)
    return full[:, :, rows, cols]


@pytest.mark.parametrize("pi", [0, 1])
@pytest.mark.parametrize("n", [0, 1, 2, 3])
@pytest.mark.parametrize("s", [1, 2, 3])
def test_p8_conv_equals_masked_square_conv(oracle, n, s, pi):
    for (H, W) in [(12, 13), (7, 8)]:
        if H < 2 * s:
            continue
        xn = rand((2, 3, H, W), 10 + n)
        wn = rand((4, 3, oracle.num_taps(n)), 20 + s)
        bn = rand((4,), 30)
        y = oracle.conv2d_fwd(xn, wn, bn, n=n, s=s, pi=pi)
        x = torch.tensor(xn, requires_grad=True)
        w = torch.tensor(wn, requires_grad=True)
        b = torch.tensor(bn, requires_grad=True)
        yt = torch_hexconv(x, w, b, n, s, pi)
        np.testing.assert_allclose(y, yt.detach().numpy(), rtol=0, atol=1e-12)
        # gradients by autograd through the library formulation
        g = rand(y.shape, 40)
        yt.backward(torch.tensor(g))
        dx, dw, db = oracle.conv2d_bwd(xn, wn, g, n=n, s=s, pi=pi)
        np.testing.assert_allclose(dx, x.grad.numpy(), atol=1e-11)
        np.testing.assert_allclose(dw, w.grad.numpy(), atol=1e-11)
        np.testing.assert_allclose(db, b.grad.numpy(), atol=1e-11)


def torch_hexpool(x, n, s, pi, mode):
    H, W = x.shape[-2:]
    B, C = x.shape[:2]
    outs = []
    for p in (0, 1):
        offs = phys_tap_offsets(n, p)
        mask = torch.zeros((2 * n + 1) ** 2, dtype=torch.bool)
        for (dc, dr) in offs:
            mask[(dr + n) * (2 * n + 1) + (dc + n)] = True
        pad_val = -math.inf if mode == "max" else 0.0
        xp = F.pad(x, (n, n, n, n), value=pad_val)
        u = F.unfold(xp.reshape(B * C, 1, H + 2 * n, W + 2 * n), 2 * n + 1).view(B, C, -1, H, W)
        u = u[:, :, mask]
        if mode == "max":
            outs.append(u.max(dim=2).values)
        elif mode == "avg_pad":  # zero padding counted: divide by the number of taps
            outs.append(u.sum(2) / len(offs))
        else:
            ones = F.pad(torch.ones(1, 1, H, W, dtype=x.dtype), (n, n, n, n))
            cnt = F.unfold(ones, 2 * n + 1).view(1, 1, -1, H, W)[:, :, mask].sum(2)
            outs.append(u.sum(2) / cnt)
    colpar = torch.tensor([(c + pi) % 2 for c in range(W)])
    full = torch.where(colpar.view(1, 1, 1, W) == 0, outs[0], outs[1])
    lat = phys_lattice(H, W, s, pi)
    rows = torch.tensor([r for (_, rs) in lat for r in rs]).view(len(lat), -1).T
    cols = torch.tensor([c for (c, _) in lat]).view(1, -1).expand_as(rows)
    return full[:, :, rows, cols]


@pytest.mark.parametrize("pi", [0, 1])
@pytest.mark.parametrize("mode", ["max", "avg", "avg_pad"])
def test_p8_pool_equals_unfold(oracle, mode, pi):
    for n in (1, 2):
        for s in (1, 2, 3):
            for (H, W) in [(12, 13), (9, 8)]:
                xn = rand((2, 3, H, W), 50 + n + s)
                y, am = oracle.pool2d_fwd(xn, n=n, s=s, pi=pi, mode=mode)
                x = torch.tensor(xn, requires_grad=True)
                yt = torch_hexpool(x, n, s, pi, mode)
                np.testing.assert_allclose(y, yt.detach().numpy(), rtol=0, atol=1e-13)
                g = rand(y.shape, 60)
                yt.backward(torch.tensor(g))  # continuous random input -> no ties
                dx = oracle.pool2d_bwd(g, am, H, W, n=n, s=s, pi=pi, mode=mode)
                np.testing.assert_allclose(dx, x.grad.numpy(), atol=1e-12)


# ----------------------------------------------------------------- P13 / P14: symmetry, conservation
def rot60_map(H, W, centre, pi=0):
    """Physical 60-degree rotation about a centre pixel: dict cell -> rotated cell
    (only cells whose image lies in the grid)."""
    xc, yc = phys(*centre, pi)
    pos = {}
    for r in range(H):
        for c in range(W):
            x, y = phys(r, c, pi)
            pos[(round(x, 6), round(y, 6))] = (r, c)
    ca, sa = math.cos(math.pi / 3), math.sin(math.pi / 3)
    out = {}
    for r in range(H):
        for c in range(W):
            x, y = phys(r, c, pi)
            dx, dy = x - xc, y - yc
            xr, yr = xc + ca * dx - sa * dy, yc + sa * dx + ca * dy
            k = (round(xr, 6), round(yr, 6))
            if k in pos:
                out[(r, c)] = pos[k]
    return out


def test_p13_rotation_equivariance(oracle):
    H, W = 21, 22
    for pi in (0, 1):
        for centre in [(10, 10), (10, 11)]:
            rot = rot60_map(H, W, centre, pi)
            xc, yc = phys(*centre, pi)
            R_in = 5
            rng = np.random.default_rng(7)
            x = np.zeros((1, 1, H, W))
            for (r, c) in rot:
                xx, yy = phys(r, c, pi)
                if math.hypot(xx - xc, yy - yc) <= R_in + 1e-9:
                    x[0, 0, r, c] = rng.standard_normal()
            xr = np.zeros_like(x)
            for a, b in rot.items():
                xr[0, 0, b[0], b[1]] = x[0, 0, a[0], a[1]]
            for n in (1, 2):
                T = oracle.num_taps(n)
                w = rng.standard_normal((1, 1, T))
                # rotate the kernel: tap t at physical offset v moves to rot(v)
                offs0 = phys_tap_offsets(n, 0)
                cen = (2 * n + 2, 2 * n + 2)
                rk = rot60_map(4 * n + 6, 4 * n + 6, cen, 0)
                idx = {o: t for t, o in enumerate(offs0)}
                wr = np.zeros_like(w)
                for t, (dc, dr) in enumerate(offs0):
                    a = (cen[0] + dr, cen[1] + dc)
                    b = rk[a]
                    wr[0, 0, idx[(b[1] - cen[1], b[0] - cen[0])]] = w[0, 0, t]
                y = oracle.conv2d_fwd(x, w, n=n, pi=pi)
                yr = oracle.conv2d_fwd(xr, wr, n=n, pi=pi)
                for a, b in rot.items():
                    xx, yy = phys(*a, pi)
                    if math.hypot(xx - xc, yy - yc) <= R_in + n + 1e-9:
                        assert abs(yr[0, 0, b[0], b[1]] - y[0, 0, a[0], a[1]]) < 1e-12


def test_p13_debug_kernel_keeps_symmetry(oracle):
    # PAPER.md:220-224, Fig.5: 6-fold symmetric shapes convolved with the
    # all-ones (debug) kernel keep their symmetry
    H, W = 21, 22
    centre = (10, 10)
    rot = rot60_map(H, W, centre)
    xc, yc = phys(*centre)
    x = np.zeros((1, 1, H, W))
    for (r, c) in rot:
        xx, yy = phys(r, c)
        d = math.hypot(xx - xc, yy - yc)
        if d <= 4 + 1e-9:
            x[0, 0, r, c] = math.cos(d)  # rotation-invariant function of the distance
    for n in (1, 2):
        y = oracle.conv2d_fwd(x, np.ones((1, 1, oracle.num_taps(n))), n=n)
        for a, b in rot.items():
            xx, yy = phys(*a)
            if math.hypot(xx - xc, yy - yc) <= 4 + n + 1e-9:
                assert abs(y[0, 0, a[0], a[1]] - y[0, 0, b[0], b[1]]) < 1e-12


def test_p14_conservation(oracle):
    for pi in (0, 1):
        for n in (1, 2):
            for (H, W) in [(7, 9), (10, 6)]:
                x = rand((1, 1, H, W), 70)
                y = oracle.conv2d_fwd(x, np.ones((1, 1, oracle.num_taps(n))), n=n, pi=pi)
                counts = np.array([[len(phys_neigh(H, W, r, c, n, pi)) for c in range(W)] for r in range(H)])
                assert abs(y.sum() - (x[0, 0] * counts).sum()) < 1e-10


# ----------------------------------------------------------------- P15 / P16: linearity, adjoint, FD
def test_p15_linearity_and_adjoint(oracle):
    for pi in (0, 1):
        for n, s in [(1, 1), (2, 2), (1, 3), (3, 1)]:
            H, W = 11, 12
            x1, x2 = rand((2, 3, H, W), 80), rand((2, 3, H, W), 81)
            w = rand((4, 3, oracle.num_taps(n)), 82)
            a, b = 0.7, -1.3
            y = oracle.conv2d_fwd(a * x1 + b * x2, w, n=n, s=s, pi=pi)
            yl = a * oracle.conv2d_fwd(x1, w, n=n, s=s, pi=pi) + b * oracle.conv2d_fwd(x2, w, n=n, s=s, pi=pi)
            np.testing.assert_allclose(y, yl, atol=1e-12)
            g = rand(y.shape, 83)
            dx, dw, _ = oracle.conv2d_bwd(x1, w, g, n=n, s=s, pi=pi)
            y1 = oracle.conv2d_fwd(x1, w, n=n, s=s, pi=pi)
            assert abs((y1 * g).sum() - (x1 * dx).sum()) < 1e-10
            assert abs((y1 * g).sum() - (w * dw).sum()) < 1e-10


def test_p16_finite_differences(oracle):
    rng = np.random.default_rng(90)
    for pi in (0, 1):
        for n, s in [(1, 1), (2, 2), (1, 2)]:
            H, W = 6, 7
            x = rng.standard_normal((1, 2, H, W))
            w = rng.standard_normal((2, 2, oracle.num_taps(n)))
            bb = rng.standard_normal((2,))
            y = oracle.conv2d_fwd(x, w, bb, n=n, s=s, pi=pi)
            g = rng.standard_normal(y.shape)
            dx, dw, db = oracle.conv2d_bwd(x, w, g, n=n, s=s, pi=pi)
            L = lambda xx, ww, bv: (oracle.conv2d_fwd(xx, ww, bv, n=n, s=s, pi=pi) * g).sum()
            h = 1e-6
            for _ in range(12):
                i = tuple(rng.integers(0, d) for d in x.shape)
                xp, xm = x.copy(), x.copy()
                xp[i] += h
                xm[i] -= h
                fd = (L(xp, w, bb) - L(xm, w, bb)) / (2 * h)
                assert abs(fd - dx[i]) <= 1e-5 * max(1.0, abs(fd))
                j = tuple(rng.integers(0, d) for d in w.shape)
                wp, wm = w.copy(), w.copy()
                wp[j] += h
                wm[j] -= h
                fd = (L(x, wp, bb) - L(x, wm, bb)) / (2 * h)
                assert abs(fd - dw[j]) <= 1e-5 * max(1.0, abs(fd))
            fd = (L(x, w, bb + np.array([h, 0])) - L(x, w, bb - np.array([h, 0]))) / (2 * h)
            assert abs(fd - db[0]) <= 1e-5 * max(1.0, abs(fd))


# ----------------------------------------------------------------- P17: pools
def test_p17_pool_pins(oracle):
    # constant -> constant (avg)
    for n, s in [(1, 1), (2, 2), (1, 3)]:
        y, _ = oracle.pool2d_fwd(np.full((1, 2, 9, 10), 3.25), n=n, s=s, mode="avg")
        assert np.all(y == 3.25)
    # impulse -> footprint (max)
    x = np.zeros((1, 1, 6, 6))
    x[0, 0, 2, 2] = 1.0
    y, _ = oracle.pool2d_fwd(x, n=1, s=1, mode="max")
    assert {tuple(v) for v in np.argwhere(y[0, 0] == 1).tolist()} == \
        {tuple(v) for v in GOLD["impulse_conv"]["support"]}
    # corrected corner ramp (A11): 1/3 under pi = 0
    ramp = np.tile(np.arange(5.0)[:, None], (1, 5))[None, None]
    y, _ = oracle.pool2d_fwd(ramp, n=1, s=1, mode="avg")
    assert abs(y[0, 0, 0, 0] - GOLD["ramp_avg_corner"]["value"]) < 1e-15
    # max >= avg on non-negative input
    xn = np.abs(rand((2, 3, 11, 12), 100))
    for s in (1, 2):
        ymax, _ = oracle.pool2d_fwd(xn, n=1, s=s, mode="max")
        yavg, _ = oracle.pool2d_fwd(xn, n=1, s=s, mode="avg")
        assert np.all(ymax >= yavg)
    # ties -> first in-grid tap in canonical order (A9)
    y, am = oracle.pool2d_fwd(np.zeros((1, 1, 5, 6)), n=1, s=1, mode="max")
    m = oracle.gather_map(5, 6, 1, 1)
    first = np.argmax(m >= 0, axis=-1)
    assert np.array_equal(am[0, 0], first)
    # max pool with monotone ramp picks the lowest in-grid row
    y, am = oracle.pool2d_fwd(ramp, n=1, s=1, mode="max")
    for r in range(5):
        for c in range(5):
            assert y[0, 0, r, c] == max(rr for (rr, cc) in phys_neigh(5, 5, r, c, 1))


def test_p17_include_pad_avg(oracle):
    # include-pad average (f4): all-ones input gives in-grid count / T(n) -- the in-grid count of
    # every window read off the gather map, T(n) the closed form 3n(n+1)+1 (P1); interior = 1
    for n, s, pi in [(1, 1, 0), (2, 1, 1), (1, 2, 0), (2, 3, 1)]:
        y, _ = oracle.pool2d_fwd(np.ones((1, 1, 9, 10)), n=n, s=s, pi=pi, mode="avg_pad")
        m = oracle.gather_map(9, 10, n, s, pi)
        T = 3 * n * (n + 1) + 1
        np.testing.assert_allclose(y[0, 0], (m >= 0).sum(-1) / T, rtol=0, atol=1e-15)
        assert y.max() == 1.0
    # = in-grid average x in-grid count / T on random data
    xn = rand((2, 3, 11, 12), 120)
    for n, s in [(1, 1), (2, 2)]:
        ya, _ = oracle.pool2d_fwd(xn, n=n, s=s, mode="avg")
        yp, _ = oracle.pool2d_fwd(xn, n=n, s=s, mode="avg_pad")
        cnt = (oracle.gather_map(11, 12, n, s) >= 0).sum(-1)
        np.testing.assert_allclose(yp, ya * cnt / (3 * n * (n + 1) + 1), rtol=1e-14, atol=1e-15)


def test_p17_pool_bwd_fd(oracle):
    rng = np.random.default_rng(110)
    for mode in ("max", "avg", "avg_pad"):
        for n, s in [(1, 1), (1, 2), (2, 2)]:
            x = rng.standard_normal((1, 2, 7, 8))
            y, am = oracle.pool2d_fwd(x, n=n, s=s, mode=mode)
            g = rng.standard_normal(y.shape)
            dx = oracle.pool2d_bwd(g, am, 7, 8, n=n, s=s, mode=mode)
            L = lambda xx: (oracle.pool2d_fwd(xx, n=n, s=s, mode=mode)[0] * g).sum()
            h = 1e-7
            for _ in range(15):
                i = tuple(rng.integers(0, d) for d in x.shape)
                xp, xm = x.copy(), x.copy()
                xp[i] += h
                xm[i] -= h
                fd = (L(xp) - L(xm)) / (2 * h)
                assert abs(fd - dx[i]) <= 1e-5 * max(1.0, abs(fd))


# ----------------------------------------------------------------- P18: stride-1 dgrad = reversed-tap fwd
def test_p18_dgrad_is_reversed_transposed_fwd(oracle):
    for pi in (0, 1):
        for n in (1, 2, 3):
            x = rand((2, 3, 9, 10), 120)
            w = rand((4, 3, oracle.num_taps(n)), 121)
            g = rand((2, 4, 9, 10), 122)
            dx, _, _ = oracle.conv2d_bwd(x, w, g, n=n, s=1, pi=pi)
            wt = np.ascontiguousarray(np.transpose(w, (1, 0, 2))[:, :, ::-1])
            np.testing.assert_allclose(dx, oracle.conv2d_fwd(g, wt, n=n, s=1, pi=pi), atol=1e-12)


def test_errors(oracle):
    with pytest.raises(ValueError):
        oracle.out_shape(1, 5, 2)          # A7: odd columns have no lattice row -> empty
    with pytest.raises(ValueError):
        oracle.conv2d_fwd(np.zeros((1, 2, 4, 4)), np.zeros((1, 3, 7)), n=1)  # channel mismatch
    with pytest.raises(ValueError):
        oracle.pool2d_fwd(np.zeros((1, 1, 4, 4)), n=0)


def test_wgrad_point_evaluation_matches_dense(oracle):
    # the point-evaluation entry used for full-size checks equals the dense adjoint
    for layout in ("NCHW", "NHWC"):
        for n, s, pi in [(1, 1, 0), (2, 2, 1), (3, 1, 1)]:
            x = rand((2, 3, 9, 10), 130).astype(np.float32)
            w = rand((4, 3, oracle.num_taps(n)), 131)
            Ho, Wo, _ = oracle.out_shape(9, 10, s, pi)
            g = rand((2, 4, Ho, Wo), 132).astype(np.float32)
            _, dw, _ = oracle.conv2d_bwd(x, w, g, n=n, s=s, pi=pi)
            pts = [(co, ci, t) for co in range(4) for ci in range(3) for t in range(oracle.num_taps(n))]
            xx, gg = (x, g) if layout == "NCHW" else (x.transpose(0, 2, 3, 1).copy(), g.transpose(0, 2, 3, 1).copy())
            got = oracle.conv2d_bwd_weight_at(xx, gg, pts, n=n, s=s, pi=pi, layout=layout)
            np.testing.assert_allclose(got, [dw[p] for p in pts], atol=1e-10)
            # bf16 storage: the bit patterns of bf16-representable values convert exactly
            xb = (xx.view(np.uint32) >> 16).astype(np.uint16)
            x_trunc = (xb.astype(np.uint32) << 16).view(np.float32)
            got_b = oracle.conv2d_bwd_weight_at(xb, gg, pts, n=n, s=s, pi=pi, layout=layout)
            ref_b = oracle.conv2d_bwd_weight_at(x_trunc, gg, pts, n=n, s=s, pi=pi, layout=layout)
            np.testing.assert_allclose(got_b, ref_b, atol=1e-12)


def test_pool_bwd_rejects_invalid_argmax(oracle):
    # the max-pool backward routes dy through an argmax produced by the code under test: an index
    # >= T, or one naming an off-grid neighbour, must fail the check rather than write out of bounds
    H, W, n, s = 6, 7, 1, 2
    Ho, Wo, _ = oracle.out_shape(H, W, s)
    dy = np.ones((1, 1, Ho, Wo))
    ok = np.zeros((1, 1, Ho, Wo), dtype=np.uint8) + 3          # tap 3 = the centre (always in-grid)
    oracle.pool2d_bwd(dy, ok, H, W, n=n, s=s)
    with pytest.raises(ValueError):
        oracle.pool2d_bwd(dy, ok + 4, H, W, n=n, s=s)            # tap index 7 >= T(1)
    m = oracle.gather_map(H, W, n, s)
    t_off = int(np.nonzero(m[0, 0] < 0)[0][0])                  # a corner tap outside the grid
    bad = ok.copy()
    bad[0, 0, 0, 0] = t_off
    with pytest.raises(ValueError):
        oracle.pool2d_bwd(dy, bad, H, W, n=n, s=s)
    with pytest.raises(ValueError):
        oracle.pool2d_bwd(dy, None, H, W, n=n, s=s)
    with pytest.raises(ValueError):
        oracle.pool2d_bwd(dy[..., :-1], ok[..., :-1], H, W, n=n, s=s)   # dy not on the lattice
