"""CPU-only checks of the C-ABI library: it loads, exports every symbol that
include/hexconv.h declares, and its host-side geometry (tap tables, output
shapes, argument validation) agrees bit-exactly with the oracle.  No kernel is
launched here."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def abi():
    from paper_1903_01814_b200 import build
    build.build()
    from paper_1903_01814_b200 import _abi
    return _abi


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hexconv.h")).read()
    return sorted(set(re.findall(r"^HEX_API\s+[\w\s\*]+?\b(hex_\w+)\s*\(", src, flags=re.M)))


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ["hex_conv2d_fwd", "hex_conv2d_bwd_data", "hex_conv2d_bwd_weight", "hex_pool2d_fwd",
              "hex_pool2d_bwd", "hex_output_shape", "hex_num_taps", "hex_tap_offsets",
              "hex_conv2d_gather_map", "hex_conv2d_workspace_size", "hex_status_string"]:
        assert s in syms


def test_library_exports_every_declared_symbol(abi):
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\sT\s(hex_\w+)", out))
    for s in declared_symbols():
        assert s in exported, s
        assert hasattr(abi.lib(), s)
    assert set(abi.EXPORTED) == set(declared_symbols())


def test_library_is_sm100a(abi):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_num_taps(abi, oracle):
    for n in range(0, 8):
        assert abi.num_taps(n) == oracle.num_taps(n)
    assert abi.num_taps(-1) == -1


def test_tap_offsets_bit_exact(abi, oracle):
    for n in range(0, abi.MAX_N + 1):
        for p in (0, 1):
            assert abi.tap_offsets(n, p) == oracle.tap_offsets(n, p)


def test_tap_axial_bit_exact(abi, oracle):
    # custom-kernel element order (reading A2): the library's axial tap list is the oracle's
    for n in range(0, abi.MAX_N + 1):
        assert abi.tap_axial(n) == oracle.tap_list(n)
    with pytest.raises(abi.HexError):
        abi.tap_axial(-1)


def test_switch_hook_rejects_unknown_names(abi):
    L = abi.lib()
    assert L.hex_debug_set_switch(b"HEXCONV_NOT_A_SWITCH", b"1") == 1  # HEX_ERR_INVALID_ARG
    assert L.hex_debug_set_switch(None, None) == 1
    with abi.switch("HEXCONV_NO_TF32"):
        pass  # set and restored without touching a GPU


def test_output_shape_bit_exact(abi, oracle):
    for pi in (0, 1):
        for s in range(1, 7):
            for H in range(1, 15):
                for W in range(1, 15):
                    try:
                        ref = oracle.out_shape(H, W, s, pi)
                    except ValueError:
                        with pytest.raises(abi.HexError) as e:
                            abi.output_shape(H, W, s, pi)
                        assert e.value.status == 3  # HEX_ERR_EMPTY_LATTICE
                        continue
                    assert abi.output_shape(H, W, s, pi) == ref


def test_validation_without_launch(abi):
    L = abi.lib()
    d = abi.ConvDesc(1, 1, 1, 8, 8, -1, 1, 0, abi.F32, abi.NCHW)
    dummy = ctypes.c_void_p(16)
    assert L.hex_conv2d_fwd(ctypes.byref(d), dummy, dummy, None, 0, dummy, None, 0, None) == 1
    d = abi.ConvDesc(1, 1, 1, 8, 8, 1, 0, 0, abi.F32, abi.NCHW)
    assert L.hex_conv2d_fwd(ctypes.byref(d), dummy, dummy, None, 0, dummy, None, 0, None) == 1
    d = abi.ConvDesc(1, 1, 1, 1, 5, 1, 2, 0, abi.F32, abi.NCHW)   # A7: empty lattice
    assert L.hex_conv2d_fwd(ctypes.byref(d), dummy, dummy, None, 0, dummy, None, 0, None) == 3
    d = abi.ConvDesc(1, 1, 1, 8, 8, 8, 1, 0, abi.F32, abi.NCHW)   # n > HEX_MAX_N
    assert L.hex_conv2d_fwd(ctypes.byref(d), dummy, dummy, None, 0, dummy, None, 0, None) == 8
    d = abi.ConvDesc(1, 1, 1, 8, 8, 1, 1, 0, 7, abi.NCHW)          # bad dtype
    assert L.hex_conv2d_fwd(ctypes.byref(d), dummy, dummy, None, 0, dummy, None, 0, None) == 4
    d = abi.ConvDesc(1, 1, 1, 8, 8, 1, 1, 0, abi.F32, 5)           # bad layout
    assert L.hex_conv2d_fwd(ctypes.byref(d), dummy, dummy, None, 0, dummy, None, 0, None) == 5
    d = abi.ConvDesc(1, 1, 1, 8, 8, 1, 1, 0, abi.F32, abi.NCHW)
    assert L.hex_conv2d_fwd(ctypes.byref(d), None, dummy, None, 0, dummy, None, 0, None) == 1
    d = abi.ConvDesc(0, 1, 1, 8, 8, 1, 1, 0, abi.F32, abi.NCHW)    # empty batch
    assert L.hex_conv2d_fwd(ctypes.byref(d), dummy, dummy, None, 0, dummy, None, 0, None) == 2
    p = abi.PoolDesc(1, 1, 8, 8, 0, 1, 0, abi.F32, abi.NCHW, abi.POOL_MAX)  # pool n = 0
    assert L.hex_pool2d_fwd(ctypes.byref(p), dummy, dummy, None, None) == 1
    p = abi.PoolDesc(1, 1, 8, 8, 1, 1, 0, abi.F32, abi.NCHW, abi.POOL_MAX)  # max bwd needs argmax
    assert L.hex_pool2d_bwd(ctypes.byref(p), dummy, None, dummy, None) == 1
    sz = ctypes.c_size_t()
    d = abi.ConvDesc(2, 3, 4, 9, 9, 1, 1, 0, abi.F32, abi.NCHW)
    assert L.hex_conv2d_workspace_size(ctypes.byref(d), 2, ctypes.byref(sz)) == 0 and sz.value > 0
    assert L.hex_conv2d_workspace_size(ctypes.byref(d), 7, ctypes.byref(sz)) == 1
    assert L.hex_status_string(3) == b"empty lattice"


def test_product_never_imports_oracle():
    # the oracle is test infrastructure: the product package must not reference it
    pkg = os.path.join(ROOT, "paper_1903_01814_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                for pat in ("import oracle", "from oracle", "liboracle", '#include "../../oracle', "oracle/hexoracle.h"):
                    assert pat not in txt, (f, pat)


def test_custom_kernel_taps_canonical(oracle):
    # tap_axial (the custom-kernel helper's tap order) is the oracle's canonical tap list (A2, P1)
    from paper_1903_01814_b200 import functional as F
    for n in range(0, 5):
        assert F.tap_axial(n) == [tuple(t) for t in oracle.tap_list(n)]
    k = F.ring_kernel([1.0, 0.5, 0.25], device="cpu")
    assert k.shape == (1, 1, 19)
    taps = F.tap_axial(2)
    for t, (a, b) in enumerate(taps):
        assert k[0, 0, t].item() == [1.0, 0.5, 0.25][(abs(a) + abs(b) + abs(a + b)) // 2]
    d = F.custom_kernel(1, {(0, 0): 2.0, (1, -1): -1.0}, 2, 3, device="cpu")
    assert d.shape == (2, 3, 7) and d.sum().item() == 6.0


def test_bench_launches_n_ranks():
    # `python bench.py --gpus 2` without a launcher starts two ranks itself (torchrun on 127.0.0.1)
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--launch-check"],
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert sorted(d["rank"] for d in lines) == [0, 1]
    assert all(d["world"] == 2 for d in lines)


def test_bench_reference_arm_line():
    # the reference arm (`bench.py --impl reference`: the fp64 oracle on the host cores, a bounded sample of the
    # config-5 step) prints one JSON line with the contract's keys
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "3"], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["impl"] == "reference" and d["n_gpus"] == 1 and d["steps"] == 1 and d["warmup"] == 3
    for k in ("metric", "value", "unit", "ms_per_step", "higher_is_better", "scaling", "vs_baseline", "dtype",
              "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["value"] > 0 and d["unit"] == "images/s" and d["dtype"] == "f64"
    assert d["e2e"]["value"] == d["value"] and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert "workload" in d["config"]
