"""CPU-side checks of the C ABI: the library loads without a GPU, exports every
symbol include/spconv.h declares, and its host-only entry points validate
geometry exactly as the header documents (no kernel launches here)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2104_08314_b200 import build
    build.build()
    import paper_2104_08314_b200 as p
    return p


def header_functions():
    txt = open(os.path.join(ROOT, "include", "spconv.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b([a-z_0-9]+)\s*\(", txt)) - {"defined", "sizeof"})


def test_header_symbols_exported(lib):
    names = header_functions()
    assert "cpo_encode" in names and "select_layer_algo" in names and len(names) >= 12
    so = ctypes.CDLL(lib.LIB_PATH)
    for n in names:
        assert hasattr(so, n), n
    assert set(lib.EXPORTED) <= set(names)


def test_so_has_sm100a_code(lib):
    import subprocess
    out = subprocess.run(["cuobjdump", "--list-elf", lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def _d(**kw):
    d = dict(N=1, C=4, H=8, W=8, K=4, R=3, S=3, stride_h=1, stride_w=1,
             pad_top=1, pad_bottom=1, pad_left=1, pad_right=1)
    d.update(kw)
    return d


def test_capacity_matches_header_formula(lib):
    d = _d(N=2, C=5, H=14, W=14)
    pc, dc, ic, ws = lib.spc_encode_capacity(d)
    Ow1 = 16 - 3 + 1
    assert pc == 10 * (3 + 2 * (1 + Ow1))
    assert dc == ic == 2 * 5 * 14 * 14
    assert ws > 4 * dc
    d1 = _d(R=7, S=1, pad_left=0, pad_right=0, pad_top=3, pad_bottom=3)
    assert lib.spc_encode_capacity(d1)[0] == 4 * (1 + 8)


@pytest.mark.parametrize("kw,status", [
    (dict(R=1, S=1, pad_top=0, pad_bottom=0, pad_left=0, pad_right=0), -2),   # pointwise
    (dict(pad_left=1, pad_right=2), -2),                                     # asymmetric W pad (A16)
    (dict(pad_left=3, pad_right=3), -2),                                     # pad >= K_w
    (dict(W=2, pad_left=0, pad_right=0, S=2), -2),                           # Wp < 2S-1 (A17)
    (dict(H=0), -1),
    (dict(stride_h=0), -1),
])
def test_capacity_rejects(lib, kw, status):
    with pytest.raises(lib.SpcError) as e:
        lib.spc_encode_capacity(_d(**kw))
    assert e.value.status == status


def test_binding_refuses_cpu_tensors(lib):
    import torch
    d = _d()
    with pytest.raises(ValueError):
        lib.binding._ptr(torch.zeros(4))


def test_im2col_engine_resolution(lib):
    """SPC_GEMM_AUTO (the default) picks the tcgen05 3xTF32 kernel for layers of >= 2^28 MACs,
    or >= 2^26 MACs over >= 20 output tiles or with C*R*S >= 2048, whose C*R*S is a multiple of 4 (TMA row
    pitches), cuBLAS FP32 otherwise; an explicit
    TC_3XTF32 falls back to cuBLAS FP32 when C*R*S % 4 != 0 (include/spconv.h)."""
    prev = lib.spc_get_im2col_gemm()
    try:
        lib.spc_set_im2col_gemm(lib.SPC_GEMM_AUTO)
        big = _d(N=32, C=64, H=56, W=56, K=64)            # 3.7e9 MACs, CRS = 576
        mid = _d(N=1, C=64, H=56, W=56, K=64)             # cfg2: 1.2e8 MACs, 25 tiles
        few = _d(N=8, C=384, H=8, W=8, K=384, R=1, S=3, pad_top=0, pad_bottom=0)   # 2.3e8 MACs, 12 tiles
        small = _d(N=1, C=16, H=14, W=14, K=16)           # cfg1: 4.5e5 MACs
        deep = _d(N=8, C=256, H=14, W=14, K=256, stride_h=2, stride_w=2)   # cfg3 s2: 8 tiles, CRS 2304
        assert lib.spc_im2col_engine(deep) == lib.SPC_GEMM_TC_3XTF32
        odd = _d(N=32, C=65, H=56, W=56, K=64)            # CRS = 585
        assert lib.spc_im2col_engine(big) == lib.SPC_GEMM_TC_3XTF32
        assert lib.spc_im2col_engine(mid) == lib.SPC_GEMM_TC_3XTF32
        assert lib.spc_im2col_engine(few) == lib.SPC_GEMM_CUBLAS_FP32
        assert lib.spc_im2col_engine(small) == lib.SPC_GEMM_CUBLAS_FP32
        assert lib.spc_im2col_engine(odd) == lib.SPC_GEMM_CUBLAS_FP32
        lib.spc_set_im2col_gemm(lib.SPC_GEMM_TC_3XTF32)
        assert lib.spc_im2col_engine(small) == lib.SPC_GEMM_TC_3XTF32
        assert lib.spc_im2col_engine(odd) == lib.SPC_GEMM_CUBLAS_FP32
        lib.spc_set_im2col_gemm(lib.SPC_GEMM_SIMT)
        assert lib.spc_im2col_engine(big) == lib.SPC_GEMM_SIMT
        with pytest.raises(lib.SpcError):
            lib.spc_set_im2col_gemm(6)
    finally:
        lib.spc_set_im2col_gemm(prev)


def test_cps_inline_toggle(lib):
    """spc_set_cps_inline: 0 / 1 accepted and read back, anything else SPC_EINVAL (host only)."""
    prev = lib.spc_get_cps_inline()
    try:
        for on in (True, False):
            lib.spc_set_cps_inline(on)
            assert lib.spc_get_cps_inline() is on
        raw = ctypes.CDLL(lib.LIB_PATH)
        raw.spc_set_cps_inline.argtypes = [ctypes.c_int32]
        assert raw.spc_set_cps_inline(2) == lib.SPC_EINVAL
        assert lib.spc_get_cps_inline() is False
    finally:
        lib.spc_set_cps_inline(prev)
