"""CPU oracle for arXiv 2104.08314 (CPO / CPS sparse-activation convolution).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` leg may import this package.  It shares no
code with the CUDA path (paper_2104_08314_b200/) and never imports it.

The arithmetic lives in ``oracle.c`` (plain single-threaded C, FP64
accumulation), which follows the paper step by step:

  direct_conv        Eq. 1
  im2col / gemm      im2col lowering + naive GEMM           PAPER.md:76, SI Eq. 6 (:592-595)
  mec_lower          MEC lowering                           PAPER.md:78, SI Eq. 11 (:618-622)
  encode(cps=0)      CPO encoding, Alg. 1 (+ SI Alg. 5)
  encode(cps=1)      CPS encoding, Alg. 3
  decode             inverse of the encoding (independent)
  sparse_conv        Alg. 2 / Alg. 4 / SI Alg. 6
  set4_census        C'_k, C''_k of SI Eq. 5
  mac_count          exact multiply-adds of the sparse conv reading A27
  cscc_encode        CSCC (SI Alg. 5 for any K_w, s_w)
  cscc_conv          CSCC conv (SI Alg. 6 + stride)
  cscc_decode        inverse of the CSCC streams            (test of the encoder)
  encode_sa          stride-aware CPO layout (reading A32)  SI Eq. 2
  decode_sa / sparse_conv_sa  its inverse and Alg. 2 over it

Sizes (SI Eqs. 2-6, 11) are written out in ``sizes.py``.

Pins (tests/test_oracle_*.py, all "-m 'not gpu'"): Fig. 1 streams from the
paper's prose (tests/golden/fig1.json); SI Eq. 3/4/5 lengths exactly;
decode(encode(x)) == x; direct == numpy im2col @ matmul == torch conv2d (fp64);
sparse oracle conv == direct conv bit-exactly on integer data over a random
sweep; im2col / MEC materialised sizes == Eq. 6 / Eq. 11 and the worked
numbers 400 / 160.  Parity unpinned: the numeric value of the ptr tag (A1)
and the presence of an empty NOP block (A2) are conventions.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from .sizes import (S_im2col, S_mec, ptr_size_eq3, in_cps_size_eq5, op_size_eq2,  # noqa: F401
                    nop_size, da_size_eq4, S_cscc_eq17, rho_hat, p_bound_cscc, q_bound_cscc)

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

NPC = -(2 ** 31)
NPF = -(2 ** 31) + 1


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with plain gcc (no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-Wall", "-shared", "-fPIC",
                               "-o", _LIB + ".tmp", _SRC])
        os.replace(_LIB + ".tmp", _LIB)
    return _LIB


class _Desc(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in
                ("N", "C", "H", "W", "K", "R", "S", "sh", "sw", "pt", "pb", "pl", "pr")]


_lib = None


def _L():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        i64, i32, vp = ctypes.c_int64, ctypes.c_int32, ctypes.c_void_p
        P = ctypes.POINTER(_Desc)
        sig = {
            "oc_out_h": (i32, [P]), "oc_out_w": (i32, [P]),
            "oc_direct_conv": (None, [P, vp, vp, vp]),
            "oc_direct_conv_at": (None, [P, vp, vp, vp, i64, vp]),
            "oc_im2col": (i64, [P, vp, vp]),
            "oc_gemm_lowered": (None, [P, vp, vp, vp]),
            "oc_mec_lower": (i64, [P, vp, vp]),
            "oc_encode": (ctypes.c_int, [P, vp, ctypes.c_int, vp, i64, vp, i64, vp, i64, vp, vp]),
            "oc_decode": (ctypes.c_int, [P, ctypes.c_int, vp, i64, vp, i64, vp, i64, vp]),
            "oc_sparse_conv": (ctypes.c_int, [P, ctypes.c_int, vp, i64, vp, vp, vp, vp]),
            "oc_mac_count": (i64, [P, vp]),
            "oc_set4_census": (None, [P, vp, vp]),
            "oc_count_flags": (None, [vp, i64, vp, vp]),
            "oc_pattern_size": (i32, [i32]), "oc_next_offset": (i32, [i32, i32]),
            "oc_cscc_encode": (ctypes.c_int, [P, vp, vp, i64, vp, i64, vp, i64, vp, vp]),
            "oc_cscc_conv": (ctypes.c_int, [P, vp, i64, vp, i64, vp, vp, vp]),
            "oc_cscc_decode": (ctypes.c_int, [P, vp, i64, vp, i64, vp, vp]),
            "oc_encode_sa": (ctypes.c_int, [P, vp, vp, i64, vp, i64, vp, i64, vp, vp]),
            "oc_decode_sa": (ctypes.c_int, [P, vp, i64, vp, i64, vp, vp]),
            "oc_sparse_conv_sa": (ctypes.c_int, [P, vp, i64, vp, i64, vp, vp, vp]),
        }
        for name, (res, args) in sig.items():
            f = getattr(_lib, name)
            f.restype, f.argtypes = res, args
    return _lib


def _desc(d: dict) -> _Desc:
    return _Desc(d["N"], d["C"], d["H"], d["W"], d["K"], d["R"], d["S"], d["stride_h"],
                 d["stride_w"], d["pad_top"], d["pad_bottom"], d["pad_left"], d["pad_right"])


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def out_hw(d: dict) -> tuple[int, int]:
    """(Oh, Ow) = floor((I + pads - K) / s) + 1 (reading A14)."""
    dd = _desc(d)
    return _L().oc_out_h(ctypes.byref(dd)), _L().oc_out_w(ctypes.byref(dd))


def direct_conv(d: dict, x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Eq. 1 in FP64 -> float64 [N, K, Oh, Ow]."""
    Oh, Ow = out_hw(d)
    x, w = _f32(x), _f32(w)
    y = np.empty((d["N"], d["K"], Oh, Ow), dtype=np.float64)
    _L().oc_direct_conv(ctypes.byref(_desc(d)), _p(x), _p(w), _p(y))
    return y


def direct_conv_at(d: dict, x: np.ndarray, w: np.ndarray, idx: np.ndarray) -> np.ndarray:
    """Eq. 1 at output coordinates idx[i] = (n, k, y, x), FP64."""
    idx = np.ascontiguousarray(idx, dtype=np.int32).reshape(-1, 4)
    x, w = _f32(x), _f32(w)
    out = np.empty(idx.shape[0], dtype=np.float64)
    _L().oc_direct_conv_at(ctypes.byref(_desc(d)), _p(x), _p(w), _p(idx), idx.shape[0], _p(out))
    return out


def im2col(d: dict, x: np.ndarray) -> np.ndarray:
    """im2col lowered matrix [N, Oh*Ow, C*R*S]."""
    Oh, Ow = out_hw(d)
    x = _f32(x)
    L = np.empty((d["N"], Oh * Ow, d["C"] * d["R"] * d["S"]), dtype=np.float32)
    n = _L().oc_im2col(ctypes.byref(_desc(d)), _p(x), _p(L))
    assert n == L.size
    return L


def gemm_lowered(d: dict, L: np.ndarray, w: np.ndarray) -> np.ndarray:
    Oh, Ow = out_hw(d)
    L, w = _f32(L), _f32(w)
    y = np.empty((d["N"], d["K"], Oh, Ow), dtype=np.float64)
    _L().oc_gemm_lowered(ctypes.byref(_desc(d)), _p(L), _p(w), _p(y))
    return y


def mec_lower(d: dict, x: np.ndarray) -> np.ndarray:
    """MEC lowered matrices [N, C, Ow, Hp*S]."""
    _, Ow = out_hw(d)
    Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    x = _f32(x)
    M = np.empty((d["N"], d["C"], Ow, Hp * d["S"]), dtype=np.float32)
    n = _L().oc_mec_lower(ctypes.byref(_desc(d)), _p(x), _p(M))
    assert n == M.size
    return M


class Encoding(dict):
    """ptr / da / in streams plus the per-channel offset side tables."""


def encode(d: dict, x: np.ndarray, cps: bool = False) -> Encoding:
    """CPO (Alg. 1) or CPS (Alg. 3) encoding of the whole tensor, channels
    concatenated n-major then c (reading A19)."""
    x = _f32(x)
    NC = d["N"] * d["C"]
    Wp = d["W"] + d["pad_left"] + d["pad_right"]
    cap_ptr = NC * (3 + d["S"] * (2 + Wp))
    cap_da = max(1, x.size)
    ptr = np.empty(cap_ptr, dtype=np.int32)
    da = np.empty(cap_da, dtype=np.float32)
    inn = np.empty(cap_da, dtype=np.int32)
    off = np.empty(3 * (NC + 1), dtype=np.int64)
    lens = np.zeros(3, dtype=np.int64)
    rc = _L().oc_encode(ctypes.byref(_desc(d)), _p(x), int(cps), _p(ptr), cap_ptr, _p(da),
                        cap_da, _p(inn), cap_da, _p(off), _p(lens))
    if rc != 0:
        raise RuntimeError(f"oracle encode overflow, needed {lens.tolist()}")
    off = off.reshape(3, NC + 1)
    return Encoding(ptr=ptr[:lens[0]].copy(), da=da[:lens[1]].copy(), inn=inn[:lens[2]].copy(),
                    chan_ptr_off=off[0].copy(), chan_nz_off=off[1].copy(), chan_in_off=off[2].copy(),
                    cps=bool(cps))


def decode(d: dict, enc: Encoding) -> np.ndarray:
    """Dense map from the streams (independent of the encoder)."""
    x = np.empty((d["N"], d["C"], d["H"], d["W"]), dtype=np.float32)
    ptr, da, inn = enc["ptr"], enc["da"], enc["inn"]
    rc = _L().oc_decode(ctypes.byref(_desc(d)), int(enc["cps"]), _p(ptr), ptr.size, _p(da), da.size,
                        _p(inn), inn.size, _p(x))
    if rc != 0:
        raise ValueError("corrupt CPO/CPS streams")
    return x


def sparse_conv(d: dict, enc: Encoding, w: np.ndarray) -> np.ndarray:
    """Alg. 2 (CPO) / Alg. 4 (CPS) / SI Alg. 6 (K_w=1) over the streams, FP64."""
    Oh, Ow = out_hw(d)
    w = _f32(w)
    y = np.empty((d["N"], d["K"], Oh, Ow), dtype=np.float64)
    ptr = enc["ptr"]
    rc = _L().oc_sparse_conv(ctypes.byref(_desc(d)), int(enc["cps"]), _p(ptr), ptr.size,
                             _p(enc["da"]), _p(enc["inn"]), _p(w), _p(y))
    if rc != 0:
        raise ValueError("corrupt CPO/CPS streams")
    return y


def mac_count(d: dict, x: np.ndarray) -> int:
    """Exact multiply-adds of the sparse conv: sum over NZEs of covering (output, tap) pairs, times K."""
    return int(_L().oc_mac_count(ctypes.byref(_desc(d)), _p(_f32(x))))


def set4_census(d: dict, x: np.ndarray) -> np.ndarray:
    """[C'_1..C'_4, C''_1..C''_4] of SI Eq. 5."""
    cen = np.zeros(8, dtype=np.int64)
    _L().oc_set4_census(ctypes.byref(_desc(d)), _p(_f32(x)), _p(cen))
    return cen


def count_flags(ptr: np.ndarray) -> tuple[int, int]:
    """(count_NPF, count_NPC) in a ptr stream."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    ptr = np.ascontiguousarray(ptr, dtype=np.int32)
    _L().oc_count_flags(_p(ptr), ptr.size, ctypes.byref(a), ctypes.byref(b))
    return a.value, b.value


def pattern_size(p: int) -> int:
    return int(_L().oc_pattern_size(p))


def next_offset(p: int, g: int) -> int:
    return int(_L().oc_next_offset(p, g))


def cscc_encode(d: dict, x: np.ndarray) -> Encoding:
    """CSCC streams (SI Alg. 5 for any K_w and s_w; Eq. 17 layout)."""
    x = _f32(x)
    NC = d["N"] * d["C"]
    _, Ow = out_hw(d)
    cap_ptr = NC * (Ow + 1)
    cap_da = max(1, NC * Ow * d["S"] * (d["H"] + d["pad_top"] + d["pad_bottom"]))
    ptr = np.empty(cap_ptr, dtype=np.int32)
    da = np.empty(cap_da, dtype=np.float32)
    inn = np.empty(cap_da, dtype=np.int32)
    off = np.empty(3 * (NC + 1), dtype=np.int64)
    lens = np.zeros(3, dtype=np.int64)
    rc = _L().oc_cscc_encode(ctypes.byref(_desc(d)), _p(x), _p(ptr), cap_ptr, _p(da), cap_da, _p(inn), cap_da,
                             _p(off), _p(lens))
    if rc != 0:
        raise RuntimeError(f"oracle cscc overflow, needed {lens.tolist()}")
    off = off.reshape(3, NC + 1)
    return Encoding(ptr=ptr[:lens[0]].copy(), da=da[:lens[1]].copy(), inn=inn[:lens[2]].copy(),
                    chan_ptr_off=off[0].copy(), chan_nz_off=off[1].copy(), chan_in_off=off[2].copy(),
                    cps=False, cscc=True)


def cscc_conv(d: dict, enc: Encoding, w: np.ndarray) -> np.ndarray:
    """SI Alg. 6 over CSCC streams, FP64 -> [N, K, Oh, Ow]."""
    Oh, Ow = out_hw(d)
    y = np.empty((d["N"], d["K"], Oh, Ow), dtype=np.float64)
    ptr, da = enc["ptr"], enc["da"]
    rc = _L().oc_cscc_conv(ctypes.byref(_desc(d)), _p(ptr), ptr.size, _p(da), da.size, _p(enc["inn"]),
                           _p(_f32(w)), _p(y))
    if rc != 0:
        raise ValueError("corrupt CSCC streams")
    return y


def cscc_decode(d: dict, enc: Encoding) -> np.ndarray:
    x = np.empty((d["N"], d["C"], d["H"], d["W"]), dtype=np.float32)
    ptr, da = enc["ptr"], enc["da"]
    rc = _L().oc_cscc_decode(ctypes.byref(_desc(d)), _p(ptr), ptr.size, _p(da), da.size, _p(enc["inn"]), _p(x))
    if rc != 0:
        raise ValueError("corrupt CSCC streams")
    return x


def encode_sa(d: dict, x: np.ndarray) -> Encoding:
    """Stride-aware CPO layout (reading A32; SI Eq. 2's ceil(K_w/s_w) types)."""
    x = _f32(x)
    NC = d["N"] * d["C"]
    _, Ow = out_hw(d)
    cap_ptr = NC * (2 + d["S"] * (1 + Ow))
    cap_da = max(1, x.size)
    ptr = np.empty(cap_ptr, dtype=np.int32)
    da = np.empty(cap_da, dtype=np.float32)
    inn = np.empty(cap_da, dtype=np.int32)
    off = np.empty(3 * (NC + 1), dtype=np.int64)
    lens = np.zeros(3, dtype=np.int64)
    rc = _L().oc_encode_sa(ctypes.byref(_desc(d)), _p(x), _p(ptr), cap_ptr, _p(da), cap_da, _p(inn), cap_da,
                           _p(off), _p(lens))
    if rc != 0:
        raise RuntimeError(f"oracle encode_sa overflow, needed {lens.tolist()}")
    off = off.reshape(3, NC + 1)
    return Encoding(ptr=ptr[:lens[0]].copy(), da=da[:lens[1]].copy(), inn=inn[:lens[2]].copy(),
                    chan_ptr_off=off[0].copy(), chan_nz_off=off[1].copy(), chan_in_off=off[2].copy(),
                    cps=False, stride_aware=True)


def decode_sa(d: dict, enc: Encoding) -> np.ndarray:
    x = np.empty((d["N"], d["C"], d["H"], d["W"]), dtype=np.float32)
    ptr, da = enc["ptr"], enc["da"]
    if _L().oc_decode_sa(ctypes.byref(_desc(d)), _p(ptr), ptr.size, _p(da), da.size, _p(enc["inn"]), _p(x)) != 0:
        raise ValueError("corrupt stride-aware streams")
    return x


def sparse_conv_sa(d: dict, enc: Encoding, w: np.ndarray) -> np.ndarray:
    """Alg. 2 over the stride-aware layout: an NZE of partition s, type t feeds the t+1
    partitions s..s+t covering its column (FP64)."""
    Oh, Ow = out_hw(d)
    y = np.empty((d["N"], d["K"], Oh, Ow), dtype=np.float64)
    ptr, da = enc["ptr"], enc["da"]
    if _L().oc_sparse_conv_sa(ctypes.byref(_desc(d)), _p(ptr), ptr.size, _p(da), da.size, _p(enc["inn"]),
                              _p(_f32(w)), _p(y)) != 0:
        raise ValueError("corrupt stride-aware streams")
    return y
