"""Zero-cost space pre-selector from the SI's closed-form bounds.

P(rho): the average channel density below which the CPO encoding is no larger than the
im2col lowered matrix (resp. the MEC lowered matrix), in the worst case the SI assumes
(VALID padding, no NPC, no NPF).  Reading A29: the bound is on the average
density rho_bar = sum_{n,c} rho_{n,c} / (I_n I_c).  Encoding geometry is stride-agnostic
(reading A15): partitions O_w1 = W_p - K_w + 1 and ceil(K_w / s_w) -> K_w.

Host-side arithmetic only (the oracle's copy lives in oracle/sizes.py; the two share no
code and are compared in tests/test_bounds.py).
"""
from __future__ import annotations


def _geom(d: dict):
    wp = d["W"] + d["pad_left"] + d["pad_right"]
    hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    return wp - d["S"] + 1, hp - d["R"] + 1


def rho_space_bound(d: dict, vs: str = "im2col") -> float:
    """Largest average density at which CPO is no larger than `vs` ("im2col" or "mec")."""
    ow1, oh1 = _geom(d)
    kw, kh, ih, iw = d["S"], d["R"], d["H"], d["W"]
    inner = kw * kh * oh1 if vs == "im2col" else kw * ih
    num = ow1 * (inner + 1 - kw) - 2 - kw
    return min(1.0, max(0.0, num / (2.0 * ih * iw)))


def space_preselect(d: dict, rho_bar: float, vs: str = "im2col") -> str:
    """favour_space pre-selection without timing: 'cpo' when the measured average density
    is inside P(rho), else the dense lowering."""
    if d["R"] == 1 and d["S"] == 1:
        return vs
    return "cpo" if rho_bar <= rho_space_bound(d, vs) else vs
