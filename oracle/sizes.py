"""Closed-form space model of the SI, written out as printed.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Units are stored
elements (one int32 or fp32 each), as the SI counts them.

Readings:
  * The encoding is stride-agnostic (A15), so the ptr formulas use the
    stride-1 partition count Ow1 = Wp - K_w + 1 and ceil(K_w/s_w) = K_w.
  * NOP_size is 3 iff Pad_Left = 0 (VALID) and K_w > 1, else 0 (A2; SI Alg. 5
    has no NOP block for K_w = 1).
  * S_im2col uses the actual (floor) output dims (A14); S_MEC uses the padded
    height (MEC lowers the padded map).
"""
from __future__ import annotations

import numpy as np


def _ow1(d: dict) -> int:
    return d["W"] + d["pad_left"] + d["pad_right"] - d["S"] + 1


def op_size_eq2(d: dict) -> int:
    """SI Eq. 2: (1+O_w) if K_w = 1, else (ceil(K_w/s_w) - M)(1+O_w),
    M = max(1, pad_left)."""
    ow1 = _ow1(d)
    if d["S"] == 1:
        return 1 + ow1
    M = max(1, d["pad_left"])
    return (d["S"] - M) * (1 + ow1)


def nop_size(d: dict) -> int:
    """NOP block: 3 entries for VALID padding, 0 for SAME."""
    return 3 if (d["pad_left"] == 0 and d["S"] > 1) else 0


def ptr_size_eq3(d: dict, chan_density: np.ndarray, count_npf: int) -> int:
    """SI Eq. 3:
    sum_{n,c} max(1, 1[rho_{n,c} > 0] (NOP_size + OP_size)) - count_NPF (O_w - 1)."""
    per = nop_size(d) + op_size_eq2(d)
    live = np.asarray(chan_density).reshape(-1) > 0
    total = int(np.sum(np.maximum(1, live.astype(np.int64) * per)))
    return total - count_npf * (_ow1(d) - 1)


def da_size_eq4(d: dict, chan_density: np.ndarray) -> int:
    """SI Eq. 4: DA = IN_CPO = I_h I_w sum_{n,c} rho_{n,c}."""
    return int(round(d["H"] * d["W"] * float(np.sum(chan_density))))


def in_cps_size_eq5(census: np.ndarray) -> int:
    """SI Eq. 5:
    sum (C'_1 + 2C'_2 + 3C'_3 + 4C'_4 + C''_1 + 2C''_2 + 2C''_3 + 2C''_4)."""
    c1, c2, c3, c4, d1, d2, d3, d4 = (int(v) for v in census)
    return c1 + 2 * c2 + 3 * c3 + 4 * c4 + d1 + 2 * d2 + 2 * d3 + 2 * d4


def _out(i, p0, p1, k, s):
    return (i + p0 + p1 - k) // s + 1


def S_im2col(d: dict) -> int:
    """SI Eq. 6: I_n O_w O_h I_c K_w K_h."""
    Oh = _out(d["H"], d["pad_top"], d["pad_bottom"], d["R"], d["stride_h"])
    Ow = _out(d["W"], d["pad_left"], d["pad_right"], d["S"], d["stride_w"])
    return d["N"] * Ow * Oh * d["C"] * d["S"] * d["R"]


def S_mec(d: dict) -> int:
    """SI Eq. 11: I_n O_w K_w I_h I_c (I_h of the padded map)."""
    Ow = _out(d["W"], d["pad_left"], d["pad_right"], d["S"], d["stride_w"])
    Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    return d["N"] * Ow * d["S"] * Hp * d["C"]


def channel_density(x: np.ndarray) -> np.ndarray:
    """rho_{n,c}: fraction of NZEs in each channel plane."""
    N, C, H, W = x.shape
    return (x.reshape(N, C, H * W) != 0).sum(axis=2) / float(H * W)


# ---- SI space-complexity bounds, written out as printed ----------
#
# Reading A29: the printed P(rho) bounds the SUM of the channel densities
# with a factor I_n I_c, then clips it to [0, 1]; only the average channel density
# rho_bar = sum_{n,c} rho_{n,c} / (I_n I_c) makes the clip meaningful, so the bound is
# taken on rho_bar:  rho_bar <= B / (I_n I_c).  Worst case as stated: M = 1 (VALID),
# no NPC, no NPF, K_w > s_w; ceil(K_w / s_w) = K_w for the stride-agnostic encoding (A15).

def _kw_ceil(d: dict) -> int:
    return d["S"]


def p_bound_im2col(d: dict) -> float:
    """Average density below which S_CPO <= S_im2col:
    (O_w (K_w K_h O_h + 1 - ceil(K_w/s_w)) - 2 - ceil(K_w/s_w)) / (2 I_h I_w), in [0, 1].
    O_w, O_h here are the stride-1 partition counts of the encoding (A15)."""
    ow, oh = _ow1(d), d["H"] + d["pad_top"] + d["pad_bottom"] - d["R"] + 1
    kc = _kw_ceil(d)
    b = (ow * (d["S"] * d["R"] * oh + 1 - kc) - 2 - kc) / (2.0 * d["H"] * d["W"])
    return min(1.0, max(0.0, b))


def p_bound_mec(d: dict) -> float:
    """Average density below which S_CPO <= S_MEC:
    (O_w (K_w I_h + 1 - ceil(K_w/s_w)) - 2 - ceil(K_w/s_w)) / (2 I_h I_w), in [0, 1]."""
    ow = _ow1(d)
    kc = _kw_ceil(d)
    b = (ow * (d["S"] * d["H"] + 1 - kc) - 2 - kc) / (2.0 * d["H"] * d["W"])
    return min(1.0, max(0.0, b))


def s_cpo_worst(d: dict, rho_bar: float) -> float:
    """Worst-case CPO size of the derivation:
    I_n I_c (3 + (ceil(K_w/s_w) - 1)(1 + O_w)) + 2 I_h I_w sum rho."""
    ow = _ow1(d)
    return d["N"] * d["C"] * (3 + (_kw_ceil(d) - 1) * (1 + ow)) + 2 * d["H"] * d["W"] * d["N"] * d["C"] * rho_bar


# ---- CSCC (SI §1.3) ------------------------------------------------
#
# Reading A30: CSCC lowers the PADDED map (like MEC, S2), one K_w-wide
# submatrix per output column at stride s_w, so I_h = Hp and O_w = the real output width.
# Reading A31: as A29, the printed P / Q bounds are taken on averages: rho_bar = average
# channel density, rho_hat_bar = average (over images) lowered-matrix density.

def _ow(d: dict) -> int:
    return _out(d["W"], d["pad_left"], d["pad_right"], d["S"], d["stride_w"])


def rho_hat(d: dict, lowered_nnz: int) -> float:
    """rho_hat = sum_i rho_hat_i: the lowered-matrix densities of the
    batch, each over O_w K_w I_h I_c elements."""
    Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    return lowered_nnz / float(_ow(d) * d["S"] * Hp * d["C"])


def S_cscc_eq17(d: dict, rho_hat_sum: float) -> float:
    """SI Eq. 17: I_n I_c (O_w + 1) + 2 O_w K_w I_h I_c rho_hat."""
    Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    ow = _ow(d)
    return d["N"] * d["C"] * (ow + 1) + 2.0 * ow * d["S"] * Hp * d["C"] * rho_hat_sum


def _kc(d: dict) -> int:
    return -(-d["S"] // d["stride_w"])          # ceil(K_w / s_w)


def p_bound_cscc(d: dict, rho_hat_bar: float) -> float:
    """Average channel density below which S_CPO (worst case) <= S_CSCC:
    rho_bar <= (2 O_w K_w Hp rho_hat_bar + (O_w + 1)(2 - ceil(K_w/s_w)) - 3) / (2 H W),
    clipped to [0, 1] (reading A31: the printed bound divided by I_n I_c; the CPO DA / IN
    term counts the H x W map's NZEs, the lowered matrix the padded Hp rows, reading A30)."""
    Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    ow, kc = _ow(d), _kc(d)
    b = (2.0 * ow * d["S"] * Hp * rho_hat_bar + (ow + 1) * (2 - kc) - 3) / (2.0 * d["H"] * d["W"])
    return min(1.0, max(0.0, b))


def q_bound_cscc(d: dict) -> float:
    """Q(rho_hat): the least average lowered-matrix density for which the
    P bound above is non-negative: (3 - (O_w + 1)(2 - ceil(K_w/s_w))) / (2 O_w I_h K_w)."""
    Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    ow, kc = _ow(d), _kc(d)
    return (3.0 - (ow + 1) * (2 - kc)) / (2.0 * ow * Hp * d["S"])


def s_cpo_worst_kc(d: dict, rho_bar: float) -> float:
    """Worst-case CPO size of the CSCC derivation with ceil(K_w/s_w):
    I_n I_c (3 + (kc - 1)(1 + O_w)) + 2 H W I_n I_c rho_bar."""
    ow, kc = _ow(d), _kc(d)
    return d["N"] * d["C"] * (3 + (kc - 1) * (1 + ow)) + 2.0 * d["H"] * d["W"] * d["N"] * d["C"] * rho_bar


# ---- stride-aware layout (reading A32, NEXT-4) ----------------------------------------

def sa_column_cover(d: dict) -> np.ndarray:
    """cov(w) of every padded column: output partitions s (stride s_w) with s*s_w <= w < s*s_w + K_w."""
    Wp = d["W"] + d["pad_left"] + d["pad_right"]
    cov = np.zeros(Wp, np.int64)
    for s in range(_ow(d)):
        cov[s * d["stride_w"]: s * d["stride_w"] + d["S"]] += 1
    return cov


def ptr_size_sa(d: dict, live_channels: int, count_npf: int) -> int:
    """ptr length of the stride-aware layout in the form of SI Eq. 3:
    every live channel carries one (1 + O_w) block per coverage type present -- the
    coverage-1 block (the NOP generalisation) plus Eq. 2's ceil(K_w/s_w) - 1 overlap blocks
    (M = 1) -- each NPF block saving O_w - 1 entries; a dead channel is one NPC entry."""
    ow = _ow(d)
    types = len(set(int(c) for c in sa_column_cover(d)) - {0})
    nc = d["N"] * d["C"]
    return (nc - live_channels) + live_channels * types * (1 + ow) - count_npf * (ow - 1)


def op_size_eq2_strided(d: dict) -> int:
    """SI Eq. 2 as printed with M = 1: (ceil(K_w/s_w) - 1)(1 + O_w), O_w at the real stride."""
    return (_kc(d) - 1) * (1 + _ow(d))
