"""Test helpers: fixture loading, independent numpy references, tolerance check."""
from __future__ import annotations

import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
NPF = -(2 ** 31) + 1


def load_fig1():
    with open(os.path.join(GOLDEN, "fig1.json")) as f:
        g = json.load(f)
    d = {k: v for k, v in g["geometry"].items() if not k.startswith("_")}
    x = np.zeros((1, 1, 8, 8), dtype=np.float32)
    nz = g["nzes"]
    for r, c, v in zip(nz["rows"], nz["cols"], nz["vals"]):
        x[0, 0, r, c] = v
    exp = dict(g["expected"])
    exp["ptr"] = [NPF if v == "NPF" else v for v in exp["ptr"]]
    return d, x, exp


def np_conv_einsum(d: dict, x: np.ndarray, w: np.ndarray) -> np.ndarray:
    """Independent Eq. 1 reference: sum over kernel taps of shifted-slice einsums (FP64)."""
    N, C, H, W = x.shape
    K, _, R, S = w.shape
    sh, sw = d["stride_h"], d["stride_w"]
    xp = np.zeros((N, C, H + d["pad_top"] + d["pad_bottom"], W + d["pad_left"] + d["pad_right"]))
    xp[:, :, d["pad_top"]:d["pad_top"] + H, d["pad_left"]:d["pad_left"] + W] = x
    Oh = (xp.shape[2] - R) // sh + 1
    Ow = (xp.shape[3] - S) // sw + 1
    y = np.zeros((N, K, Oh, Ow))
    for l in range(R):
        for m in range(S):
            patch = xp[:, :, l:l + sh * (Oh - 1) + 1:sh, m:m + sw * (Ow - 1) + 1:sw]
            y += np.einsum("nchw,kc->nkhw", patch, w[:, :, l, m].astype(np.float64))
    return y


def within_tol(got: np.ndarray, ref: np.ndarray, rel: float = 1e-4, abs_: float = 1e-5):
    """north_star tolerance: |got - ref| <= max(rel*|ref|, abs_) per element."""
    err = np.abs(got.astype(np.float64) - ref)
    bound = np.maximum(rel * np.abs(ref), abs_)
    bad = err > bound
    return (not bad.any()), float(err.max(initial=0.0)), int(bad.sum())


def valid_sparse_geometry(d: dict) -> bool:
    """Preconditions of the canonical encoding."""
    R, S = d["R"], d["S"]
    Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
    Wp = d["W"] + d["pad_left"] + d["pad_right"]
    if R == 1 and S == 1:
        return False
    if Hp < R or Wp < S:
        return False
    if S > 1 and (d["pad_left"] != d["pad_right"] or d["pad_left"] > S - 1 or Wp < 2 * S - 1):
        return False
    if S == 1 and (d["pad_left"] or d["pad_right"]):
        return False
    if d["pad_top"] > R - 1 or d["pad_bottom"] > R - 1:
        return False
    return True
