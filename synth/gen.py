"""Seeded synthetic activation maps and weights.

The paper measures on ImageNet activations of pretrained CNNs (PAPER.md:441,
:443); neither the dataset nor the weights are available, so these seeded
generators stand in for them, with the shapes/densities/structure that
BASELINE.json's configs name (dead channels, 8x8 all-zero regions,
clustered NZEs from a smoothed Gaussian field).  The paper's own footnote says
it verified its code with "randomized feature maps".

Nothing here implements the method: no encoding, no convolution.
"""
from __future__ import annotations

import numpy as np


def _rng(*seed) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(list(seed) if len(seed) > 1 else seed[0]))


def _box3(z: np.ndarray) -> np.ndarray:
    """3x3 box mean over valid windows: z[..., H+2, W+2] -> [..., H, W]."""
    H, W = z.shape[-2] - 2, z.shape[-1] - 2
    acc = np.zeros(z.shape[:-2] + (H, W), dtype=np.float64)
    for dy in range(3):
        for dx in range(3):
            acc += z[..., dy:dy + H, dx:dx + W]
    return acc / 9.0


def clustered_relu(N: int, C: int, H: int, W: int, density: float, seed: int,
                   dead_frac: float = 0.0, zero_tile_frac: float = 0.0) -> np.ndarray:
    """ReLU(3x3-box-blurred N(0,1) field - t), t chosen per image so that exactly
    round(density*C*H*W) elements are non-zero.

    dead_frac: fraction of channels forced all-zero (drawn once, shared by images).
    zero_tile_frac: fraction of aligned 8x8 tiles forced all-zero (per image, all channels).
    Returns float32 [N, C, H, W]; every non-zero is positive and normal.
    """
    if not (0.0 <= density <= 1.0):
        raise ValueError("density must be in [0, 1]")
    n_dead = int(round(dead_frac * C))
    dead = _rng(seed).permutation(C)[:n_dead]
    tiles_y, tiles_x = H // 8, W // 8
    n_tiles = int(round(zero_tile_frac * tiles_y * tiles_x))
    out = np.zeros((N, C, H, W), dtype=np.float32)
    k = int(round(density * C * H * W))
    for n in range(N):
        rng = _rng(seed, n)
        blur = _box3(rng.standard_normal((C, H + 2, W + 2)))
        live = np.ones((C, H, W), dtype=bool)
        live[dead] = False
        if n_tiles:
            for t in rng.choice(tiles_y * tiles_x, size=n_tiles, replace=False):
                ty, tx = divmod(int(t), tiles_x)
                live[:, ty * 8:(ty + 1) * 8, tx * 8:(tx + 1) * 8] = False
        vals = blur[live]
        if k > vals.size:
            raise ValueError(f"density {density} needs {k} NZEs but only {vals.size} live cells")
        if k == 0:
            continue
        if k == vals.size:
            thr = -np.inf
        else:
            # (k+1)-th largest live value: exactly k values lie strictly above it
            thr = np.partition(vals, vals.size - k - 1)[vals.size - k - 1]
        sel = live & (blur > thr)
        x = np.where(sel, blur - (thr if np.isfinite(thr) else blur.min() - 1.0), 0.0)
        out[n] = x.astype(np.float32)
    return out


def he_normal(K: int, C: int, R: int, S: int, seed: int) -> np.ndarray:
    """float32(N(0,1) * sqrt(2/(C*R*S))), KCRS layout, drawn from seed+10000."""
    w = _rng(seed + 10000).standard_normal((K, C, R, S)) * np.sqrt(2.0 / (C * R * S))
    return w.astype(np.float32)


def random_sparse(N: int, C: int, H: int, W: int, density: float, seed: int) -> np.ndarray:
    """i.i.d. Bernoulli(density) support with uniform(0.1, 1) values (unclustered)."""
    rng = _rng(seed, 7)
    mask = rng.random((N, C, H, W)) < density
    vals = rng.uniform(0.1, 1.0, (N, C, H, W))
    return np.where(mask, vals, 0.0).astype(np.float32)


def int_map(N: int, C: int, H: int, W: int, density: float, seed: int, vmax: int = 8) -> np.ndarray:
    """Integer-valued map (values in [1, vmax]) for bit-exact comparisons."""
    rng = _rng(seed, 11)
    mask = rng.random((N, C, H, W)) < density
    vals = rng.integers(1, vmax + 1, (N, C, H, W))
    return np.where(mask, vals, 0).astype(np.float32)


def int_weights(K: int, C: int, R: int, S: int, seed: int, vmax: int = 8) -> np.ndarray:
    """Integer-valued weights in [-vmax, vmax]."""
    return _rng(seed, 13).integers(-vmax, vmax + 1, (K, C, R, S)).astype(np.float32)
