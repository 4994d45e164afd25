"""BASELINE.json workload catalogue: shapes, pads, strides, densities, seeds.

cfg1..cfg5 follow BASELINE.json "configs" in order;
cfg5 is the 16 non-pointwise 3x3 layers of a ResNet-50 v1.5 stack.
Descriptors are plain dicts with the C-ABI field names
(N,C,H,W,K,R,S,stride_h,stride_w,pad_top,pad_bottom,pad_left,pad_right).
"""
from __future__ import annotations

import numpy as np


def layer_desc(N, C, H, W, K, R, S, sh=1, sw=1, pt=0, pb=0, pl=0, pr=0) -> dict:
    return dict(N=N, C=C, H=H, W=W, K=K, R=R, S=S, stride_h=sh, stride_w=sw,
                pad_top=pt, pad_bottom=pb, pad_left=pl, pad_right=pr)


CONFIGS = {
    # 1) single 3x3 layer, batch 1, 16->16 @14x14, rho 0.2, 2/16 dead channels
    "cfg1": dict(desc=layer_desc(1, 16, 14, 14, 16, 3, 3, 1, 1, 1, 1, 1, 1),
                 density=0.20, dead_frac=2 / 16, zero_tile_frac=0.0, seed=101,
                 select_seeds=[1101, 1102, 1103, 1104, 1105]),
    # 2) ResNet-style 3x3, batch 1, 64->64 @56x56, rho 0.3, 5% dead, 10% 8x8 zero tiles
    "cfg2": dict(desc=layer_desc(1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1, 1, 1),
                 density=0.30, dead_frac=0.05, zero_tile_frac=0.10, seed=102,
                 select_seeds=[1201, 1202, 1203, 1204, 1205]),
    # 3) deep 3x3, batch 8, 256->256 @14x14, rho 0.1, 20% dead; also stride 2 and a density sweep
    "cfg3": dict(desc=layer_desc(8, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1, 1, 1),
                 density=0.10, dead_frac=0.20, zero_tile_frac=0.0, seed=103,
                 select_seeds=[1301, 1302, 1303, 1304, 1305],
                 sweep=[0.05, 0.1, 0.2, 0.3, 0.5]),
    "cfg3s2": dict(desc=layer_desc(8, 256, 14, 14, 256, 3, 3, 2, 2, 1, 1, 1, 1),
                   density=0.10, dead_frac=0.20, zero_tile_frac=0.0, seed=103,
                   select_seeds=[1301, 1302, 1303, 1304, 1305]),
    # 4) Inception-v3 asymmetric pair, batch 8, 192 @17x17: 1x7 pad (0,3) then 7x1 pad (3,0)
    "cfg4a": dict(desc=layer_desc(8, 192, 17, 17, 192, 1, 7, 1, 1, 0, 0, 3, 3),
                  density=0.05, dead_frac=0.15, zero_tile_frac=0.0, seed=104,
                  select_seeds=[1401, 1402, 1403, 1404, 1405]),
    "cfg4b": dict(desc=layer_desc(8, 192, 17, 17, 192, 7, 1, 1, 1, 3, 3, 0, 0),
                  density=None, dead_frac=0.0, zero_tile_frac=0.0, seed=104,
                  select_seeds=[1401, 1402, 1403, 1404, 1405],
                  note="input = ReLU(cfg4a output)"),
}

# Shape catalog beyond the BASELINE configs (SURVEY.md §8(f) NEXT-4 "shape sweeps"): the
# non-pointwise layer shapes of the paper's other CNNs -- Inception-v3 (5x5 and 3x3 at 35x35,
# 1x7 / 7x1 at 17x17 with 128 / 160 channels, 1x3 / 3x1 at 8x8) and a VGG-style 3x3 at
# 112x112 (outside the strip kernel's row range: the generic kernel).  Synthetic inputs as
# cfg3/cfg4 (clustered ReLU, batch 8, He weights); crossover sweeps only (tools/crossover.py).
CATALOG = {
    "iv3_5x5_35": dict(desc=layer_desc(8, 48, 35, 35, 64, 5, 5, 1, 1, 2, 2, 2, 2), density=0.3, seed=201),
    "iv3_3x3_35": dict(desc=layer_desc(8, 64, 35, 35, 96, 3, 3, 1, 1, 1, 1, 1, 1), density=0.3, seed=202),
    "iv3_3x3_35b": dict(desc=layer_desc(8, 96, 35, 35, 96, 3, 3, 1, 1, 1, 1, 1, 1), density=0.3, seed=203),
    "iv3_1x7_17": dict(desc=layer_desc(8, 128, 17, 17, 128, 1, 7, 1, 1, 0, 0, 3, 3), density=0.3, seed=204),
    "iv3_7x1_17": dict(desc=layer_desc(8, 160, 17, 17, 160, 7, 1, 1, 1, 3, 3, 0, 0), density=0.3, seed=205),
    "iv3_1x3_8": dict(desc=layer_desc(8, 384, 8, 8, 384, 1, 3, 1, 1, 0, 0, 1, 1), density=0.3, seed=206),
    "iv3_3x1_8": dict(desc=layer_desc(8, 384, 8, 8, 384, 3, 1, 1, 1, 1, 1, 0, 0), density=0.3, seed=207),
    "vgg_3x3_112": dict(desc=layer_desc(1, 128, 112, 112, 128, 3, 3, 1, 1, 1, 1, 1, 1), density=0.3, seed=208),
    "s2_3x3_112": dict(desc=layer_desc(2, 128, 112, 112, 128, 3, 3, 2, 2, 1, 1, 1, 1), density=0.3, seed=209),
}
for _c in CATALOG.values():
    _c.update(dead_frac=0.0, zero_tile_frac=0.0)

# ResNet-50 v1.5 non-pointwise 3x3 layers (C_in == C_out), all pad 1.
_CFG5 = ([(64, 56, 1)] * 3 + [(128, 56, 2)] + [(128, 28, 1)] * 3 +
         [(256, 28, 2)] + [(256, 14, 1)] * 5 + [(512, 14, 2)] + [(512, 7, 1)] * 2)


def cfg5_layers(batch: int = 32, seed: int = 105) -> list[dict]:
    """16 layers; per-layer density ~ U(0.05, 0.5) drawn from `seed`; each layer's
    input generated independently."""
    rho = np.random.Generator(np.random.PCG64(seed)).uniform(0.05, 0.5, len(_CFG5))
    layers = []
    for i, (ch, hw, s) in enumerate(_CFG5):
        layers.append(dict(desc=layer_desc(batch, ch, hw, hw, ch, 3, 3, s, s, 1, 1, 1, 1),
                           density=float(rho[i]), dead_frac=0.0, zero_tile_frac=0.0,
                           seed=seed * 1000 + i, name=f"L{i:02d}_{ch}@{hw}s{s}"))
    return layers
