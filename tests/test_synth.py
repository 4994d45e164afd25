"""The seeded generator hits the BASELINE.json structure exactly (Appendix B recipe)."""
import numpy as np

from synth import CONFIGS, clustered_relu, cfg5_layers


def test_exact_density_dead_channels_and_tiles():
    c = CONFIGS["cfg2"]
    d = c["desc"]
    x = clustered_relu(1, 16, 56, 56, c["density"], c["seed"], dead_frac=0.25, zero_tile_frac=0.1)
    assert int((x != 0).sum()) == round(0.3 * 16 * 56 * 56)
    assert (x >= 0).all() and np.isfinite(x).all()
    dead = [ch for ch in range(16) if not x[0, ch].any()]
    assert len(dead) >= 4
    # 8x8 tiles that are zero in every channel: at least round(0.1 * 49) = 5
    tiles = sum(1 for ty in range(7) for tx in range(7)
                if not x[0, :, ty * 8:ty * 8 + 8, tx * 8:tx * 8 + 8].any())
    assert tiles >= 5
    assert d["C"] == 64


def test_seeded_reproducible():
    a = clustered_relu(2, 4, 14, 14, 0.1, 7)
    b = clustered_relu(2, 4, 14, 14, 0.1, 7)
    assert np.array_equal(a, b)
    assert not np.array_equal(a[0], a[1])


def test_cfg5_catalogue():
    L = cfg5_layers(batch=4)
    assert len(L) == 16
    assert all(0.05 <= l["density"] <= 0.5 for l in L)
    assert [l["desc"]["stride_h"] for l in L].count(2) == 3
