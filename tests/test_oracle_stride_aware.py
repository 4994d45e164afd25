"""Oracle pins of the stride-aware CPO layout (reading A32: partitions
are the output columns at stride s_w, SI Eq. 2's ceil(K_w/s_w) coverage types).
CPU only."""
import numpy as np
import pytest

from oracle import sizes
from synth import clustered_relu, he_normal, int_map, int_weights, layer_desc

KERNELS = [(3, 3), (5, 5), (1, 7), (7, 1), (3, 1), (1, 3), (2, 2), (3, 5), (4, 4)]


def strided_cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        R, S = KERNELS[rng.integers(len(KERNELS))]
        sh, sw = int(rng.integers(1, 4)), int(rng.integers(2, 4))
        pl = int(rng.integers(0, S))
        pt, pb = (int(rng.integers(0, R)) for _ in range(2))
        H = int(rng.integers(max(1, R - pt - pb), 13))
        W = int(rng.integers(max(1, S - 2 * pl), 16))
        if W + 2 * pl < S or H + pt + pb < R:
            continue
        d = layer_desc(int(rng.integers(1, 3)), int(rng.integers(1, 5)), H, W, int(rng.integers(1, 4)), R, S, sh, sw,
                       pt, pb, pl, pl)
        out.append((d, float(rng.choice([0.0, 0.05, 0.3, 0.6, 1.0])), int(rng.integers(1 << 30))))
    return out


CASES = strided_cases(300, 4)


def test_stride_aware_sweep(oracle_mod):
    """300 random strided cases (s_w in {2, 3}, s_h in 1..3, VALID / SAME / partial pads):
    conv over the layout == direct Eq. 1 conv exactly; decode == x on the covered columns;
    DA == NZEs of the covered columns; ptr length == the Eq. 3 form of reading A32."""
    for d, rho, seed in CASES:
        x = int_map(d["N"], d["C"], d["H"], d["W"], rho, seed)
        w = int_weights(d["K"], d["C"], d["R"], d["S"], seed)
        e = oracle_mod.encode_sa(d, x)
        assert np.array_equal(oracle_mod.sparse_conv_sa(d, e, w), oracle_mod.direct_conv(d, x, w)), d
        cov = sizes.sa_column_cover(d)[d["pad_left"]: d["pad_left"] + d["W"]] > 0
        xc = x * cov[None, None, None, :]
        assert np.array_equal(oracle_mod.decode_sa(d, e), xc), d
        assert e["da"].size == e["inn"].size == int(np.count_nonzero(xc))
        live = int((xc.reshape(d["N"] * d["C"], -1) != 0).any(axis=1).sum())
        npf, npc = oracle_mod.count_flags(e["ptr"])
        assert npc == d["N"] * d["C"] - live
        assert e["ptr"].size == sizes.ptr_size_sa(d, live, npf), d


def test_stride_aware_matches_eq2_type_count():
    """For K_w > s_w the overlap blocks (coverage >= 2) number ceil(K_w/s_w) - 1, SI Eq. 2 with
    M = 1: OP_size = (ceil(K_w/s_w) - 1)(1 + O_w)."""
    for (S, sw, W, p) in [(3, 2, 14, 1), (3, 2, 56, 1), (5, 2, 20, 2), (7, 2, 17, 3), (7, 3, 17, 3), (4, 3, 13, 0)]:
        d = layer_desc(1, 1, 5, W, 1, 1, S, 1, sw, 0, 0, p, p)
        cov = sizes.sa_column_cover(d)
        overlap_types = len(set(int(c) for c in cov) - {0, 1})
        assert overlap_types * (1 + sizes._ow(d)) == sizes.op_size_eq2_strided(d), (S, sw, W)


def test_stride_aware_fig1_like_example(oracle_mod):
    """4x5 map, K = 3x3 VALID, s = 2 (O_w = 2): columns 0,1 owned by partition 0 with coverage 1,
    column 2 by partition 0 with coverage 2 (shared with partition 1), columns 3,4 by partition 1,
    coverage 1 -- written out by hand:
      type 0 block [1, c_0, c_1]: col 0 rows {1}, col 1 rows {0, 2}, col 3 rows {3}, col 4 {}
                   -> DA (1,0)=10 (0,1)=1 (2,1)=21 | (3,3)=33 ; c = [3, 4]
      type 1 block [2, c_0, -1]: col 2 rows {1, 3} -> (1,2)=12, (3,2)=32 ; c = [2, -1]."""
    d = layer_desc(1, 1, 4, 5, 1, 3, 3, 1, 2)
    x = np.zeros((1, 1, 4, 5), np.float32)
    x[0, 0, 1, 0] = 10; x[0, 0, 0, 1] = 1; x[0, 0, 2, 1] = 21; x[0, 0, 3, 3] = 33
    x[0, 0, 1, 2] = 12; x[0, 0, 3, 2] = 32
    e = oracle_mod.encode_sa(d, x)
    assert e["ptr"].tolist() == [1, 3, 4, 2, 2, -1]
    assert e["da"].tolist() == [10, 1, 21, 33, 12, 32]
    # IN = L + h*K_w: (1,0) -> 0+3, (0,1) -> 1, (2,1) -> 1+6, (3,3) partition 1 L=1 -> 1+9,
    # (1,2) L=2 -> 2+3, (3,2) -> 2+9
    assert e["inn"].tolist() == [3, 1, 7, 10, 5, 11]


def test_stride_aware_smaller_ptr_at_stride_2(oracle_mod):
    """At s_w = 2 the layout stores about half the ptr entries of the stride-agnostic one (Ow vs
    Ow1 partitions) with the same DA, and the same conv result (cfg3 s2 / cfg5 s2 shapes)."""
    for (C, H) in [(16, 14), (8, 28), (4, 56)]:
        d = layer_desc(2, C, H, H, 8, 3, 3, 2, 2, 1, 1, 1, 1)
        x = clustered_relu(2, C, H, H, 0.2, 5)
        w = he_normal(8, C, 3, 3, 5)
        sa, agn = oracle_mod.encode_sa(d, x), oracle_mod.encode(d, x)
        assert sa["da"].size == agn["da"].size
        assert sa["ptr"].size < 0.6 * agn["ptr"].size
        np.testing.assert_allclose(oracle_mod.sparse_conv_sa(d, sa, w), oracle_mod.sparse_conv(d, agn, w),
                                   rtol=1e-12, atol=1e-12)
