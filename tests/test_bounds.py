"""SI space bounds P(rho): oracle pinned to exact encoding sizes, product
pre-selector compared with the oracle."""
import numpy as np
import pytest

import oracle
from oracle import sizes
from paper_2104_08314_b200.bounds import cscc_q_bound, rho_space_bound, space_preselect
from synth import int_map, layer_desc

SHAPES = [layer_desc(1, 3, 14, 14, 4, 3, 3, 1, 1, 0, 0, 0, 0), layer_desc(2, 2, 9, 11, 4, 3, 3, 1, 1, 0, 0, 0, 0),
          layer_desc(1, 2, 17, 17, 4, 1, 7, 1, 1, 0, 0, 0, 0), layer_desc(1, 2, 8, 8, 4, 5, 5, 1, 1, 0, 0, 0, 0),
          layer_desc(1, 4, 7, 7, 4, 3, 3, 1, 1, 0, 0, 0, 0)]


@pytest.mark.parametrize("i", range(len(SHAPES)))
def test_p_bound_is_the_exact_worst_case_crossover(oracle_mod, i):
    """In the SI worst case (VALID, no NPC, no NPF) S_CPO = ptr + 2 nnz exactly (Eq. 3, 4), so
    P(rho) must be exactly the density where S_CPO meets S_im2col: encode real maps just
    below and just above it with the oracle and compare sizes."""
    d = SHAPES[i]
    rb = sizes.p_bound_im2col(d)
    s_i2c = sizes.S_im2col(d)
    hw, nc = d["H"] * d["W"], d["N"] * d["C"]
    # worst-case closed form equals the bound at rho = rb
    assert abs(sizes.s_cpo_worst(d, rb) - s_i2c) <= 1e-6 * s_i2c or rb in (0.0, 1.0)
    for target, expect_le in ((max(0.0, rb - 0.03), True), (min(1.0, rb + 0.03), False)):
        if rb >= 1.0 and not expect_le:
            continue
        # a full map with target density in every channel and every column populated
        rng = np.random.default_rng(i)
        x = np.zeros((d["N"], d["C"], d["H"], d["W"]), np.float32)
        k = int(round(target * hw))
        for n in range(d["N"]):
            for c in range(d["C"]):
                cells = rng.permutation(hw)[:k]
                x[n, c].flat[cells] = 1.0
        enc = oracle_mod.encode(d, x)
        npc, npf = oracle_mod.count_flags(enc["ptr"])
        if npc or npf:
            continue   # outside the worst case the bound is conservative, not exact
        s_cpo = len(enc["ptr"]) + len(enc["da"]) + len(enc["inn"])
        assert (s_cpo <= s_i2c) == expect_le, (d, target, s_cpo, s_i2c)


@pytest.mark.parametrize("i", range(len(SHAPES)))
def test_mec_bound_matches_its_closed_form(i):
    """Unclipped, the MEC bound is where the worst-case CPO size meets S_MEC (VALID padding,
    so the padded height of reading S2 equals I_h); clipped at 1, CPO is smaller at every density."""
    d = SHAPES[i]
    rb = sizes.p_bound_mec(d)
    s_mec = sizes.S_mec(d)
    if 0.0 < rb < 1.0:
        assert abs(sizes.s_cpo_worst(d, rb) - s_mec) <= 1e-6 * s_mec
    elif rb >= 1.0:
        assert sizes.s_cpo_worst(d, 1.0) <= s_mec


@pytest.mark.parametrize("seed", range(40))
def test_product_bound_equals_oracle(seed):
    rng = np.random.default_rng(seed)
    R, S = [(3, 3), (1, 7), (7, 1), (5, 5), (3, 1), (1, 3)][seed % 6]
    pl = int(rng.integers(0, S))
    d = layer_desc(int(rng.integers(1, 5)), int(rng.integers(1, 64)), int(rng.integers(R, 60)),
                   int(rng.integers(2 * S, 60)), 8, R, S, 1, 1, int(rng.integers(0, R)), int(rng.integers(0, R)),
                   pl, pl)
    assert rho_space_bound(d, "im2col") == pytest.approx(sizes.p_bound_im2col(d), abs=1e-12)
    assert rho_space_bound(d, "mec") == pytest.approx(sizes.p_bound_mec(d), abs=1e-12)
    d2 = dict(d, stride_w=int(rng.integers(1, 3)))
    for rh in (0.0, 0.03, 0.2, 0.7):
        assert rho_space_bound(d2, "cscc", rh) == pytest.approx(sizes.p_bound_cscc(d2, rh), abs=1e-12)
    assert cscc_q_bound(d2) == pytest.approx(sizes.q_bound_cscc(d2), abs=1e-12)


def test_preselector_routes_by_the_bound():
    d = layer_desc(1, 64, 56, 56, 64, 3, 3, 1, 1, 1, 1, 1, 1)
    rb = rho_space_bound(d)
    assert space_preselect(d, rb * 0.9) == "cpo"
    assert space_preselect(d, min(1.0, rb * 1.1 + 1e-3)) in ("im2col", "cpo")
    assert space_preselect(layer_desc(1, 4, 8, 8, 4, 1, 1), 0.01) == "im2col"
    q = cscc_q_bound(d)
    assert space_preselect(d, 0.0, "cscc", max(0.0, q) + 0.05) == "cpo"
    assert space_preselect(d, 1.0, "cscc", 0.0) == "cscc"


MEC_SHAPES = [layer_desc(1, 4, 7, 7, 4, 3, 3, 1, 1, 0, 0, 0, 0), layer_desc(1, 3, 20, 5, 4, 3, 3, 1, 1, 0, 0, 0, 0),
              layer_desc(2, 2, 30, 6, 4, 1, 3, 1, 1, 0, 0, 0, 0)]


@pytest.mark.parametrize("i", range(len(MEC_SHAPES)))
def test_mec_bound_on_real_encodings(oracle_mod, i):
    """P(rho) against MEC on real oracle encodings: S_MEC of Eq. 11 equals the
    size of the MEC lowered matrix the oracle builds (SI Eq. 11 matrix, VALID); maps just below the
    bound encode no larger than S_MEC, maps just above it larger (worst case: no NPC / NPF)."""
    d = MEC_SHAPES[i]
    rb = sizes.p_bound_mec(d)
    assert 0.0 < rb < 1.0
    s_mec = sizes.S_mec(d)
    hw = d["H"] * d["W"]
    for target, expect_le in ((rb - 0.03, True), (min(1.0, rb + 0.03), False)):
        rng = np.random.default_rng(i)
        x = np.zeros((d["N"], d["C"], d["H"], d["W"]), np.float32)
        k = int(round(target * hw))
        for n in range(d["N"]):
            for c in range(d["C"]):
                x[n, c].flat[rng.permutation(hw)[:k]] = 1.0
        assert oracle_mod.mec_lower(d, x).size == s_mec
        enc = oracle_mod.encode(d, x)
        npc, npf = oracle_mod.count_flags(enc["ptr"])
        assert not npc and not npf
        s_cpo = len(enc["ptr"]) + len(enc["da"]) + len(enc["inn"])
        assert (s_cpo <= s_mec) == expect_le, (d, target, s_cpo, s_mec)
