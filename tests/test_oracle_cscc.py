"""Oracle pins of the CSCC baseline (the paper's comparison method, PAPER.md:441, :505;
encoder = SI Alg. 5 generalised to any K_w / s_w as PAPER.md:1343 says the original is;
conv = SI Alg. 6; size = SI Eq. 17) and of the CSCC space bounds
P(rho), Q(rho_hat).  CPU only."""
import numpy as np
import pytest

from synth import int_map, int_weights, clustered_relu, he_normal, layer_desc
from test_oracle_sweep import CASES


def _xp(d, x):
    return np.pad(x, ((0, 0), (0, 0), (d["pad_top"], d["pad_bottom"]), (d["pad_left"], d["pad_right"])))


def _ow(d):
    return (d["W"] + d["pad_left"] + d["pad_right"] - d["S"]) // d["stride_w"] + 1


def cscc_from_definition(d, x):
    """CSR of each output column's K_w-wide submatrix of the padded map, row-major inside it
    (the lowered matrix LM of SI Eq. 17), written with numpy slicing: the streams CSCC defines."""
    xp = _xp(d, x)
    ptr, da, inn = [], [], []
    for n in range(d["N"]):
        for c in range(d["C"]):
            ptr.append(0)
            cnt = 0
            for s in range(_ow(d)):
                sub = xp[n, c, :, s * d["stride_w"]: s * d["stride_w"] + d["S"]].reshape(-1)
                nzi = np.flatnonzero(sub != 0)
                da.extend(sub[nzi].tolist())
                inn.extend(nzi.tolist())
                cnt += nzi.size
                ptr.append(cnt)
    return np.array(ptr, np.int32), np.array(da, np.float32), np.array(inn, np.int32)


def test_cscc_hand_example(oracle_mod):
    """2x3 map, K = 2x2, VALID, s = 1 (O_w = 2), written out by hand from SI Alg. 5:
    submatrix 0 = cols 0-1: (0,0)=1 -> IN 0, (1,1)=3 -> IN 1 + 1*2 = 3; submatrix 1 =
    cols 1-2: (0,2)=2 -> IN 1, (1,1)=3 -> IN 0 + 2 = 2; ptr = [0, 2, 4]."""
    d = layer_desc(1, 1, 2, 3, 1, 2, 2)
    x = np.array([[[[1, 0, 2], [0, 3, 0]]]], np.float32)
    e = oracle_mod.cscc_encode(d, x)
    assert e["ptr"].tolist() == [0, 2, 4]
    assert e["da"].tolist() == [1, 3, 2, 3]
    assert e["inn"].tolist() == [0, 3, 1, 2]
    w = np.array([[[[1, 10], [100, 1000]]]], np.float32)
    # O[0][0] = 1*1 + 3*1000, O[0][1] = 2*10 + 3*100
    assert oracle_mod.cscc_conv(d, e, w).reshape(-1).tolist() == [3001.0, 320.0]


def test_cscc_sweep_streams_conv_sizes(oracle_mod):
    """Over the 400-case integer sweep (strides 1/2, 1x7 / 7x1 / 5x5 / 2x2 / 3x5, VALID / SAME /
    partial pads, densities 0..1): streams == CSR of the lowered submatrices (numpy), SI Alg. 6
    conv == direct Eq. 1 conv exactly, decode(encode(x)) == x on the covered columns, lengths ==
    SI Eq. 17 with rho_hat from the numpy-lowered matrix, DA == nnz of the MEC lowering (SI Eq. 11
    matrix, the same submatrices)."""
    for d, rho, seed in CASES:
        x = int_map(d["N"], d["C"], d["H"], d["W"], rho, seed)
        w = int_weights(d["K"], d["C"], d["R"], d["S"], seed)
        e = oracle_mod.cscc_encode(d, x)
        p, a, i = cscc_from_definition(d, x)
        assert np.array_equal(e["ptr"], p) and np.array_equal(e["da"], a) and np.array_equal(e["inn"], i), d
        assert np.array_equal(oracle_mod.cscc_conv(d, e, w), oracle_mod.direct_conv(d, x, w)), d
        # decode: every column some submatrix covers comes back; the others are never read
        cov = np.zeros(d["W"] + d["pad_left"] + d["pad_right"], bool)
        for s in range(_ow(d)):
            cov[s * d["stride_w"]: s * d["stride_w"] + d["S"]] = True
        keep = cov[d["pad_left"]: d["pad_left"] + d["W"]]
        assert np.array_equal(oracle_mod.cscc_decode(d, e), x * keep[None, None, None, :]), d
        nnz_lm = int(a.size)
        rh = oracle_mod.rho_hat(d, nnz_lm)
        total = e["ptr"].size + e["da"].size + e["inn"].size
        assert abs(total - oracle_mod.S_cscc_eq17(d, rh)) < 1e-6 * max(1, total), d
        assert e["ptr"].size == d["N"] * d["C"] * (_ow(d) + 1)
        assert nnz_lm == int(np.count_nonzero(oracle_mod.mec_lower(d, x)))


def test_cscc_corrupt_streams_rejected(oracle_mod):
    d = layer_desc(1, 2, 6, 6, 2, 3, 3, 1, 1, 1, 1, 1, 1)
    x = int_map(1, 2, 6, 6, 0.5, 3)
    e = oracle_mod.cscc_encode(d, x)
    bad = dict(e)
    bad["ptr"] = e["ptr"].copy()
    bad["ptr"][3] = bad["ptr"][2] - 1            # decreasing count
    with pytest.raises(ValueError):
        oracle_mod.cscc_decode(d, type(e)(bad))
    with pytest.raises(ValueError):
        oracle_mod.cscc_conv(d, type(e)(bad), int_weights(2, 2, 3, 3, 1))


def test_cscc_real_valued_close(oracle_mod):
    d = layer_desc(2, 16, 14, 14, 8, 3, 3, 2, 2, 1, 1, 1, 1)
    x = clustered_relu(2, 16, 14, 14, 0.2, 3, dead_frac=0.25)
    w = he_normal(8, 16, 3, 3, 3)
    np.testing.assert_allclose(oracle_mod.cscc_conv(d, oracle_mod.cscc_encode(d, x), w),
                               oracle_mod.direct_conv(d, x, w), rtol=1e-12, atol=1e-12)


SHAPES = [layer_desc(1, 8, 14, 14, 8, 3, 3, 1, 1, 0, 0, 0, 0), layer_desc(2, 4, 12, 17, 4, 1, 7, 1, 1),
          layer_desc(1, 6, 9, 9, 6, 5, 5, 1, 1, 0, 0, 0, 0), layer_desc(1, 4, 28, 28, 4, 3, 3, 1, 1, 0, 0, 0, 0)]


@pytest.mark.parametrize("i", range(len(SHAPES)))
def test_cscc_bound_is_the_exact_worst_case_crossover(oracle_mod, i):
    """P(rho) for CSCC (reading A31): at the bound the worst-case CPO size
    equals S_CSCC of Eq. 17 exactly (when the bound is inside (0, 1)); below it CPO is no
    larger; Q(rho_hat) is exactly where the bound reaches 0.  And on real
    encodings (VALID, stride 1, where the worst case applies): average density <= P(rho_hat
    of the map) implies measured CPO size <= measured CSCC size."""
    d = SHAPES[i]
    from oracle import sizes
    q = oracle_mod.q_bound_cscc(d)
    assert oracle_mod.p_bound_cscc(d, q) == 0.0
    assert oracle_mod.p_bound_cscc(d, q + 1e-3) > 0.0 or q + 1e-3 > 1
    for rh in (0.02, 0.05, 0.1, 0.2):
        pb = oracle_mod.p_bound_cscc(d, rh)
        s_cscc = oracle_mod.S_cscc_eq17(d, rh * d["N"])
        if 0.0 < pb < 1.0:
            assert abs(sizes.s_cpo_worst_kc(d, pb) - s_cscc) < 1e-6 * s_cscc
            assert sizes.s_cpo_worst_kc(d, pb * 0.99) < s_cscc
    rng = np.random.default_rng(i)
    for rho in (0.02, 0.05, 0.1, 0.2, 0.4):
        x = int_map(d["N"], d["C"], d["H"], d["W"], rho, int(rng.integers(1 << 30)))
        cpo = oracle_mod.encode(d, x)
        cs = oracle_mod.cscc_encode(d, x)
        rbar = float((x != 0).mean())
        rh_bar = oracle_mod.rho_hat(d, cs["da"].size) / d["N"]
        s_cpo = cpo["ptr"].size + cpo["da"].size + cpo["inn"].size
        s_cs = cs["ptr"].size + cs["da"].size + cs["inn"].size
        if rbar <= oracle_mod.p_bound_cscc(d, rh_bar):
            assert s_cpo <= s_cs, (rho, s_cpo, s_cs)
