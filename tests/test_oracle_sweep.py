"""Oracle pins against mathematics: Eq. 1 via independent references, exact
round trips, the SI closed-form sizes, and CPO/CPS conv == direct conv
bit-exactly on integer data over a randomized sweep (SPEC.md acceptance 1, 3, 4, 8 ideas)."""
import numpy as np
import pytest
import torch

from helpers import np_conv_einsum, valid_sparse_geometry
from synth import int_map, int_weights, clustered_relu, he_normal, layer_desc

KERNELS = [(3, 3), (4, 4), (5, 5), (1, 7), (7, 1), (3, 1), (1, 3), (2, 2), (3, 5)]


def random_cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        R, S = KERNELS[rng.integers(len(KERNELS))]
        sh, sw = (int(v) for v in rng.choice([1, 2], 2, p=[0.7, 0.3]))
        pl = int(rng.integers(0, S)) if S > 1 else 0
        pt, pb = (int(rng.integers(0, R)) for _ in range(2))
        H = int(rng.integers(max(1, R - pt - pb), 13))
        W = int(rng.integers(max(1, 2 * S - 1 - 2 * pl), 14))
        d = layer_desc(int(rng.integers(1, 3)), int(rng.integers(1, 5)), H, W,
                       int(rng.integers(1, 4)), R, S, sh, sw, pt, pb, pl, pl)
        if not valid_sparse_geometry(d):
            continue
        rho = float(rng.choice([0.0, 0.05, 0.3, 0.6, 1.0]))
        out.append((d, rho, int(rng.integers(1 << 30))))
    return out


CASES = random_cases(400, 2104)


def test_direct_conv_matches_independent_references(oracle_mod):
    d = layer_desc(2, 3, 9, 11, 4, 3, 3, 1, 1, 1, 1, 1, 1)
    x = clustered_relu(2, 3, 9, 11, 0.3, 5)
    w = he_normal(4, 3, 3, 3, 5)
    ref = oracle_mod.direct_conv(d, x, w)
    np.testing.assert_allclose(ref, np_conv_einsum(d, x, w), rtol=1e-12, atol=1e-13)
    t = torch.nn.functional.conv2d(torch.from_numpy(x).double(), torch.from_numpy(w).double(),
                                   stride=1, padding=1).numpy()
    np.testing.assert_allclose(ref, t, rtol=1e-12, atol=1e-13)
    # brute-force im2col + naive GEMM, and im2col + numpy matmul
    L = oracle_mod.im2col(d, x)
    np.testing.assert_allclose(oracle_mod.gemm_lowered(d, L, w), ref, rtol=1e-12, atol=1e-13)
    mm = np.matmul(L.astype(np.float64), w.reshape(4, -1).T.astype(np.float64))  # [N, P, K]
    np.testing.assert_allclose(mm.transpose(0, 2, 1).reshape(ref.shape), ref, rtol=1e-12, atol=1e-13)


@pytest.mark.parametrize("case", range(0, 400, 40))
def test_direct_conv_strided_asymmetric(oracle_mod, case):
    d, rho, seed = CASES[case]
    x = int_map(d["N"], d["C"], d["H"], d["W"], rho, seed)
    w = int_weights(d["K"], d["C"], d["R"], d["S"], seed)
    ref = oracle_mod.direct_conv(d, x, w)
    assert np.array_equal(ref, np_conv_einsum(d, x, w))
    t = torch.nn.functional.conv2d(
        torch.nn.functional.pad(torch.from_numpy(x).double(),
                                (d["pad_left"], d["pad_right"], d["pad_top"], d["pad_bottom"])),
        torch.from_numpy(w).double(), stride=(d["stride_h"], d["stride_w"])).numpy()
    assert np.array_equal(ref, t)


def test_sweep_sparse_conv_exact_and_sizes(oracle_mod):
    """Over 400 random cases (1x7, 7x1, 3x1, 4x4, 5x5, strides 1/2, VALID/SAME/partial pads,
    densities 0..1): decode(encode(x)) == x, DA == popcount (Eq. 4), ptr length == SI
    Eq. 3 with the actual NPF count, IN_CPS == SI Eq. 5 and <= IN_CPO (Eq. 24),
    CPO conv == CPS conv == direct conv exactly (integer data)."""
    for d, rho, seed in CASES:
        x = int_map(d["N"], d["C"], d["H"], d["W"], rho, seed)
        w = int_weights(d["K"], d["C"], d["R"], d["S"], seed)
        ref = oracle_mod.direct_conv(d, x, w)
        cpo = oracle_mod.encode(d, x, cps=False)
        cps = oracle_mod.encode(d, x, cps=True)
        assert np.array_equal(oracle_mod.decode(d, cpo), x), d
        assert np.array_equal(oracle_mod.decode(d, cps), x), d
        nnz = int((x != 0).sum())
        rho_nc = oracle_mod.sizes.channel_density(x)
        assert cpo["da"].size == cpo["inn"].size == nnz == oracle_mod.da_size_eq4(d, rho_nc)
        assert np.array_equal(cps["da"], cpo["da"]) and np.array_equal(cps["ptr"], cpo["ptr"])
        npf, npc = oracle_mod.count_flags(cpo["ptr"])
        assert npc == int((rho_nc.reshape(-1) == 0).sum())
        assert cpo["ptr"].size == oracle_mod.ptr_size_eq3(d, rho_nc, npf), d
        cen = oracle_mod.set4_census(d, x)
        if d["S"] > 1:
            assert cps["inn"].size == oracle_mod.in_cps_size_eq5(cen), d
        assert cps["inn"].size <= cpo["inn"].size
        for enc in (cpo, cps):
            assert np.array_equal(oracle_mod.sparse_conv(d, enc, w), ref), d
        # channel offsets are exclusive prefix sums of the segments
        assert cpo["chan_ptr_off"][-1] == cpo["ptr"].size
        assert cpo["chan_nz_off"][-1] == nnz
        assert cps["chan_in_off"][-1] == cps["inn"].size


def test_decoded_cps_indices_equal_cpo(oracle_mod):
    """Expanding the CPS overlapK_w entries ({index, pattern} / negated singles, Alg. 4)
    gives exactly the CPO index sequence (SPEC.md cps-codec invariant)."""
    d = layer_desc(1, 1, 13, 10, 2, 3, 3, 1, 1, 1, 1, 1, 1)
    x = int_map(1, 1, 13, 10, 0.6, 9)
    cpo, cps = oracle_mod.encode(d, x), oracle_mod.encode(d, x, cps=True)
    ptr = cpo["ptr"]                       # [2, c_0..c_9] (or [2, NPF]) then [3, c_0..c_9]
    n1 = 0 if ptr[1] == oracle_mod.NPF else int(ptr[1 + 9 - 1])
    assert np.array_equal(cps["inn"][:n1], cpo["inn"][:n1])
    idx, inn, i = [], cps["inn"][n1:], 0
    while i < inn.size:
        e = int(inn[i])
        if e < 0:
            idx.append(-e); i += 1
        else:
            p = int(inn[i + 1]); idx.append(e)
            for g in range(1, oracle_mod.pattern_size(p) + 1):
                idx.append(idx[-1] + 3 * oracle_mod.next_offset(p, g))
            i += 2
    assert idx == cpo["inn"][n1:].tolist()


def test_mac_count_density_one_and_zero(oracle_mod):
    d = layer_desc(2, 3, 9, 9, 5, 3, 3)
    x = np.ones((2, 3, 9, 9), dtype=np.float32)
    assert oracle_mod.mac_count(d, x) == 2 * 7 * 7 * 9 * 3 * 5
    assert oracle_mod.mac_count(d, np.zeros_like(x)) == 0


def test_skip_flags_dead_channels(oracle_mod):
    """50% all-zero channels encode as single NPC entries (SPEC.md acceptance 8)."""
    d = layer_desc(1, 8, 12, 12, 2, 3, 3, 1, 1, 1, 1, 1, 1)
    x = int_map(1, 8, 12, 12, 0.3, 4)
    x[:, ::2] = 0
    enc = oracle_mod.encode(d, x)
    offs = enc["chan_ptr_off"]
    for c in range(0, 8, 2):
        assert offs[c + 1] - offs[c] == 1 and enc["ptr"][offs[c]] == oracle_mod.NPC
        assert enc["chan_nz_off"][c + 1] == enc["chan_nz_off"][c]
    rho = oracle_mod.sizes.channel_density(x)
    assert enc["ptr"].size == oracle_mod.ptr_size_eq3(d, rho, oracle_mod.count_flags(enc["ptr"])[0])


def test_im2col_mec_sizes_match_eq6_eq11(oracle_mod):
    for d, rho, seed in CASES[:60]:
        x = int_map(d["N"], d["C"], d["H"], d["W"], rho, seed)
        assert oracle_mod.im2col(d, x).size == oracle_mod.S_im2col(d)
        assert oracle_mod.mec_lower(d, x).size == oracle_mod.S_mec(d)


def test_real_valued_sparse_conv_close(oracle_mod):
    d = layer_desc(2, 16, 14, 14, 8, 3, 3, 2, 2, 1, 1, 1, 1)
    x = clustered_relu(2, 16, 14, 14, 0.2, 3, dead_frac=0.25)
    w = he_normal(8, 16, 3, 3, 3)
    ref = oracle_mod.direct_conv(d, x, w)
    for cps in (False, True):
        got = oracle_mod.sparse_conv(d, oracle_mod.encode(d, x, cps=cps), w)
        np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-12)


def test_direct_conv_at_equals_direct_conv_everywhere(oracle_mod):
    """oc_direct_conv_at (Eq. 1 at chosen output coordinates) is the reference
    of the sampled GPU parity tests: over the 400-case integer sweep (strides 1/2, asymmetric
    H pads, 1x7 / 7x1 / 5x5 / 2x2 / 3x5, VALID / SAME / partial pads) it must equal the pinned
    direct_conv and the independent numpy einsum on EVERY output coordinate (all boundary
    rows / columns included), exactly; plus one real-valued case at 1e-12."""
    for d, rho, seed in CASES:
        x = int_map(d["N"], d["C"], d["H"], d["W"], rho, seed)
        w = int_weights(d["K"], d["C"], d["R"], d["S"], seed)
        ref = oracle_mod.direct_conv(d, x, w)
        idx = np.argwhere(np.ones(ref.shape, dtype=bool))          # every (n, k, y, x)
        got = oracle_mod.direct_conv_at(d, x, w, idx)
        assert np.array_equal(got, ref.reshape(-1)), d
        assert np.array_equal(got, np_conv_einsum(d, x, w).reshape(-1)), d
    d = layer_desc(3, 16, 14, 14, 8, 3, 3, 2, 2, 1, 1, 1, 1)
    x = clustered_relu(3, 16, 14, 14, 0.2, 3, dead_frac=0.25)
    w = he_normal(8, 16, 3, 3, 3)
    ref = np_conv_einsum(d, x, w)
    rng = np.random.default_rng(7)
    idx = np.stack([rng.integers(0, s, 500) for s in ref.shape], axis=1)
    np.testing.assert_allclose(oracle_mod.direct_conv_at(d, x, w, idx), ref[tuple(idx.T)], rtol=1e-12, atol=1e-13)
