"""CUDA path vs the CPU oracle, element by element, through the C ABI.

Encodings (ptr, DA bits, IN, side tables, lengths) must be bit-exact; conv
outputs within |gpu - ref| <= max(1e-4 |ref|, 1e-5) of the FP64 oracle
(BASELINE.json north_star), and exactly equal on integer-valued data.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from gpu_util import GpuLayer, assert_streams_equal  # noqa: E402
from helpers import within_tol, valid_sparse_geometry  # noqa: E402
from synth import (CATALOG, CONFIGS, cfg5_layers, clustered_relu, he_normal, int_map, int_weights,  # noqa: E402
                   layer_desc)

import paper_2104_08314_b200 as spc  # noqa: E402

KERNELS = [(3, 3, 1), (3, 3, 2), (1, 7, 1), (7, 1, 1), (4, 4, 1), (5, 5, 1), (3, 1, 1), (1, 3, 2), (2, 2, 1),
           (3, 5, 2)]


def _cases(n, seed):
    rng = np.random.default_rng(seed)
    out = []
    while len(out) < n:
        R, S, s = KERNELS[rng.integers(len(KERNELS))]
        pl = int(rng.integers(0, S)) if S > 1 else 0
        pt, pb = (int(rng.integers(0, R)) for _ in range(2))
        H = int(rng.integers(max(1, R - pt - pb), 20))
        W = int(rng.integers(max(1, 2 * S - 1 - 2 * pl), 20))
        d = layer_desc(int(rng.integers(1, 4)), int(rng.integers(1, 9)), H, W,
                       int(rng.choice([1, 5, 32, 40, 70])), R, S, s, s, pt, pb, pl, pl)
        if not valid_sparse_geometry(d):
            continue
        out.append((d, float(rng.choice([0.0, 0.05, 0.3, 0.6, 1.0])), int(rng.integers(1 << 30))))
    return out


SWEEP = _cases(80, 7)


@pytest.mark.parametrize("i", range(len(SWEEP)))
def test_sweep_integer_exact(oracle_mod, i):
    d, rho, seed = SWEEP[i]
    x = int_map(d["N"], d["C"], d["H"], d["W"], rho, seed)
    w = int_weights(d["K"], d["C"], d["R"], d["S"], seed)
    ref = oracle_mod.direct_conv(d, x, w)
    xg = torch.from_numpy(x).cuda()
    L = GpuLayer(d, w)
    for cps in (False, True):
        L.encode(xg, cps)
        assert_streams_equal(L.streams(), oracle_mod.encode(d, x, cps=cps), f"{d} cps={cps}")
        got = L.conv().cpu().numpy()
        assert np.array_equal(got, ref), f"{d} cps={cps} max err {np.abs(got - ref).max()}"
    assert np.array_equal(L.im2col(xg).cpu().numpy(), ref)


def _check_conv(got, ref, what):
    ok, err, nbad = within_tol(got, ref)
    assert ok, f"{what}: {nbad} elements out of tolerance, max abs err {err}"


def _layer_case(oracle_mod, d, x, w, full=True, samples=4000, seed=0):
    xg = torch.from_numpy(x).cuda()
    L = GpuLayer(d, w)
    outs = {}
    for cps in (False, True):
        L.encode(xg, cps)
        assert_streams_equal(L.streams(), oracle_mod.encode(d, x, cps=cps), f"cps={cps}")
        outs[cps] = L.conv().cpu().numpy()
    outs["im2col"] = L.im2col(xg).cpu().numpy()
    if full:
        ref = oracle_mod.direct_conv(d, x, w)
        for k, v in outs.items():
            _check_conv(v, ref, f"algo {k}")
    else:
        rng = np.random.default_rng(seed)
        shp = outs[False].shape
        idx = np.stack([rng.integers(0, s, samples) for s in shp], axis=1)
        ref = oracle_mod.direct_conv_at(d, x, w, idx)
        for k, v in outs.items():
            got = v[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]]
            _check_conv(got, ref, f"algo {k} (sampled)")
        # properties that hold everywhere: CPO == CPS closely, finite
        assert np.isfinite(outs[False]).all()
        _check_conv(outs[True], outs[False].astype(np.float64), "cps vs cpo")
    return outs


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg3s2"])
def test_baseline_configs_full(oracle_mod, name):
    c = CONFIGS[name]
    d = c["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"], c["dead_frac"],
                       c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    _layer_case(oracle_mod, d, x, w, full=True)


@pytest.mark.parametrize("rho", [0.05, 0.2, 0.3, 0.5])
def test_cfg3_density_sweep(oracle_mod, rho):
    c = CONFIGS["cfg3"]
    d = c["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], rho, c["seed"], c["dead_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    _layer_case(oracle_mod, d, x, w, full=False)


def test_cfg4_pair_relu_chain(oracle_mod):
    a, b = CONFIGS["cfg4a"], CONFIGS["cfg4b"]
    da, db = a["desc"], b["desc"]
    x = clustered_relu(da["N"], da["C"], da["H"], da["W"], a["density"], a["seed"], a["dead_frac"])
    w1 = he_normal(da["K"], da["C"], da["R"], da["S"], a["seed"])
    w2 = he_normal(db["K"], db["C"], db["R"], db["S"], a["seed"] + 1)
    L1 = GpuLayer(da, w1)
    L1.encode(torch.from_numpy(x).cuda())
    assert_streams_equal(L1.streams(), oracle_mod.encode(da, x), "1x7")
    y1 = L1.conv(relu=True).cpu().numpy()          # ReLU fused in the epilogue
    ref1 = np.maximum(oracle_mod.direct_conv(da, x, w1), 0.0)
    _check_conv(y1, ref1, "1x7 + relu")
    # the 7x1 layer consumes the GPU intermediate; both sides encode the same tensor
    rho = float((y1 != 0).mean())
    assert 0.2 < rho < 0.8
    _layer_case(oracle_mod, db, y1, w2, full=True)


@pytest.mark.parametrize("li", range(16))
def test_cfg5_layers_sampled(oracle_mod, li):
    layer = cfg5_layers(batch=32)[li]
    d = layer["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], layer["density"], layer["seed"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], layer["seed"])
    _layer_case(oracle_mod, d, x, w, full=False, samples=3000, seed=li)


@pytest.mark.parametrize("name", sorted(CATALOG))
def test_catalog_shapes_sampled(oracle_mod, name):
    """Every shape-catalog layer (5x5, 3x3, 1x7, 7x1, 1x3, 3x1 kernels; 112x112 maps at s1 / s2):
    encodings bit-exact, sampled outputs of CPO / CPS / im2col within tolerance."""
    c = CATALOG[name]
    d = c["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    _layer_case(oracle_mod, d, x, w, full=False, samples=2000, seed=c["seed"])


@pytest.mark.parametrize("shape", [(48, 64, 56, 56), (96, 128, 28, 28)])
def test_encoder_multi_round_tiles(oracle_mod, shape):
    """Batches whose tiles outnumber the resident CTAs (the cfg5 stack at batch 256 on one
    GPU): the encoder's persistent multi-round path must still emit the oracle's streams
    bit for bit, and the conv must stay within tolerance on sampled outputs."""
    N, C, H, W = shape
    d = layer_desc(N, C, H, W, C, 3, 3, 1, 1, 1, 1, 1, 1)
    x = clustered_relu(N, C, H, W, 0.25, 77)
    w = he_normal(C, C, 3, 3, 77)
    _layer_case(oracle_mod, d, x, w, full=False, samples=2000, seed=5)


@pytest.mark.parametrize("shape", [(12, 16, 56, 56, 64), (24, 24, 28, 28, 128)])
def test_balanced_mode_full(oracle_mod, shape, capfd, monkeypatch):
    """Grids whose units (strip, k-block, image) outnumber the SMs unevenly run in the
    balanced mode (persistent CTAs over equal-work channel ranges; a unit split between
    CTAs is summed from flag-published partials).  Full-output parity, ReLU fusion, and
    bit-identical repeats (the flags must be left zeroed for the next launch)."""
    N, C, H, W, K = shape
    d = layer_desc(N, C, H, W, K, 3, 3, 1, 1, 1, 1, 1, 1)
    x = clustered_relu(N, C, H, W, 0.3, 91, 0.05, 0.1)
    w = he_normal(K, C, 3, 3, 91)
    monkeypatch.setenv("SPC_PLAN_DEBUG", "1")
    L = GpuLayer(d, w)
    L.encode(torch.from_numpy(x).cuda())
    assert_streams_equal(L.streams(), oracle_mod.encode(d, x), "balanced")
    y1 = L.conv().cpu().numpy()
    err = capfd.readouterr().err
    assert "sk_ctas 0" not in err and "sk_ctas" in err, err
    ref = oracle_mod.direct_conv(d, x, w)
    _check_conv(y1, ref, "balanced mode")
    for _ in range(3):
        assert np.array_equal(L.conv().cpu().numpy(), y1)
    _check_conv(L.conv(relu=True).cpu().numpy(), np.maximum(ref, 0.0), "balanced mode + relu")
    # CPS: the expanded indices feed the same balanced conv
    L.encode(torch.from_numpy(x).cuda(), cps=True)
    assert_streams_equal(L.streams(), oracle_mod.encode(d, x, cps=True), "balanced cps")
    _check_conv(L.conv().cpu().numpy(), ref, "balanced mode, CPS")


def _stream_slice(enc_gpu, c0, c1):
    """GPU streams of channels [c0, c1) (global n*C + c indices) with offsets rebased to 0."""
    cp, cz, ci = (enc_gpu[k].astype(np.int64) for k in ("chan_ptr_off", "chan_nz_off", "chan_in_off"))
    return dict(ptr=enc_gpu["ptr"][cp[c0]:cp[c1]], da=enc_gpu["da"][cz[c0]:cz[c1]], inn=enc_gpu["inn"][ci[c0]:ci[c1]],
                chan_ptr_off=cp[c0:c1 + 1] - cp[c0], chan_nz_off=cz[c0:c1 + 1] - cz[c0],
                chan_in_off=ci[c0:c1 + 1] - ci[c0])


@pytest.mark.parametrize("li", [0, 8])
def test_stack_layer_full_batch(oracle_mod, li):
    """A cfg5 layer at the stack's full per-GPU batch (256 images, the size bench.py times at
    N = 1: multi-round encoder tiles, the tcgen05 GEMM over 256 x P rows).  Streams bit-exact
    for the first and the last two images (the tail checks the prefix sums at the end of the
    long stream); sampled outputs of CPO and im2col within tolerance over all 256 images."""
    from paper_2104_08314_b200.stack import tile_images
    layer = cfg5_layers(batch=256)[li]
    d = layer["desc"]
    base = clustered_relu(8, d["C"], d["H"], d["W"], layer["density"], layer["seed"])
    x = tile_images(base, 256)
    w = he_normal(d["K"], d["C"], d["R"], d["S"], layer["seed"])
    xg = torch.from_numpy(x).cuda()
    L = GpuLayer(d, w)
    L.encode(xg)
    got = L.streams()
    C = d["C"]
    for n0 in (0, 254):        # images 254, 255 repeat base images 6, 7
        d2 = dict(d, N=2)
        ref = oracle_mod.encode(d2, base[n0 % 8:n0 % 8 + 2])
        assert_streams_equal(_stream_slice(got, n0 * C, (n0 + 2) * C), ref, f"images {n0}, {n0 + 1}")
    y_cpo = L.conv().cpu().numpy()
    y_i2c = L.im2col(xg).cpu().numpy()
    rng = np.random.default_rng(li)
    idx = np.stack([rng.integers(0, s, 3000) for s in y_cpo.shape], axis=1)
    ref = oracle_mod.direct_conv_at(d, x, w, idx)
    for name, y in (("cpo", y_cpo), ("im2col", y_i2c)):
        _check_conv(y[idx[:, 0], idx[:, 1], idx[:, 2], idx[:, 3]], ref, f"L{li} batch 256 {name}")


# ------------------------------------------------------------------ edge cases

def _desc3(**kw):
    d = layer_desc(2, 6, 13, 11, 40, 3, 3, 1, 1, 1, 1, 1, 1)
    d.update(kw)
    return d


def test_all_zero_input_is_all_npc(oracle_mod):
    d = _desc3()
    x = np.zeros((2, 6, 13, 11), dtype=np.float32)
    L = GpuLayer(d, int_weights(40, 6, 3, 3, 1))
    L.encode(torch.from_numpy(x).cuda())
    s = L.streams()
    assert (s["ptr"] == spc.SPC_NPC).all() and s["ptr"].size == 12 and s["da"].size == 0
    assert not L.conv().any()


def test_density_one_and_single_corners(oracle_mod):
    d = _desc3(pad_top=0, pad_bottom=0, pad_left=0, pad_right=0)
    w = int_weights(40, 6, 3, 3, 2)
    for x in (np.ones((2, 6, 13, 11), np.float32),):
        _layer_case(oracle_mod, d, x, w)
    x = np.zeros((2, 6, 13, 11), np.float32)
    x[0, 0, 0, 0] = 3; x[0, 1, 12, 10] = 5; x[1, 5, 0, 10] = -2; x[1, 2, 12, 0] = 7
    _layer_case(oracle_mod, d, x, w)


def test_negative_zero_and_denormals(oracle_mod):
    """-0.0 is zero, a denormal is an NZE (IEEE != 0, reading A21)."""
    d = _desc3()
    x = np.zeros((2, 6, 13, 11), np.float32)
    x[0, 0, 3, 3] = -0.0
    x[0, 1, 4, 4] = np.float32(1e-40)
    x[1, 2, 5, 5] = 1.0
    L = GpuLayer(d, int_weights(40, 6, 3, 3, 2))
    L.encode(torch.from_numpy(x).cuda())
    ref = oracle_mod.encode(d, x)
    assert ref["da"].size == 2
    assert_streams_equal(L.streams(), ref)


def test_relu_fusion_and_repeat(oracle_mod):
    d = _desc3()
    x = clustered_relu(2, 6, 13, 11, 0.4, 3)
    w = he_normal(40, 6, 3, 3, 3)
    L = GpuLayer(d, w)
    xg = torch.from_numpy(x).cuda()
    first = None
    for _ in range(3):   # the encoder workspace must come back clean every launch
        L.encode(xg)
        s = L.streams()
        if first is None:
            first = s
        assert_streams_equal(s, first)
    y = L.conv(relu=True).cpu().numpy()
    _check_conv(y, np.maximum(oracle_mod.direct_conv(d, x, w), 0), "relu")


def test_capacity_overflow_reported(oracle_mod):
    d = _desc3()
    x = clustered_relu(2, 6, 13, 11, 0.5, 4)
    L = GpuLayer(d, caps=(1000, 100, 100))
    L.encode(torch.from_numpy(x).cuda())
    with pytest.raises(spc.SpcError) as e:
        spc.spc_encoding_lengths(L.enc)
    assert e.value.status == spc.SPC_ECAPACITY


def test_unsupported_geometry_raises():
    L = GpuLayer(_desc3())
    x = torch.zeros((2, 6, 13, 11), device="cuda")
    with pytest.raises(spc.SpcError) as e:
        spc.cpo_encode(_desc3(pad_left=1, pad_right=0), x, L.enc, L.ws)
    assert e.value.status == spc.SPC_EUNSUPPORTED


def test_select_layer_algo_argmin():
    c = CONFIGS["cfg1"]
    d = c["desc"]
    M = 5
    xs = np.stack([clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], s, c["dead_frac"])
                   for s in c["select_seeds"]])
    w = torch.from_numpy(he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])).cuda()
    ws = torch.empty(spc.spc_select_ws_bytes(d), dtype=torch.uint8, device="cuda")
    samples = torch.from_numpy(xs).cuda()
    for mode, allowed in ((spc.SPC_FAVOUR_TIME, {0, 1}), (spc.SPC_FAVOUR_SPACE, {0, 2}),
                          (spc.SPC_BEST_OF_THREE, {0, 1, 2})):
        choice, t = spc.select_layer_algo(d, samples, M, w, mode, 3, ws)
        assert choice in allowed and all(v > 0 for v in t)
        cand = [a for a in allowed]
        assert t[choice] <= min(t[a] for a in cand) + 1e-9
    # pointwise -> im2col, sparse times reported as -1
    dp = dict(d, R=1, S=1, pad_top=0, pad_bottom=0, pad_left=0, pad_right=0)
    ws2 = torch.empty(spc.spc_select_ws_bytes(dp), dtype=torch.uint8, device="cuda")
    wp = torch.from_numpy(he_normal(d["K"], d["C"], 1, 1, 1)).cuda()
    choice, t = spc.select_layer_algo(dp, samples, M, wp, spc.SPC_BEST_OF_THREE, 2, ws2)
    assert choice == spc.SPC_ALGO_IM2COL and t[1] == -1 and t[2] == -1


@pytest.mark.parametrize("engine", [spc.SPC_GEMM_SIMT, spc.SPC_GEMM_CUBLAS_FP32, spc.SPC_GEMM_CUBLAS_BF16X9,
                                    spc.SPC_GEMM_TC_3XTF32, spc.SPC_GEMM_AUTO])
def test_im2col_gemm_engines_within_tolerance(oracle_mod, engine):
    """Every dense-baseline GEMM engine that the selector may use meets the fp32 tolerance."""
    c = CONFIGS["cfg3"]
    d = dict(c["desc"], N=2)
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], 0.3, c["seed"], c["dead_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    ref = oracle_mod.direct_conv(d, x, w)
    L = GpuLayer(d, w)
    prev = spc.spc_get_im2col_gemm()
    try:
        spc.spc_set_im2col_gemm(engine)
        try:
            got = L.im2col(torch.from_numpy(x).cuda()).cpu().numpy()
        except spc.SpcError as e:
            if e.status == spc.SPC_EUNSUPPORTED:
                pytest.skip(str(e))
            raise
        _check_conv(got, ref, f"gemm engine {spc.GEMM_NAMES[engine]}")
        got_relu = L.im2col(torch.from_numpy(x).cuda(), relu=True).cpu().numpy()
        _check_conv(got_relu, np.maximum(ref, 0.0), f"gemm engine {engine} + relu")
    finally:
        spc.spc_set_im2col_gemm(prev)


def test_tc_gemm_minimal_workspace(oracle_mod):
    """With only the lowered matrix as workspace (4 * S_im2col) the tcgen05 engine splits the
    weights per tile in shared memory instead of once into the workspace tail: same tolerance."""
    d = layer_desc(2, 256, 14, 14, 256, 3, 3, 1, 1, 1, 1, 1, 1)
    x = clustered_relu(2, 256, 14, 14, 0.3, 13)
    w = he_normal(256, 256, 3, 3, 13)
    ref = oracle_mod.direct_conv(d, x, w)
    prev = spc.spc_get_im2col_gemm()
    try:
        spc.spc_set_im2col_gemm(spc.SPC_GEMM_TC_3XTF32)
        Oh, Ow = spc.out_hw(d)
        ws = torch.empty(2 * 256 * 9 * Oh * Ow, dtype=torch.float32, device="cuda")
        assert 4 * ws.numel() < spc.spc_im2col_ws_bytes(d)
        y = torch.empty((2, 256, Oh, Ow), dtype=torch.float32, device="cuda")
        spc.im2col_conv_forward(d, torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda(), y, False, ws)
        _check_conv(y.cpu().numpy(), ref, "tc 3xtf32, minimal workspace")
    finally:
        spc.spc_set_im2col_gemm(prev)


def test_im2col_tf32_engine_runs():
    """The 1-term TF32 engine is a crossover reference only: it must run, not meet 1e-4."""
    d = layer_desc(1, 16, 14, 14, 16, 3, 3, 1, 1, 1, 1, 1, 1)
    x = int_map(1, 16, 14, 14, 0.3, 5)
    w = int_weights(16, 16, 3, 3, 5)
    L = GpuLayer(d, w)
    prev = spc.spc_get_im2col_gemm()
    try:
        spc.spc_set_im2col_gemm(spc.SPC_GEMM_CUBLAS_TF32)
        got = L.im2col(torch.from_numpy(x).cuda()).cpu().numpy()
        assert np.isfinite(got).all()
    finally:
        spc.spc_set_im2col_gemm(prev)
    with pytest.raises(spc.SpcError):
        spc.spc_set_im2col_gemm(7)


@pytest.mark.parametrize("shape", [(1, 64, 56, 56, 64, 1), (2, 256, 14, 14, 256, 1), (2, 128, 28, 28, 128, 2),
                                   (1, 5, 9, 11, 70, 1), (2, 3, 17, 17, 33, 1), (3, 512, 7, 7, 512, 1),
                                   (3, 4, 9, 11, 70, 1), (5, 8, 13, 10, 200, 2),
                                   (2, 64, 16, 16, 64, 1), (2, 256, 16, 16, 256, 1)])   # M, CRS tile exactly
def test_tc_gemm_3xtf32_shapes(oracle_mod, shape):
    """tcgen05 3xTF32 baseline GEMM vs the FP64 oracle on ragged shapes (P, K, CRS not tile
    multiples; CRS % 4 != 0 runs the cuBLAS FP32 fallback).  The TMEM accumulator is drained into
    fp32 register sums every 256 CRS, which keeps CRS = 4608 (512 channels) inside the strict
    north_star tolerance too (one tensor-core accumulation over all of CRS left ~2e-5 absolute
    error on near-zero outputs)."""
    N, C, H, W, K, s = shape
    d = layer_desc(N, C, H, W, K, 3, 3, s, s, 1, 1, 1, 1)
    x = clustered_relu(N, C, H, W, 0.3, 11)
    w = he_normal(K, C, 3, 3, 11)
    ref = oracle_mod.direct_conv(d, x, w)
    L = GpuLayer(d, w)
    prev = spc.spc_get_im2col_gemm()
    try:
        spc.spc_set_im2col_gemm(spc.SPC_GEMM_TC_3XTF32)
        got = L.im2col(torch.from_numpy(x).cuda()).cpu().numpy()
    finally:
        spc.spc_set_im2col_gemm(prev)
    _check_conv(got, ref, f"tc 3xtf32 {shape}")


# ------------------------------------------------ warp-specialised conv (v2) configurations

@pytest.mark.parametrize("shape", [
    (2, 40, 14, 14, 256, 1),     # 14x14 @ 256, s1: 2x4 tiles x 4 channels per lane, cluster split
    (3, 24, 7, 7, 512, 1),       # 7x7 @ 512, s1: 4x4 tiles x 2 channels per lane, 8 k-groups
    (2, 20, 14, 14, 512, 2),     # 14 -> 7 @ 512, s2
    (2, 36, 28, 28, 256, 2),     # 28 -> 14 @ 256, s2
    (1, 300, 14, 14, 256, 1),    # many chunks (NST-stage ring wraps several times), ragged last chunk
])
@pytest.mark.parametrize("rho", [0.0, 0.07, 0.4, 1.0])
@pytest.mark.parametrize("cps", [False, "expand", "inline"])
def test_ws_conv_integer_exact(oracle_mod, shape, rho, cps):
    """The warp-specialised conv (ws_conv.cuh) against the oracle's Eq. 1 on integer data:
    every output element exactly equal (ragged chunks, all-zero and dense maps, cluster split).
    CPS encodings: "expand" = the separate Alg. 4 expansion pass, "inline" = the producers decode
    the CPS stream themselves (Alg. 4) -- from shared memory, or through the
    workspace for chunks beyond the stage (rho = 1.0)."""
    N, C, H, W, K, s = shape
    d = layer_desc(N, C, H, W, K, 3, 3, s, s, 1, 1, 1, 1)
    x = int_map(N, C, H, W, rho, 1000 + C)
    x[:, ::7] = 0                                   # some NPC channels
    w = int_weights(K, C, 3, 3, 7)
    L = GpuLayer(d, w)
    L.encode(torch.from_numpy(x).cuda(), bool(cps))
    prev = spc.spc_get_cps_inline()
    try:
        spc.spc_set_cps_inline(cps == "inline")
        y = L.conv().cpu().numpy()
    finally:
        spc.spc_set_cps_inline(prev)
    assert spc.spc_last_conv_kernel() == 2          # the warp-specialised kernel ran
    ref = oracle_mod.direct_conv(d, x, w)
    assert np.array_equal(y, ref.astype(np.float32)), np.abs(y - ref).max()
