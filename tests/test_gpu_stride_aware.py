"""Stride-aware CPO layout on the GPU (cpo_encode_strided + sparse_conv_forward; reading A32,
SI Eq. 2) against the oracle (oracle.encode_sa / sparse_conv_sa, pinned in
tests/test_oracle_stride_aware.py): streams bit-exact, outputs exact on integer data.  Both encoders:
the single-pass one (a workspace given: the canonical encoder's kernel with the layout's column
order and blocks) and the three-launch one (no workspace)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from helpers import within_tol  # noqa: E402
from synth import CONFIGS, cfg5_layers, clustered_relu, he_normal, int_map, int_weights, layer_desc  # noqa: E402

import paper_2104_08314_b200 as spc  # noqa: E402


def run_gpu(d, x, w, one_pass=True):
    enc = spc.alloc_strided_encoding(d)
    xg = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    spc.cpo_encode_strided(d, xg, enc, spc.alloc_workspace(d) if one_pass else None)
    wg = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    wp = torch.empty_like(wg).reshape(-1)
    spc.spc_pack_weights(d, wg, wp)
    Oh, Ow = spc.spc_output_dims(d)
    y = torch.empty((d["N"], d["K"], Oh, Ow), dtype=torch.float32, device="cuda")
    spc.sparse_conv_forward(d, enc, wp, y)
    p, a, i = spc.spc_encoding_lengths(enc)
    s = dict(ptr=enc.ptr[:p].cpu().numpy(), da=enc.da[:a].cpu().numpy(), inn=enc.inn[:i].cpu().numpy(),
             chan_ptr_off=enc.chan_ptr_off.cpu().numpy(), chan_nz_off=enc.chan_nz_off.cpu().numpy())
    return s, y.cpu().numpy()


def check_streams(s, ref):
    for k in ("ptr", "inn", "chan_ptr_off", "chan_nz_off"):
        assert np.array_equal(s[k], ref[k]), k
    assert np.array_equal(s["da"].view(np.int32), ref["da"].view(np.int32))


GEOMS = [(3, 3, 2, 1), (3, 3, 2, 0), (5, 5, 2, 2), (1, 7, 3, 3), (3, 5, 2, 1), (2, 2, 2, 0), (4, 4, 3, 1), (3, 3, 1, 1)]


@pytest.mark.parametrize("one_pass", [True, False])
@pytest.mark.parametrize("gi", range(len(GEOMS)))
@pytest.mark.parametrize("rho", [0.0, 0.1, 0.5, 1.0])
def test_strided_integer_exact(oracle_mod, gi, rho, one_pass):
    R, S, st, pad = GEOMS[gi]
    pv, ph = min(pad, R - 1), min(pad, S - 1)
    d = layer_desc(2, 6, 15, 17, 70, R, S, st, st, pv, pv, ph, ph)
    x = int_map(2, 6, 15, 17, rho, 41 + gi)
    x[:, 1] = 0
    w = int_weights(70, 6, R, S, gi)
    s, y = run_gpu(d, x, w, one_pass)
    check_streams(s, oracle_mod.encode_sa(d, x))
    assert np.array_equal(y, oracle_mod.direct_conv(d, x, w).astype(np.float32))


@pytest.mark.parametrize("name", ["cfg3s2", "L03", "L07", "L13"])
def test_strided_paper_shapes(oracle_mod, name):
    if name == "cfg3s2":
        c = CONFIGS[name]
    else:
        c = cfg5_layers(batch=2)[int(name[1:])]
    d = dict(c["desc"])
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"], c.get("dead_frac", 0.0),
                       c.get("zero_tile_frac", 0.0))
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    s, y = run_gpu(d, x, w)
    ref = oracle_mod.encode_sa(d, x)
    check_streams(s, ref)
    ok, worst, nbad = within_tol(y, oracle_mod.direct_conv(d, x, w))
    assert ok, (worst, nbad)
    agn = oracle_mod.encode(d, x)
    assert s["ptr"].size < 0.6 * agn["ptr"].size          # about half the ptr of the stride-1 layout


@pytest.mark.parametrize("shape", [(48, 64, 56, 56, 2), (96, 128, 28, 28, 2), (64, 96, 29, 31, 3)])
def test_strided_single_pass_multi_round(oracle_mod, shape):
    """Batches whose encoder tiles outnumber the resident CTAs (several rounds of the single-pass
    encoder), odd sizes with columns no partition covers: streams equal the oracle's and the
    three-launch encoder's, bit for bit."""
    N, C, H, W, st = shape
    d = layer_desc(N, C, H, W, 8, 3, 3, st, st, 1, 1, 1, 1)
    x = clustered_relu(N, C, H, W, 0.25, 78)
    xg = torch.from_numpy(x).cuda()
    out = []
    for ws in (spc.alloc_workspace(d), None):
        enc = spc.alloc_strided_encoding(d)
        spc.cpo_encode_strided(d, xg, enc, ws)
        p, a, i = spc.spc_encoding_lengths(enc)
        out.append(dict(ptr=enc.ptr[:p].cpu().numpy(), da=enc.da[:a].cpu().numpy(), inn=enc.inn[:i].cpu().numpy(),
                        chan_ptr_off=enc.chan_ptr_off.cpu().numpy(), chan_nz_off=enc.chan_nz_off.cpu().numpy()))
    check_streams(out[0], out[1])
    check_streams(out[0], oracle_mod.encode_sa(d, x))
