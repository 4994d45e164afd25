"""CSCC baseline on the GPU (cscc.cu, C ABI cscc_encode / cscc_conv_forward) against the
oracle (oracle.cscc_encode / cscc_conv, pinned in tests/test_oracle_cscc.py): streams and side
tables bit-exact, outputs exact on integer data and within the 1e-4 / 1e-5 tolerance on real
data (SI Alg. 5/6; SI Eq. 17)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from helpers import within_tol  # noqa: E402
from synth import CONFIGS, cfg5_layers, clustered_relu, he_normal, int_map, int_weights, layer_desc  # noqa: E402

import paper_2104_08314_b200 as spc  # noqa: E402

GEOMS = [(3, 3, 1, 1), (3, 3, 2, 1), (1, 7, 1, 0), (7, 1, 1, 0), (5, 5, 1, 2), (3, 3, 1, 0), (2, 2, 2, 0),
         (1, 1, 1, 0), (3, 5, 2, 1)]


def run_gpu(d, x, w):
    enc = spc.alloc_cscc_encoding(d)
    xg = torch.from_numpy(np.ascontiguousarray(x)).cuda()
    spc.cscc_encode(d, xg, enc)
    wg = torch.from_numpy(np.ascontiguousarray(w)).cuda()
    wp = torch.empty_like(wg).reshape(-1)
    spc.spc_pack_weights(d, wg, wp)
    Oh, Ow = spc.spc_output_dims(d)
    y = torch.empty((d["N"], d["K"], Oh, Ow), dtype=torch.float32, device="cuda")
    spc.cscc_conv_forward(d, enc, wp, y)
    p, a, i = spc.spc_encoding_lengths(enc)
    s = dict(ptr=enc.ptr[:p].cpu().numpy(), da=enc.da[:a].cpu().numpy(), inn=enc.inn[:i].cpu().numpy(),
             chan_ptr_off=enc.chan_ptr_off.cpu().numpy(), chan_nz_off=enc.chan_nz_off.cpu().numpy())
    return s, y.cpu().numpy()


def check_streams(s, ref):
    for k in ("ptr", "inn", "chan_ptr_off", "chan_nz_off"):
        assert np.array_equal(s[k], ref[k]), k
    assert np.array_equal(s["da"].view(np.int32), ref["da"].view(np.int32))


@pytest.mark.parametrize("gi", range(len(GEOMS)))
@pytest.mark.parametrize("rho", [0.0, 0.1, 0.5, 1.0])
def test_cscc_integer_exact(oracle_mod, gi, rho):
    R, S, st, pad = GEOMS[gi]
    pv, ph = min(pad, R - 1), min(pad, S - 1)
    d = layer_desc(2, 5, 15, 13, 70, R, S, st, st, pv, pv, ph, ph)
    x = int_map(2, 5, 15, 13, rho, 31 + gi)
    w = int_weights(70, 5, R, S, gi)
    s, y = run_gpu(d, x, w)
    check_streams(s, oracle_mod.cscc_encode(d, x))
    assert np.array_equal(y, oracle_mod.direct_conv(d, x, w).astype(np.float32))


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg3s2", "cfg4a"])
def test_cscc_baseline_configs(oracle_mod, name):
    c = CONFIGS[name]
    d = dict(c["desc"])
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    s, y = run_gpu(d, x, w)
    check_streams(s, oracle_mod.cscc_encode(d, x))
    ok, worst, nbad = within_tol(y, oracle_mod.direct_conv(d, x, w))
    assert ok, (worst, nbad)


def test_cscc_eq17_size_and_capacity_flag(oracle_mod):
    d = layer_desc(3, 8, 14, 14, 16, 3, 3, 1, 1, 1, 1, 1, 1)
    x = clustered_relu(3, 8, 14, 14, 0.3, 5)
    s, _ = run_gpu(d, x, he_normal(16, 8, 3, 3, 5))
    rh = oracle_mod.rho_hat(d, s["da"].size)
    assert abs(s["ptr"].size + 2 * s["da"].size - oracle_mod.S_cscc_eq17(d, rh)) < 1e-6 * s["da"].size
    enc = spc.alloc_cscc_encoding(d, caps=(10, 10, 10))
    spc.cscc_encode(d, torch.from_numpy(x).cuda(), enc)
    with pytest.raises(spc.SpcError) as e:
        spc.spc_encoding_lengths(enc)
    assert e.value.status == spc.SPC_ECAPACITY
