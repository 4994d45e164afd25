"""NEXT-1: the convolution emits its output already CPO-encoded for the next layer
(sparse_conv_encode_forward).  The emitted encoding must be bit-identical to the oracle's
encoding (Alg. 1) of the same GPU intermediate, and to the stand-alone GPU encoder's; layer 2
consuming it gives the same outputs as layer 2 after a separate encode."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from gpu_util import GpuLayer, assert_streams_equal  # noqa: E402
from helpers import within_tol  # noqa: E402
from synth import CONFIGS, clustered_relu, he_normal, int_map, int_weights, layer_desc  # noqa: E402

import paper_2104_08314_b200 as spc  # noqa: E402


def enc_streams(enc):
    p, a, i = spc.spc_encoding_lengths(enc)
    return dict(ptr=enc.ptr[:p].cpu().numpy(), da=enc.da[:a].cpu().numpy(), inn=enc.inn[:i].cpu().numpy(),
                chan_ptr_off=enc.chan_ptr_off.cpu().numpy(), chan_nz_off=enc.chan_nz_off.cpu().numpy(),
                chan_in_off=enc.chan_in_off.cpu().numpy())


def run_chain(oracle_mod, d1, d2, x, w1, w2, relu=True, reps=2):
    L1 = GpuLayer(d1, w1)
    L1.encode(torch.from_numpy(x).cuda())
    out = spc.alloc_encoding(d2)
    ws = spc.alloc_fused_workspace(d1)
    for _ in range(reps):     # the masks must come back zeroed for the next launch
        spc.sparse_conv_encode_forward(d1, L1.enc, L1.wp, L1.y, relu, d2, out, ws)
        fused = enc_streams(out)
    y1 = L1.y.cpu().numpy()
    # bit-exact vs the oracle's Alg. 1 on the same GPU intermediate
    assert_streams_equal(fused, oracle_mod.encode(d2, y1), "fused vs oracle")
    # and vs the stand-alone GPU encoder
    L2 = GpuLayer(d2, w2)
    L2.encode(L1.y)
    assert_streams_equal(fused, L2.streams(), "fused vs cpo_encode")
    # layer 2 from the fused encoding == layer 2 after a separate encode; within tolerance of Eq. 1
    yb = L2.conv().clone()
    L2.enc = out
    ya = L2.conv()
    assert torch.equal(ya, yb)
    return y1, ya.cpu().numpy()


def test_cfg4_chain_fused(oracle_mod):
    """cfg4 (BASELINE.json configs[3]): 1x7 (pad 0,3) -> ReLU -> 7x1 (pad 3,0), batch 8, 192 ch."""
    a, b = CONFIGS["cfg4a"], CONFIGS["cfg4b"]
    d1, d2 = a["desc"], b["desc"]
    x = clustered_relu(d1["N"], d1["C"], d1["H"], d1["W"], a["density"], a["seed"], a["dead_frac"])
    w1 = he_normal(d1["K"], d1["C"], 1, 7, a["seed"])
    w2 = he_normal(d2["K"], d2["C"], 7, 1, b["seed"] + 1)
    y1, y2 = run_chain(oracle_mod, d1, d2, x, w1, w2)
    ok, worst, nbad = within_tol(y2, oracle_mod.direct_conv(d2, y1, w2))
    assert ok, (worst, nbad)


@pytest.mark.parametrize("chain", [
    ((2, 40, 14, 14, 256, 3, 3, 1, 1, 1), (3, 3, 1, 1, 1)),   # warp-specialised conv -> 3x3
    ((1, 64, 56, 56, 64, 3, 3, 1, 1, 1), (3, 3, 1, 1, 1)),    # strip kernel, cluster split
    ((2, 32, 28, 28, 128, 3, 3, 2, 2, 1), (3, 3, 1, 1, 1)),   # stride-2 layer feeding a 3x3
    ((2, 16, 17, 17, 48, 1, 7, 1, 0, 3), (7, 1, 1, 3, 0)),    # asymmetric pair
    ((2, 8, 13, 11, 20, 3, 3, 1, 0, 0), (4, 4, 1, 0, 0)),     # VALID -> NOP blocks
])
@pytest.mark.parametrize("relu", [True, False])
def test_fused_chains_integer(oracle_mod, chain, relu):
    (N, C, H, W, K, R, S, st, pv, ph), (R2, S2, st2, pv2, ph2) = chain
    d1 = layer_desc(N, C, H, W, K, R, S, st, st, pv, pv, ph, ph)
    Oh, Ow = spc.spc_output_dims(d1)
    d2 = layer_desc(N, K, Oh, Ow, 24, R2, S2, st2, st2, pv2, pv2, ph2, ph2)
    x = int_map(N, C, H, W, 0.3, 5 + C)
    w1 = int_weights(K, C, R, S, 3)
    w2 = int_weights(24, K, R2, S2, 4)
    y1, y2 = run_chain(oracle_mod, d1, d2, x, w1, w2, relu=relu)
    ref1 = oracle_mod.direct_conv(d1, x, w1)
    assert np.array_equal(y1, (np.maximum(ref1, 0) if relu else ref1).astype(np.float32))
    assert np.array_equal(y2, oracle_mod.direct_conv(d2, y1, w2).astype(np.float32))
