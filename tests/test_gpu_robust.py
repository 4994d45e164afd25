"""Robustness of the CUDA path: the debug stream validator
(spc_validate_encoding, SPC_ECORRUPT; SPEC.md:295 / :713) accepts every encoding the
encoder emits and rejects corrupted ones; a convolution over an encoding the encoder
flagged (capacity overflow) writes zeros instead of indexing incomplete streams."""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from gpu_util import GpuLayer  # noqa: E402
from synth import CONFIGS, cfg5_layers, clustered_relu, he_normal, int_map, int_weights, layer_desc  # noqa: E402

import paper_2104_08314_b200 as spc  # noqa: E402


def _scratch():
    return torch.empty(64, dtype=torch.uint8, device="cuda")


def _cases():
    out = [(CONFIGS[n]["desc"], CONFIGS[n]) for n in ("cfg1", "cfg2", "cfg3", "cfg3s2")]
    for li in (0, 3, 8, 14):
        sp = cfg5_layers(batch=4)[li]
        out.append((sp["desc"], sp))
    return out


@pytest.mark.parametrize("cps", [False, True])
@pytest.mark.parametrize("i", range(8))
def test_validator_accepts_encoder_output(i, cps):
    d, c = _cases()[i]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"], c.get("dead_frac", 0.0),
                       c.get("zero_tile_frac", 0.0))
    L = GpuLayer(d)
    L.encode(torch.from_numpy(x).cuda(), cps=cps)
    spc.spc_validate_encoding(d, L.enc, _scratch())


@pytest.mark.parametrize("geom", [(3, 3, 1, 1), (3, 3, 0, 0), (1, 7, 0, 3), (7, 1, 3, 0), (4, 4, 0, 0), (5, 5, 2, 2)])
def test_validator_accepts_small_geometries(geom):
    R, S, pv, ph = geom
    d = layer_desc(2, 5, 13, 12, 8, R, S, 1, 1, pv, pv, ph, ph)
    for rho in (0.0, 0.1, 0.6, 1.0):
        x = int_map(2, 5, 13, 12, rho, 3)
        for cps in (False, True):
            L = GpuLayer(d)
            L.encode(torch.from_numpy(x).cuda(), cps=cps)
            spc.spc_validate_encoding(d, L.enc, _scratch())


def _corrupt_and_check(L, d, mutate):
    mutate(L.enc)
    torch.cuda.synchronize()
    with pytest.raises(spc.SpcError) as e:
        spc.spc_validate_encoding(d, L.enc, _scratch())
    assert e.value.status == spc.SPC_ECORRUPT, str(e.value)


MUTATIONS = {
    # a ptr count made to decrease inside a block
    "ptr_count": lambda e: e.ptr.__setitem__(3, e.ptr[2] + 1000),
    # a block tag changed
    "ptr_tag": lambda e: e.ptr.__setitem__(0, 9),
    # an IN entry moved outside the padded rows
    "in_row": lambda e: e.inn.__setitem__(0, 10_000),
    # an IN entry with the wrong local column
    "in_local": lambda e: e.inn.__setitem__(1, e.inn[1] + 1),
    # a DA value zeroed
    "da_zero": lambda e: e.da.__setitem__(2, 0.0),
    # a DA value made NaN
    "da_nan": lambda e: e.da.__setitem__(3, float("nan")),
    # a side-table offset shifted
    "side": lambda e: e.chan_nz_off.__setitem__(1, e.chan_nz_off[1] + 1),
}


@pytest.mark.parametrize("what", sorted(MUTATIONS))
def test_validator_rejects_corruption(what):
    d = layer_desc(1, 4, 12, 12, 8, 3, 3, 1, 1, 1, 1, 1, 1)
    x = int_map(1, 4, 12, 12, 0.5, 11)
    L = GpuLayer(d)
    L.encode(torch.from_numpy(x).cuda())
    spc.spc_validate_encoding(d, L.enc, _scratch())
    _corrupt_and_check(L, d, MUTATIONS[what])


def test_validator_rejects_bad_cps_pattern():
    d = layer_desc(1, 1, 16, 10, 4, 3, 3, 1, 1, 1, 1, 1, 1)
    x = np.zeros((1, 1, 16, 10), np.float32)
    x[0, 0, 3:6, 4] = [1, 2, 3]        # padded rows 4..6 of one column: {index, pattern 7}
    L = GpuLayer(d)
    L.encode(torch.from_numpy(x).cuda(), cps=True)
    spc.spc_validate_encoding(d, L.enc, _scratch())
    ii = L.enc.inn[:2].cpu().numpy()
    assert ii[0] >= 0 and ii[1] == 7
    _corrupt_and_check(L, d, lambda e: e.inn.__setitem__(1, 3))   # a 2-bit "pattern"


def test_conv_over_flagged_encoding_writes_zeros():
    """An encoding whose capacities overflowed is flagged on the device (overflow word);
    the convolution then writes y = 0 instead of reading incomplete streams, and the
    host-side length query reports SPC_ECAPACITY."""
    d = layer_desc(2, 6, 13, 11, 40, 3, 3, 1, 1, 1, 1, 1, 1)
    x = clustered_relu(2, 6, 13, 11, 0.5, 4)
    L = GpuLayer(d, he_normal(40, 6, 3, 3, 4), caps=(1000, 100, 100))
    L.encode(torch.from_numpy(x).cuda())
    L.y.fill_(123.0)
    y = L.conv().cpu().numpy()
    assert not y.any()
    with pytest.raises(spc.SpcError) as e:
        spc.spc_encoding_lengths(L.enc)
    assert e.value.status == spc.SPC_ECAPACITY
    # re-encoding into a large enough encoding clears bit 0 and the conv is live again
    L2 = GpuLayer(d, he_normal(40, 6, 3, 3, 4))
    L2.enc.lengths.fill_(1)
    L2.encode(torch.from_numpy(x).cuda())
    assert L2.conv().abs().sum().item() > 0


@pytest.mark.parametrize("shape", [(1, 256, 14, 14, 256, 1), (1, 128, 28, 28, 256, 2), (1, 512, 7, 7, 512, 1)])
def test_conv_without_workspace_on_cluster_shapes(oracle_mod, shape):
    """Warp-specialised conv shapes whose plan splits the input channels over a cluster when a
    workspace (L2 partials) is given: without one the launch falls back to one CTA per unit and
    must size its shared memory for all the channels (round 2 regression: the side tables were
    sized for the split, the barriers landed outside the allocation).  CPO and the stride-aware
    layout, integer data, exact."""
    N, C, H, W, K, st = shape
    d = layer_desc(N, C, H, W, K, 3, 3, st, st, 1, 1, 1, 1)
    x = int_map(N, C, H, W, 0.2, 17)
    w = int_weights(K, C, 3, 3, 17)
    ref = oracle_mod.direct_conv(d, x, w).astype(np.float32)
    xg, wg = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    wp = torch.empty_like(wg).reshape(-1)
    spc.spc_pack_weights(d, wg, wp)
    Oh, Ow = spc.spc_output_dims(d)
    ws = spc.alloc_workspace(d)
    for strided in (False, True):
        enc = spc.alloc_strided_encoding(d) if strided else spc.alloc_encoding(d)
        if strided:
            spc.cpo_encode_strided(d, xg, enc, ws)
        else:
            spc.cpo_encode(d, xg, enc, ws)
        for conv_ws in (None, ws):
            y = torch.full((N, K, Oh, Ow), float("nan"), device="cuda")
            spc.sparse_conv_forward(d, enc, wp, y, False, conv_ws)
            assert np.array_equal(y.cpu().numpy(), ref), (strided, conv_ws is None)


def test_last_conv_kernel_reports_the_launch():
    """spc_last_conv_kernel names the kernel the last sparse conv launched (bench's roofline label):
    the warp-specialised kernel on cfg3's 14x14 @ 256 layer, the strip kernel on cfg2's 56x56 @ 64."""
    for name, kind in (("cfg3", 2), ("cfg2", 1)):
        d = CONFIGS[name]["desc"]
        x = clustered_relu(d["N"], d["C"], d["H"], d["W"], 0.1, 3)
        L = GpuLayer(d, he_normal(d["K"], d["C"], 3, 3, 3))
        L.encode(torch.from_numpy(x).cuda())
        L.conv()
        torch.cuda.synchronize()
        assert spc.spc_last_conv_kernel() == kind, (name, spc.spc_last_conv_kernel())


FLAGGED_BALANCED_CHILD = r"""
import sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
from gpu_util import GpuLayer
from synth import clustered_relu, he_normal, layer_desc
d = layer_desc(12, 16, 56, 56, 64, 3, 3, 1, 1, 1, 1, 1, 1)
x = clustered_relu(12, 16, 56, 56, 0.3, 91, 0.05, 0.1)
L = GpuLayer(d, he_normal(64, 16, 3, 3, 91), caps=(100000, 1000, 1000))
L.encode(torch.from_numpy(x).cuda())
L.y.fill_(123.0)
y = L.conv().cpu().numpy()
print("zeros" if not y.any() else "nonzero")
"""


def test_flagged_encoding_through_balanced_mode():
    """A flagged (overflowed) encoding on a shape that runs the balanced strip kernel
    (persistent CTAs over equal-work channel ranges): every segment is walked as empty and
    y = 0 -- round 2 regression: a flagged segment did not advance the CTA's work range, so
    the kernel spun on the same segment.  Runs in a child process with a timeout."""
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-c", FLAGGED_BALANCED_CHILD, root], capture_output=True, text=True,
                       timeout=180, env=dict(os.environ, SPC_PLAN_DEBUG="1"))
    assert r.returncode == 0, r.stderr[-2000:]
    assert "sk_ctas 0" not in r.stderr and "sk_ctas" in r.stderr, r.stderr[-2000:]   # the balanced mode ran
    assert r.stdout.strip().endswith("zeros"), r.stdout
