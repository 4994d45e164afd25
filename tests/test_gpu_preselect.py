"""The SI space pre-selector (spc_space_preselect / spc_space_bound) checked
against REAL GPU encodings: whenever it predicts CPO no larger than the im2col lowered matrix
(resp. CSCC's lowered matrix), the lengths the GPU encoder reports confirm it (SURVEY.md §8(f)
NEXT-3); and the CSCC bound is the exact crossover of the worst-case sizes."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA GPU", allow_module_level=True)

from gpu_util import GpuLayer  # noqa: E402
from synth import CATALOG, cfg5_layers, clustered_relu, layer_desc  # noqa: E402

import paper_2104_08314_b200 as spc  # noqa: E402
from paper_2104_08314_b200.bounds import space_preselect  # noqa: E402

SHAPES = ([sp["desc"] for sp in cfg5_layers(batch=2)[::3]] + [dict(CATALOG[k]["desc"], N=2) for k in CATALOG] +
          [layer_desc(2, 16, 14, 14, 8, 3, 3, 1, 1, 0, 0, 0, 0), layer_desc(2, 16, 9, 30, 8, 1, 7, 1, 1, 0, 0, 0, 0)])


@pytest.mark.parametrize("i", range(len(SHAPES)))
def test_preselector_agrees_with_gpu_sizes(i):
    d = dict(SHAPES[i])
    if d["H"] * d["W"] > 112 * 112:
        d["N"] = 1
    Oh, Ow = spc.spc_output_dims(d)
    s_i2c = d["N"] * Oh * Ow * d["C"] * d["R"] * d["S"]
    for rho in (0.02, 0.1, 0.3, 0.6, 0.95):
        x = clustered_relu(d["N"], d["C"], d["H"], d["W"], rho, 77 + i)
        xg = torch.from_numpy(x).cuda()
        L = GpuLayer(d).encode(xg)
        s_cpo = sum(spc.spc_encoding_lengths(L.enc))
        rbar = float((x != 0).mean())
        if space_preselect(d, rbar, "im2col") == "cpo":
            assert s_cpo <= s_i2c, (d, rho, s_cpo, s_i2c)
        if d["stride_w"] == 1:
            enc = spc.alloc_cscc_encoding(d)
            spc.cscc_encode(d, xg, enc)
            p, a, q = spc.spc_encoding_lengths(enc)
            Hp = d["H"] + d["pad_top"] + d["pad_bottom"]
            rh_bar = a / float(Ow * d["S"] * Hp * d["C"]) / d["N"]
            if space_preselect(d, rbar, "cscc", rh_bar) == "cpo":
                assert s_cpo <= p + a + q, (d, rho, s_cpo, p + a + q)
