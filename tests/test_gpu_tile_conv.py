"""Parity of the register-tiled conv (tile_conv_kernel, opt-in development switch SPC_TC=1,
DESIGN.md §7): the same Alg. 2 convSpMv as the default kernels, so on
integer data (every product and partial sum exact in fp32) its output must equal the oracle's
direct convolution (Eq. 1) exactly -- CPO and CPS encodings, ReLU fused, cluster channel split,
several pairs per CTA touching two images, ragged tiles and channel chunks.  The switch is read
once per process, so the checks run in a child process."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np, torch
sys.path.insert(0, sys.argv[1]); sys.path.insert(0, sys.argv[1] + "/tests")
import oracle
import paper_2104_08314_b200 as spc
from gpu_util import GpuLayer
from synth import int_map, int_weights, layer_desc
oracle.build()
out = []
shapes = [(2, 256, 14, 14, 256, 0.1), (3, 128, 28, 28, 128, 0.2), (8, 512, 7, 7, 512, 0.3),
          (1, 64, 56, 56, 64, 0.3), (2, 30, 13, 11, 64, 0.4), (5, 9, 14, 14, 128, 0.5)]
for i, (N, C, H, W, K, rho) in enumerate(shapes):
    d = layer_desc(N, C, H, W, K, 3, 3, 1, 1, 1, 1, 1, 1)
    x = int_map(N, C, H, W, rho, 40 + i)
    w = int_weights(K, C, 3, 3, 40 + i)
    ref = oracle.direct_conv(d, x, w)
    for cps in (False, True):
        L = GpuLayer(d, w)
        L.encode(torch.from_numpy(x).cuda(), cps)
        for relu in (False, True):
            L.y.fill_(float("nan"))
            y = L.conv(relu).cpu().numpy().astype(np.float64)
            want = np.maximum(ref, 0) if relu else ref
            out.append(dict(shape=[N, C, H, W, K], cps=cps, relu=relu, kernel=spc.spc_last_conv_kernel(),
                            exact=bool(np.array_equal(y, want)), maxerr=float(np.nanmax(np.abs(y - want)))))
print(json.dumps(out))
"""


@pytest.mark.gpu
def test_tile_conv_exact_on_integer_data():
    env = dict(os.environ, SPC_TC="1")
    r = subprocess.run([sys.executable, "-c", CHILD, ROOT], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    rows = json.loads(r.stdout.strip().splitlines()[-1])
    assert len(rows) == 24
    for row in rows:
        assert row["kernel"] == 3, row          # the register-tiled kernel ran
        assert row["exact"], row
