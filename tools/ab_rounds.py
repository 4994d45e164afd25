"""Encode / conv device times of one tree's library (development A/B between builds).

  python tools/ab_rounds.py <tree root> cfg5L0 cfg5L4 ...  (prints one JSON line per workload)
Graph-captured encode and conv separately, L2 flushed before every rep, median of 30.
"""
import json
import sys

root = sys.argv[1]
sys.path.insert(0, root)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from bench import workload  # noqa: E402
from paper_2104_08314_b200.layer import SparseConvLayer  # noqa: E402
from synth import clustered_relu, he_normal  # noqa: E402

flush = torch.empty(64 * 2 ** 20, device="cuda")


def timed(gr, n=30):
    for _ in range(3):
        gr.replay()
    ts = []
    for _ in range(n):
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); gr.replay(); b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b) * 1e3)
    return round(float(np.median(ts)), 2)


for wl in sys.argv[2:]:
    name, _, rho = wl.partition("@")
    c = workload(name)
    d = c["desc"]
    dens = float(rho) if rho else (c["density"] or 0.3)
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], dens, c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    L = SparseConvLayer(d, torch.from_numpy(w).cuda())
    xg = torch.from_numpy(x).cuda()
    ge = L.capture(lambda: L.encode(xg, "cpo"))
    L.encode(xg, "cpo")
    gc = L.capture(lambda: L.conv())
    gs = L.capture(lambda: (L.encode(xg, "cpo"), L.conv()))
    print(json.dumps({"tree": root, "workload": wl, "encode_us": timed(ge), "conv_us": timed(gc), "step_us": timed(gs)}), flush=True)
