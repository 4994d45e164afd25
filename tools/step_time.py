"""cfg2-style step time (CPO encode + conv in one graph, L2 flushed, event-timed; mean and
median of N) for a few workloads -- quick A/B of library variants via SPC_LIB_OVERRIDE.

  python tools/step_time.py [workload ...]
"""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from bench import workload
from synth import clustered_relu, he_normal
from paper_2104_08314_b200.layer import SparseConvLayer

flush = torch.empty(64 * 2 ** 20, device="cuda")
for wl in sys.argv[1:] or ["cfg1", "cfg2", "cfg3", "cfg4a"]:
    c = workload(wl); d = c["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    L = SparseConvLayer(d, torch.from_numpy(w).cuda())
    xg = torch.from_numpy(x).cuda()
    g = L.capture(lambda: L.forward(xg, "cpo"))
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(300)]
    for a, b in ev:
        flush.zero_(); a.record(); g.replay(); b.record()
    torch.cuda.synchronize()
    ts = np.array([a.elapsed_time(b) * 1e3 for a, b in ev])
    print(json.dumps({"workload": wl, "step_us_mean": round(float(ts.mean()), 2), "step_us_median": round(float(np.median(ts)), 2)}), flush=True)
