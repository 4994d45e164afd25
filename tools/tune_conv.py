#!/usr/bin/env python
"""Sweep the sparse-conv tile configurations (SPC_TUNE) on a few workloads.

  python tools/tune_conv.py                 # parent: one subprocess per setting
  python tools/tune_conv.py --child W SET   # child: time encode / conv for workload W
Prints one JSON line per (workload, setting) with device times (CUDA graph, L2 flushed).
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SETTINGS = {
    "s1": ["auto", "1", "2", "4", "8"],
    "s2": ["auto", "1", "2", "4"],
    "x7": ["auto", "1", "2"],
}
WORKLOADS = {"cfg2": "s1", "cfg3": "s1", "cfg3s2": "s2", "cfg5L0": "s1", "cfg5L8": "s1", "cfg5L14": "s1",
             "cfg5L3": "s2", "cfg5L12": "s2", "cfg4a": "x7", "cfg4b": "x7", "cfg1": "s1"}


def child(wl: str, setting: str):
    import torch
    import numpy as np
    from bench import workload
    from synth import clustered_relu, he_normal
    from paper_2104_08314_b200.layer import SparseConvLayer
    c = workload(wl)
    d = c["desc"]
    dens = c["density"] if c["density"] is not None else 0.5
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], dens, c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    xg, wg = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    L = SparseConvLayer(d, wg)
    flush = torch.empty(64 * 2 ** 20, device="cuda")
    g_enc = L.capture(lambda: L.encode(xg, "cpo"))
    L.encode(xg, "cpo")
    g_conv = L.capture(lambda: L.conv())

    def timed(gr, n=50):
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in ev:
            flush.zero_()
            a.record(); gr.replay(); b.record()
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
        return ts[len(ts) // 2]
    t_enc, t_conv = timed(g_enc), timed(g_conv)
    Oh, Ow = L.Oh, L.Ow
    dense = 2.0 * d["N"] * d["K"] * d["C"] * d["R"] * d["S"] * Oh * Ow
    print(json.dumps({"workload": wl, "setting": setting, "enc_us": round(t_enc, 2), "conv_us": round(t_conv, 2),
                      "dense_gflops_conv": round(dense / (t_conv * 1e-6) / 1e9, 1), "density": float((x != 0).mean())}))


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--child":
        child(sys.argv[2], sys.argv[3])
        return
    wls = sys.argv[1:] or list(WORKLOADS)
    for wl in wls:
        for s in SETTINGS[WORKLOADS[wl]]:
            env = dict(os.environ)
            if s != "auto":
                env["SPC_TUNE"] = s
            r = subprocess.run([sys.executable, __file__, "--child", wl, s], env=env, capture_output=True, text=True,
                               timeout=300)
            out = r.stdout.strip().splitlines()
            print(out[-1] if out else json.dumps({"workload": wl, "setting": s, "error": r.stderr[-300:]}), flush=True)


if __name__ == "__main__":
    main()
