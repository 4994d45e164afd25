#!/usr/bin/env python
"""Device time of encode and conv (CPO) per workload, auto tile config, in one process.

  python tools/time_all.py [workload ...]
Prints one JSON line per workload (CUDA graph replay, L2 flushed between reps, mean of 200).
"""
from __future__ import annotations

import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

WORKLOADS = ["cfg1", "cfg2", "cfg3", "cfg3s2", "cfg4a", "cfg4b", "cfg5L0", "cfg5L3", "cfg5L8", "cfg5L12", "cfg5L14"]


def main():
    import torch
    from bench import workload, nze_macs
    from synth import clustered_relu, he_normal
    from paper_2104_08314_b200.layer import SparseConvLayer
    flush = torch.empty(64 * 2 ** 20, device="cuda")

    def timed(gr, n=200):
        for _ in range(3):
            gr.replay()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for a, b in ev:
            flush.zero_()
            a.record(); gr.replay(); b.record()
        torch.cuda.synchronize()
        # event resolution is 32 ns (tools/microbench/event_resolution.py), but step times on
        # this pool cluster at multiples of ~2.05 us (launch scheduling): report the mean
        ts = [a.elapsed_time(b) * 1e3 for a, b in ev]
        return sum(ts) / len(ts)

    for wl in (sys.argv[1:] or WORKLOADS):
        c = workload(wl)
        d = c["desc"]
        if os.environ.get("TIME_BATCH"):          # e.g. 256: the stack's per-GPU batch at N=1
            d = dict(d, N=int(os.environ["TIME_BATCH"]))
        dens = c["density"] if c["density"] is not None else 0.5
        if os.environ.get("TIME_DENSITY"):
            dens = float(os.environ["TIME_DENSITY"])
        x = clustered_relu(d["N"], d["C"], d["H"], d["W"], dens, c["seed"], c["dead_frac"], c["zero_tile_frac"])
        w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
        xg, wg = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
        L = SparseConvLayer(d, wg)
        g_enc = L.capture(lambda: L.encode(xg, "cpo"))
        L.encode(xg, "cpo")
        g_conv = L.capture(lambda: L.conv())
        g_i2c = L.capture(lambda: L.forward(xg, "im2col"))
        L.encode(xg, "cpo")
        t_enc, t_conv, t_i2c = timed(g_enc), timed(g_conv), timed(g_i2c)
        Oh, Ow = L.Oh, L.Ow
        macs = nze_macs(d, x, Oh, Ow)
        dense = 2.0 * d["N"] * d["K"] * d["C"] * d["R"] * d["S"] * Oh * Ow
        print(json.dumps({"workload": wl, "enc_us": round(t_enc, 2), "conv_us": round(t_conv, 2),
                          "i2c_us": round(t_i2c, 2),
                          "nze_tflops": round(2 * macs / (t_conv * 1e-6) / 1e12, 2),
                          "fp32_frac": round(2 * macs / (t_conv * 1e-6) / 74.45e12, 4),
                          "enc_gbs": round(4 * x.size / (t_enc * 1e-6) / 1e9, 1),
                          "dense_gflops_conv": round(dense / (t_conv * 1e-6) / 1e9, 1),
                          "density": round(float((x != 0).mean()), 4)}), flush=True)


if __name__ == "__main__":
    main()
