#!/usr/bin/env python
"""Conv time vs batch size for one cfg5 layer shape (wave-quantisation check).

  python tools/wave_probe.py cfg5L0 24 28 29 30 32
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from bench import workload
    from synth import clustered_relu, he_normal
    from paper_2104_08314_b200.layer import SparseConvLayer
    flush = torch.empty(64 * 2 ** 20, device="cuda")
    wl = sys.argv[1]
    c = workload(wl)
    for nb in [int(v) for v in sys.argv[2:]]:
        d = dict(c["desc"], N=nb)
        x = clustered_relu(nb, d["C"], d["H"], d["W"], c["density"] or 0.3, c["seed"], c["dead_frac"], c["zero_tile_frac"])
        w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
        xg, wg = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
        L = SparseConvLayer(d, wg)
        L.encode(xg, "cpo")
        gr = L.capture(lambda: L.conv())
        L.encode(xg, "cpo")
        for _ in range(3):
            gr.replay()
        ts = []
        for _ in range(50):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(); gr.replay(); b.record()
            torch.cuda.synchronize()
            ts.append(a.elapsed_time(b) * 1e3)
        ts.sort()
        t = ts[len(ts) // 2]
        print(json.dumps({"workload": wl, "N": nb, "conv_us": round(t, 2), "us_per_image": round(t / nb, 3)}), flush=True)
        del L
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
