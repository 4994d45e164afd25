#!/usr/bin/env python
"""Conv device time with phases switched off (probe build, development only).

  python paper_2104_08314_b200/build.py --force --probes   # here
  python tools/phase_time.py cfg5L8 [...]                   # on the GPU box
Per workload: full conv, walk only (staging/scatter of the first chunk only), staging and
scatter only (no walk).  Results of modes 1/2 are wrong by construction; only times matter.
"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SPC_LIB_OVERRIDE"] = os.path.join(ROOT, "paper_2104_08314_b200", "libspconv_probe.so")


def main():
    import torch
    from bench import workload
    from synth import clustered_relu, he_normal
    from paper_2104_08314_b200.layer import SparseConvLayer
    lib = ctypes.CDLL(os.environ["SPC_LIB_OVERRIDE"])
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
        return sorted(ts)[n // 2]

    for wl in sys.argv[1:]:
        c = workload(wl)
        d = c["desc"]
        rho = float(os.environ["PHASE_DENSITY"]) if os.environ.get("PHASE_DENSITY") else (c["density"] or 0.3)
        x = clustered_relu(d["N"], d["C"], d["H"], d["W"], rho, c["seed"], c["dead_frac"], c["zero_tile_frac"])
        w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
        L = SparseConvLayer(d, torch.from_numpy(w).cuda())
        L.encode(torch.from_numpy(x).cuda(), "cpo")
        gr = L.capture(lambda: L.conv())
        res = {"workload": wl}
        for m, name in ((0, "full_us"), (1, "walk_only_us"), (2, "no_walk_us"), (3, "no_taps_us"), (4, "no_scatter_us")):
            lib.spc_debug_set_phase_mode(m)
            torch.cuda.synchronize()
            res[name] = round(timed(gr), 2)
        lib.spc_debug_set_phase_mode(0)
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
