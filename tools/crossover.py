#!/usr/bin/env python
"""Crossover density per layer: the density rho* at which CPO (encode + sparse conv) and CPS
stop beating the GPU im2col baseline (north_star: "each layer's measured crossover density
against the GPU im2col path").

  python tools/crossover.py [--out profiles/r01_crossover.json] [workload ...]

For each layer shape: synthetic clustered-ReLU inputs at densities RHOS (same generator,
same seed per density), CUDA-graph device time with L2 flushed between reps (median of
REPS); im2col timed with every parity-passing GEMM engine plus the 1-term TF32 reference.
rho* = linear interpolation of the first sign change of t_sparse - t_im2col.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

RHOS = [0.02, 0.05, 0.1, 0.2, 0.3, 0.4, 0.5, 0.6, 0.8, 1.0]
REPS = 15


def main():
    import numpy as np
    import torch

    import paper_2104_08314_b200 as spc
    from bench import workload
    from paper_2104_08314_b200.bounds import rho_space_bound
    from paper_2104_08314_b200.layer import SparseConvLayer
    from synth import clustered_relu, he_normal

    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("workloads", nargs="*")
    args = ap.parse_args()
    wls = args.workloads or ["cfg2", "cfg3", "cfg3s2", "cfg4a", "cfg4b"] + [f"cfg5L{i}" for i in range(16)]
    flush = torch.empty(64 * 2 ** 20, device="cuda")

    def timed(gr):
        for _ in range(2):
            gr.replay()
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(REPS)]
        for a, b in ev:
            flush.zero_()
            a.record(); gr.replay(); b.record()
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
        return ts[len(ts) // 2]

    engines = {"cublas_fp32": spc.SPC_GEMM_CUBLAS_FP32, "tc_3xtf32": spc.SPC_GEMM_TC_3XTF32,
               "cublas_tf32_1term": spc.SPC_GEMM_CUBLAS_TF32}
    results = []
    for wl in wls:
        c = workload(wl)
        d = c["desc"]
        w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
        L = SparseConvLayer(d, torch.from_numpy(w).cuda())
        # im2col does not depend on the density: time it once per engine
        x0 = torch.from_numpy(clustered_relu(d["N"], d["C"], d["H"], d["W"], 0.3, c["seed"])).cuda()
        t_dense = {}
        for name, e in engines.items():
            spc.spc_set_im2col_gemm(e)
            t_dense[name] = timed(L.capture(lambda: L.forward(x0, "im2col")))
        spc.spc_set_im2col_gemm(spc.SPC_GEMM_AUTO)
        rows = []
        s_i2c = d["N"] * L.Oh * L.Ow * d["C"] * d["R"] * d["S"]
        for rho in RHOS:
            # the config's dead channels / zero tiles cap the reachable density: keep them
            # up to rho = 0.5, plain clustered maps above
            dead, zt = (c["dead_frac"], c["zero_tile_frac"]) if rho <= 0.5 else (0.0, 0.0)
            x = torch.from_numpy(clustered_relu(d["N"], d["C"], d["H"], d["W"], rho, c["seed"], dead, zt)).cuda()
            t_cpo = timed(L.capture(lambda: L.forward(x, "cpo")))
            L.forward(x, "cpo")
            cr_cpo = s_i2c / sum(L.lengths())
            t_cps = timed(L.capture(lambda: L.forward(x, "cps")))
            L.forward(x, "cps")
            cr_cps = s_i2c / sum(L.lengths())
            rows.append({"rho": rho, "cpo_us": round(t_cpo, 2), "cps_us": round(t_cps, 2),
                         "cr_cpo": round(cr_cpo, 3), "cr_cps": round(cr_cps, 3)})

        def crossing(key, ref):
            for a, b in zip(rows, rows[1:]):
                fa, fb = a[key] - ref, b[key] - ref
                if fa <= 0 < fb:
                    return round(a["rho"] + (b["rho"] - a["rho"]) * (-fa) / (fb - fa), 3)
            return None if rows[0][key] > ref else ">1.0"
        res = {"workload": wl, "shape": {k: d[k] for k in ("N", "C", "H", "W", "K", "R", "S", "stride_h")},
               "im2col_us": {k: round(v, 2) for k, v in t_dense.items()}, "sweep": rows,
               "crossover_rho": {f"cpo_vs_{k}": crossing("cpo_us", v) for k, v in t_dense.items()}}
        res["crossover_rho"].update({f"cps_vs_{k}": crossing("cps_us", v) for k, v in t_dense.items()})

        def cr_one(key):   # first density where the encoding stops being smaller than S_im2col
            for a, b in zip(rows, rows[1:]):
                if a[key] >= 1.0 > b[key]:
                    return round(a["rho"] + (b["rho"] - a["rho"]) * (a[key] - 1.0) / (a[key] - b[key]), 3)
            return ">1.0" if rows[-1][key] >= 1.0 else None
        # SI P(rho) (worst case: VALID, no NPC/NPF) must not exceed the measured CR = 1 density
        res["space"] = {"p_bound_rho_im2col": round(rho_space_bound(d, "im2col"), 4),
                        "measured_cr1_rho_cpo": cr_one("cr_cpo"), "measured_cr1_rho_cps": cr_one("cr_cps")}
        results.append(res)
        print(json.dumps({"workload": wl, "im2col_us": res["im2col_us"], "crossover_rho": res["crossover_rho"],
                          "space": res["space"]}), flush=True)
        del L
        torch.cuda.empty_cache()
    if args.out:
        with open(args.out, "w") as f:
            json.dump({"densities": RHOS, "reps": REPS, "l2": "flushed (256 MiB write) before every rep",
                       "inputs": "clustered-ReLU generator at each density; the config's dead channels / zero tiles up to rho 0.5",
                       "layers": results}, f, indent=1)


if __name__ == "__main__":
    main()
