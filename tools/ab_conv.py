"""Per-layer device times (back to back over rotating L2-cold buffer sets, bench.Rotating):
encode / conv / step for the named workloads.  Run twice with SPC_CONV_V1=0/1 for an A/B of
the warp-specialised conv against the round-1 strip kernel.

  python tools/ab_conv.py cfg3 cfg5L8 ... [--steps 200] [--rho 0.1]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
from synth import he_normal  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("names", nargs="+")
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--rho", type=float, default=None)
    ap.add_argument("--cps", action="store_true", help="also time the CPS step")
    ap.add_argument("--check", action="store_true", help="compare y against torch conv2d (fp64) on set 0")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream()
    hbm, mhz, _ = bench.load_peaks()
    p32 = bench.fp32_peak(mhz)
    for name in args.names:
        c = dict(bench.workload(name))
        if args.rho is not None:
            c["density"] = args.rho
        d = c["desc"]
        pool = bench.make_pool(c)
        w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
        row, R = bench.measure_layer(name, d, pool, w, dev, stream, args.steps, hbm, p32, im2col=False, cps=args.cps)
        if args.check:
            L = R.layers[0]
            L.forward(R.xs[0], "cpo")
            x = R.xs[0].double()
            ref = torch.nn.functional.conv2d(torch.nn.functional.pad(x, (d["pad_left"], d["pad_right"], d["pad_top"],
                                                                        d["pad_bottom"])),
                                             torch.from_numpy(w).to(dev).double(), stride=(d["stride_h"], d["stride_w"]))
            err = (L.y.double() - ref).abs()
            tol = torch.clamp(1e-4 * ref.abs(), min=1e-5)
            row["check_bad"] = int((err > tol).sum().item())
            row["check_maxerr"] = float(err.max().item())
        row["v1"] = os.environ.get("SPC_CONV_V1", "0")
        print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in row.items() if k != "shape"}))
        del R
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
