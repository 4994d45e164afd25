"""Phase timeline of tile_conv_kernel (probe build; development only).

  python paper_2104_08314_b200/build.py --force --probes   # here
  python tools/tc_probe.py cfg3 [...]                       # on the GPU box
Slots: 0 start, 1 producer-0 after griddepcontrol.wait, 2 side tables, 3/6 chunk staged, 4/7 stage
free, 5/8 lists published, 9 consumer-0 first full, 10 consumer-0 done, 11 epilogue, 12 after the
partials barrier, 13 reduction done.  Printed: per slot the median / max over CTAs of (t - t0) in us.
"""
import ctypes
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SPC_LIB_OVERRIDE"] = os.path.join(ROOT, "paper_2104_08314_b200", "libspconv_probe.so")


def main():
    import torch
    from bench import workload
    from synth import clustered_relu, he_normal
    from paper_2104_08314_b200.layer import SparseConvLayer
    lib = ctypes.CDLL(os.environ["SPC_LIB_OVERRIDE"])
    buf = np.zeros((1024, 16, 2), dtype=np.uint64)
    for wl in sys.argv[1:]:
        c = workload(wl)
        d = c["desc"]
        x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"] or 0.3, c["seed"], c["dead_frac"], c["zero_tile_frac"])
        w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
        L = SparseConvLayer(d, torch.from_numpy(w).cuda())
        L.encode(torch.from_numpy(x).cuda(), "cpo")
        for _ in range(3):
            L.conv()
        torch.cuda.synchronize()
        lib.spc_debug_probes_conv(buf.ctypes.data_as(ctypes.c_void_p), 1)
        L.conv()
        torch.cuda.synchronize()
        lib.spc_debug_probes_conv(buf.ctypes.data_as(ctypes.c_void_p), 1)
        t = buf[:, :, 0].astype(np.int64)
        used = t[:, 0] > 0
        t = t[used]
        t0 = t[:, 0].min()
        res = {"workload": wl, "ctas": int(used.sum()), "kernel_span_us": round((t[:, 13].max() - t0) / 1e3, 2)}
        for sl in range(14):
            v = t[:, sl]
            ok = v > 0
            rel = (v[ok] - t[ok, 0]) / 1e3
            if ok.any():
                res[f"s{sl}"] = [round(float(np.median(rel)), 2), round(float(rel.max()), 2)]
        start = (t[:, 0] - t0) / 1e3
        res["cta_start_us"] = [round(float(np.median(start)), 2), round(float(start.max()), 2)]
        print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
