"""Does a write-flush of L2 leave dirty lines whose write-back lands in the next timed kernel?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from bench import workload
from synth import clustered_relu, he_normal
from paper_2104_08314_b200.layer import SparseConvLayer

wbuf = torch.empty(64 * 2 ** 20, device="cuda")
rbuf = torch.ones(64 * 2 ** 20, device="cuda")
def none(): pass
def wr(): wbuf.zero_()
def wr_rd(): wbuf.zero_(); rbuf.sum()
def rd(): rbuf.sum()
for wl in ["cfg1", "cfg2", "cfg3"]:
    c = workload(wl); d = c["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    xg, wg = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    L = SparseConvLayer(d, wg)
    g_enc = L.capture(lambda: L.encode(xg, "cpo")); L.encode(xg, "cpo")
    g_conv = L.capture(lambda: L.conv())
    g_empty = L.capture(lambda: None)
    for name, fl in [("none", none), ("write", wr), ("write+read", wr_rd), ("read", rd)]:
        res = []
        for gr in (g_enc, g_conv):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(30)]
            for a, b in ev:
                fl(); a.record(); gr.replay(); b.record()
            torch.cuda.synchronize()
            ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
            res.append(ts[len(ts) // 2])
        print(wl, name, "enc %.2f conv %.2f" % tuple(res), flush=True)
