"""Phase timeline of the encoder and the strip conv from device probes.

  python paper_2104_08314_b200/build.py --force --probes     # here (CPU)
  python tools/probe_run.py cfg2 [cfg1 ...]                   # on the GPU box
Per slot: median / max over CTAs of (stamp - earliest kernel start), in us.
"""
import ctypes, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["SPC_LIB_OVERRIDE"] = os.path.join(ROOT, "paper_2104_08314_b200", "libspconv_probe.so")
import numpy as np
import torch
import paper_2104_08314_b200 as spc
from bench import workload
from synth import clustered_relu, he_normal
from paper_2104_08314_b200.layer import SparseConvLayer

lib = ctypes.CDLL(os.environ["SPC_LIB_OVERRIDE"])
buf = np.zeros((1024, 16, 2), dtype=np.uint64)


def grab(fn):
    fn(buf.ctypes.data_as(ctypes.c_void_p), 1)
    return buf.copy()


def report(name, b):
    t = b[:, :, 0].astype(np.int64)
    used = t[:, 0] > 0
    t = t[used]
    if not len(t):
        print(name, "no probes"); return
    t0 = t[:, 0].min()
    print(f"{name}: {used.sum()} CTAs, end-to-end {(t[t > 0].max() - t0) / 1e3:.2f} us")
    for s in range(16):
        col = t[:, s]
        ok = col > 0
        if not ok.any():
            continue
        rel = (col[ok] - t0) / 1e3
        print(f"   slot {s:2d}: median {np.median(rel):7.2f}  max {rel.max():7.2f}  min {rel.min():7.2f}  (n={ok.sum()})")


flush = torch.empty(64 * 2 ** 20, device="cuda")
for wl in sys.argv[1:] or ["cfg1", "cfg2"]:
    c = workload(wl); d = c["desc"]
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"] or 0.5, c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    xg, wg = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    L = SparseConvLayer(d, wg)
    for _ in range(3):
        L.forward(xg, os.environ.get("PROBE_ALGO", "cpo"))
    torch.cuda.synchronize()
    grab(lib.spc_debug_probes_enc); grab(lib.spc_debug_probes_conv)
    if os.environ.get("PROBE_GRAPH"):
        gr = L.capture(lambda: L.forward(xg, os.environ.get("PROBE_ALGO", "cpo")))
        gr.replay()
        torch.cuda.synchronize()
        grab(lib.spc_debug_probes_enc); grab(lib.spc_debug_probes_conv)
    if not os.environ.get("PROBE_NOFLUSH"):
        flush.zero_()
    if os.environ.get("PROBE_GRAPH"):
        gr.replay()
    else:
        L.forward(xg, os.environ.get("PROBE_ALGO", "cpo"))
    torch.cuda.synchronize()
    e, cv = grab(lib.spc_debug_probes_enc), grab(lib.spc_debug_probes_conv)
    print(f"== {wl}")
    report("encode", e)
    # align conv to the encoder's start
    report("conv", cv)
    te, tc = e[:, :, 0].astype(np.int64), cv[:, :, 0].astype(np.int64)
    if (te > 0).any() and (tc > 0).any():
        print(f"   conv first stamp - encoder first stamp: {(tc[tc > 0].min() - te[te > 0].min()) / 1e3:.2f} us;"
              f" encoder last stamp -> conv last stamp: {(tc.max() - te.max()) / 1e3:.2f} us")
    if os.environ.get("PROBE_DUMP"):
        np.savez(os.path.join(ROOT, "gpurun_out", f"probe_{wl}.npz"), conv=cv, enc=e,
                 chan_nz_off=L.enc.chan_nz_off.cpu().numpy(), chan_ptr_off=L.enc.chan_ptr_off.cpu().numpy())
