"""Dump tcgen05 im2col outputs of a few layers to an .npz (A/B of GEMM variants: run with and
without SPC_LIB_OVERRIDE, then compare the files bit for bit).

  python tools/tc_dump.py out.npz
"""
import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch, numpy as np
import paper_2104_08314_b200 as spc
from bench import workload
from synth import clustered_relu, he_normal
from paper_2104_08314_b200.layer import SparseConvLayer
out = {}
for wl, n in (("cfg5L0", 8), ("cfg5L8", 32), ("cfg5L14", 32)):
    c = workload(wl); d = dict(c["desc"], N=n)
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], 0.3, c["seed"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    L = SparseConvLayer(d, torch.from_numpy(w).cuda())
    spc.spc_set_im2col_gemm(4)
    y = L.forward(torch.from_numpy(x).cuda(), "im2col").cpu().numpy()
    out[wl] = y
np.savez(sys.argv[1], **out)
print("ok")
