import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
import paper_2104_08314_b200 as spc
from bench import workload
from synth import clustered_relu, he_normal
from paper_2104_08314_b200.layer import SparseConvLayer
wl = sys.argv[1]
c = workload(wl); d = c["desc"]
if len(sys.argv) > 2: d = dict(d, N=int(sys.argv[2]))
x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"] or 0.3, c["seed"])
w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
L = SparseConvLayer(d, torch.from_numpy(w).cuda())
xg = torch.from_numpy(x).cuda()
spc.spc_set_im2col_gemm(4)
for _ in range(3):
    L.forward(xg, "im2col")
torch.cuda.synchronize()
print("ok")
