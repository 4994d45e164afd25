import sys, os
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import torch
from bench import workload
from synth import clustered_relu, he_normal
from paper_2104_08314_b200.layer import SparseConvLayer
wl = sys.argv[1]
c = workload(wl); d = c["desc"]
if len(sys.argv) > 2:
    d = dict(d, N=int(sys.argv[2]))
dens = c["density"] if c["density"] is not None else 0.5
if os.environ.get("PROF_DENSITY"):
    dens = float(os.environ["PROF_DENSITY"])
x = clustered_relu(d["N"], d["C"], d["H"], d["W"], dens, c["seed"], c["dead_frac"], c["zero_tile_frac"])
w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
L = SparseConvLayer(d, torch.from_numpy(w).cuda())
xg = torch.from_numpy(x).cuda()
for _ in range(3):
    L.forward(xg, "cpo")
torch.cuda.synchronize()
print("ok")
