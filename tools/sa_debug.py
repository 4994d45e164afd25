import sys, os, torch, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import paper_2104_08314_b200 as spc
from synth import cfg5_layers, clustered_relu, he_normal
c = cfg5_layers(batch=1)[7]; d = dict(c["desc"])
x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"], c["seed"])
w = he_normal(d["K"], d["C"], 3, 3, 1)
enc = spc.alloc_strided_encoding(d)
xg = torch.from_numpy(x).cuda(); spc.cpo_encode_strided(d, xg, enc)
wg = torch.from_numpy(w).cuda(); wp = torch.empty_like(wg).reshape(-1); spc.spc_pack_weights(d, wg, wp)
ws = spc.alloc_workspace(d)
Oh, Ow = spc.spc_output_dims(d)
y = torch.empty((d["N"], d["K"], Oh, Ow), device="cuda")
spc.sparse_conv_forward(d, enc, wp, y, False, ws)
print(spc.spc_encoding_lengths(enc))
