import sys, os, torch
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "/root/repo"))
import bench, paper_2104_08314_b200 as spc
from synth import he_normal
from paper_2104_08314_b200.layer import SparseConvLayer
for name in sys.argv[1:]:
    c = bench.workload(name); d = c["desc"]
    x = torch.from_numpy(bench.make_pool(c)[:d["N"]]).cuda()
    L = SparseConvLayer(d, torch.from_numpy(he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])).cuda())
    e = L.extra_encoding("cpo_sa")
    def t(fn, n=20):
        fn(); torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(n): fn()
        b.record(); torch.cuda.synchronize(); return a.elapsed_time(b) / n * 1e3
    te = t(lambda: spc.cpo_encode_strided(d, x, e, L.ws))
    te3 = t(lambda: spc.cpo_encode_strided(d, x, e))
    tc = t(lambda: spc.sparse_conv_forward(d, e, L.wp, L.y, False, L.ws))
    te0 = t(lambda: L.encode(x)); tc0 = t(lambda: L.conv())
    print(name, "sa enc %.1f (3 launches %.1f) conv %.1f | cpo enc %.1f conv %.1f" % (te, te3, tc, te0, tc0))
