"""im2col baseline time per GEMM engine (CUDA graph, L2 flushed, median) on a few workloads."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2104_08314_b200 as spc
from bench import workload
from synth import clustered_relu, he_normal
from paper_2104_08314_b200.layer import SparseConvLayer

flush = torch.empty(64 * 2 ** 20, device="cuda")


def timed(gr, n=30):
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
    for a, b in ev:
        flush.zero_(); a.record(); gr.replay(); b.record()
    torch.cuda.synchronize()
    ts = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
    return ts[len(ts) // 2]


for wl in sys.argv[1:] or ["cfg2", "cfg3", "cfg5L0", "cfg5L8", "cfg5L14"]:
    c = workload(wl); d = c["desc"]
    if os.environ.get("TIME_BATCH"):
        d = dict(d, N=int(os.environ["TIME_BATCH"]))
    x = clustered_relu(d["N"], d["C"], d["H"], d["W"], c["density"] or 0.3, c["seed"], c["dead_frac"], c["zero_tile_frac"])
    w = he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"])
    xg, wg = torch.from_numpy(x).cuda(), torch.from_numpy(w).cuda()
    L = SparseConvLayer(d, wg)
    dense = 2.0 * d["N"] * d["K"] * d["C"] * d["R"] * d["S"] * L.Oh * L.Ow
    row = {"workload": wl}
    for e in (1, 3, 4):
        spc.spc_set_im2col_gemm(e)
        try:
            g = L.capture(lambda: L.forward(xg, "im2col"))
            t = timed(g)
        except spc.SpcError:
            row[["simt", "cublas_fp32", "cublas_bf16x9", "cublas_tf32", "tc3xtf32"][e] + "_us"] = None
            continue
        row[["simt", "cublas_fp32", "cublas_bf16x9", "cublas_tf32", "tc3xtf32"][e] + "_us"] = round(t, 2)
        row[["simt", "cublas_fp32", "cublas_bf16x9", "cublas_tf32", "tc3xtf32"][e] + "_tflops"] = round(dense / t / 1e6, 1)
    spc.spc_set_im2col_gemm(spc.SPC_GEMM_AUTO)
    print(json.dumps(row), flush=True)
