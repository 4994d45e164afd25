"""Development: the stride-aware layout through the warp-specialised conv (SPC_WS_SLOTS=1) on
L7-like geometries, one case per subprocess (an illegal access poisons the context).
  python tools/sa_ws_debug.py            # driver: runs every case
  python tools/sa_ws_debug.py N C rho ws # one case"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(N, C, rho, use_ws, H=28, K=256):
    import torch
    import paper_2104_08314_b200 as spc
    from synth import clustered_relu, he_normal, layer_desc
    d = layer_desc(N, C, H, H, K, 3, 3, 2, 2, 1, 1, 1, 1)
    x = clustered_relu(N, C, H, H, rho, 5) if rho > 0 else __import__("numpy").zeros((N, C, H, H), "float32")
    w = he_normal(K, C, 3, 3, 1)
    enc = spc.alloc_strided_encoding(d)
    xg = torch.from_numpy(x).cuda()
    ws = spc.alloc_workspace(d)
    spc.cpo_encode_strided(d, xg, enc, None if os.environ.get("SA3") else ws)
    wg = torch.from_numpy(w).cuda()
    wp = torch.empty_like(wg).reshape(-1)
    spc.spc_pack_weights(d, wg, wp)
    Oh, Ow = spc.spc_output_dims(d)
    y = torch.empty((N, K, Oh, Ow), device="cuda")
    spc.sparse_conv_forward(d, enc, wp, y, False, ws if use_ws else None)
    torch.cuda.synchronize()
    ref = torch.nn.functional.conv2d(torch.nn.functional.pad(xg.double(), (1, 1, 1, 1)), wg.double(), stride=2)
    err = (y.double() - ref).abs().max().item()
    print(f"N={N} C={C} rho={rho} ws={use_ws}: maxerr {err:.3g}", "OK" if err < 1e-3 else "BAD")


if __name__ == "__main__":
    if len(sys.argv) > 1:
        one(int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), sys.argv[4] == "1",
            *(int(v) for v in sys.argv[5:]))
        sys.exit(0)
    cases = [(1, 32, 0.3, 0), (1, 32, 0.0, 0), (1, 128, 0.3, 0)]
    for extra in ({"SPC_WS_SLOTS": "1"}, {"SPC_WS_SLOTS": "1", "SA3": "1"}, {}):
      print("==", extra)
      env = dict(os.environ, SPC_PLAN_DEBUG="1", **extra)
      for N, C, rho, ws in cases:
        r = subprocess.run([sys.executable, __file__, str(N), str(C), str(rho), str(ws)], env=env,
                           capture_output=True, text=True, timeout=120)
        plan = [l for l in r.stderr.splitlines() if "ws plan" in l][:1]
        out = r.stdout.strip().splitlines()[-1:] or [r.stderr.strip().splitlines()[-1][-160:]]
        print(out[0], "|", plan[0] if plan else "(no ws plan)")
