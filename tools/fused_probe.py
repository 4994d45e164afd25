"""Time the pieces of the fused conv+encode on the cfg4 chain (dev A/B via SPC_FUSE_DEBUG:
0 full, 1 conv + masks only, 2 conv only through the fused entry)."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
kinds = ("conv1", "conv1_fused") if os.environ.get("SPC_FUSE_DEBUG", "0") != "0" else \
    ("separate", "fused", "conv1", "conv1_fused", "encode2")
r = bench.measure_fused_chain(torch.device("cuda", 0), torch.cuda.current_stream(), 200, kinds=kinds)
r["debug"] = os.environ.get("SPC_FUSE_DEBUG", "0")
print(json.dumps({k: (round(v, 2) if isinstance(v, float) else v) for k, v in r.items() if k not in ("fused_form",)}))
