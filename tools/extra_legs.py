"""Other encodings of a layer (bench.measure_extra): the CSCC baseline and the stride-aware
layout, step time and CR against the canonical CPO path, back to back over L2-cold sets.

  python tools/extra_legs.py cscc cfg2 cfg3 ...      |   python tools/extra_legs.py cpo_sa cfg3s2 cfg5L3 ...
"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
import bench  # noqa: E402
from synth import he_normal  # noqa: E402

kind, names = sys.argv[1], sys.argv[2:]
dev, st = torch.device("cuda", 0), torch.cuda.current_stream()
for name in names:
    c = bench.workload(name)
    d = c["desc"]
    row = bench.measure_extra(name, d, bench.make_pool(c), he_normal(d["K"], d["C"], d["R"], d["S"], c["seed"]), dev, st,
                              100, [kind])
    print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items() if k != "l2"}))
    torch.cuda.empty_cache()
