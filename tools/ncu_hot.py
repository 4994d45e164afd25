#!/usr/bin/env python
"""Per-CUDA-line stall samples and instruction counts from an ncu report (needs -lineinfo).

  python tools/ncu_hot.py <file.ncu-rep> <kernel regex> [top]
"""
import csv
import io
import os
import subprocess
import sys

rep, kre = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass", "-k",
                      f"regex:{kre}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
fname, hdr, out = "?", None, []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = os.path.basename(r[1])
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0].isdigit():
        continue
    si, ii = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
    num = lambda s: int(s) if s.isdigit() else 0  # noqa: E731
    out.append((num(r[si]), num(r[ii]), f"{fname}:{r[0]}", r[1].strip()[:100]))
tot = sum(o[0] for o in out) or 1
for s, n, loc, txt in sorted(out, key=lambda o: -o[0])[:top]:
    print(f"{s:7d} {100 * s / tot:5.1f}% {n:9d}  {loc:22s} {txt}")
