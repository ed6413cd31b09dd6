"""Per-CTA phase timing of the element kernel (LOR_PHASE_TIMING=1): where a CTA's lifetime goes.
usage: python scripts/phase_timing.py [n] [p] [space]"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOR_PHASE_TIMING"] = "1"
from paper_2210_12253_b200 import meshgen as mg  # noqa: E402
from paper_2210_12253_b200.lor import LOR  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
space = sys.argv[3] if len(sys.argv) > 3 else "h1"
m = mg.box_mesh(3, (n, n, n), p)
L = LOR(m)
out = L.assemble(space)
for _ in range(4):
    L.assemble(space, out=out)
L.sync()
ts = L.debug_dump(2, space).view(np.uint64).reshape(-1, 16).astype(np.int64)
life = ts[:, 4] - ts[:, 0]
print(f"elements {len(ts)}  CTA lifetime cycles: mean {life.mean():.0f} p50 {np.median(life):.0f} p90 {np.percentile(life, 90):.0f}")
names = ["prologue", "cells", "rows (thread 0)", "rest of CTA"]
for i, nm in enumerate(names):
    d = ts[:, i + 1] - ts[:, i]
    print(f"  {nm:16s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f}")
own = ts[:, 11:15]
ok = (own > 0).all(1)
if ok.any():
    o = own[ok]
    print(f"own-row path (first own row; {ok.mean():.2f} of CTAs), start {np.median(o[:, 0] - ts[ok, 0]):.0f} after CTA start:")
    for i, nm in enumerate(["p0+positions", "values", "stores"]):
        d = o[:, i + 1] - o[:, i]
        print(f"  {nm:16s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}")
