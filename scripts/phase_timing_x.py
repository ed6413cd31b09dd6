"""Per-CTA phase clocks of the extended-frame fill k_xh1_fill (LOR_PHASE_TIMING=1).
usage: python scripts/phase_timing_x.py [n] [p]   (Cartesian n^3 mesh, H1)"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["LOR_PHASE_TIMING"] = "1"
from paper_2210_12253_b200 import meshgen as mg  # noqa: E402
from paper_2210_12253_b200.lor import LOR  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
p = int(sys.argv[2]) if len(sys.argv) > 2 else 4
L = LOR(mg.box_mesh(3, (n, n, n), p))
out = L.assemble("h1")
for _ in range(4):
    L.assemble("h1", out=out)
L.sync()
ts = L.debug_dump(2, "h1").view(np.uint64).reshape(-1, 16).astype(np.int64)
life = ts[:, 4] - ts[:, 0]
print(f"p={p} elements {len(ts)}  CTA lifetime cycles: mean {life.mean():.0f} p50 {np.median(life):.0f} p90 {np.percentile(life, 90):.0f}")
for nm, a, b in [("prologue", 0, 1), ("cells (chunk 0)", 1, 2), ("row gather", 2, 5), ("stage", 5, 3), ("write-out + rest", 3, 4)]:
    d = ts[:, b] - ts[:, a]
    print(f"  {nm:18s} mean {d.mean():8.0f}  p50 {np.median(d):8.0f}  p90 {np.percentile(d, 90):8.0f}")
