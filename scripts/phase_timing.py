"""Per-CTA phase timing of the element kernel (LOR_PHASE_TIMING=1): where a CTA's lifetime goes.
usage: LOR_PHASE_TIMING=1 python scripts/phase_timing.py [n] [p] [space]"""
import os
import sys

import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2210_12253_b200 import meshgen as mg
from paper_2210_12253_b200.lor import LOR

os.environ["LOR_PHASE_TIMING"] = "1"
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
clk = ts[:, :6]
d = np.diff(clk, axis=1)
names = ["prologue", "cells", "rows", "arrival", "finalize"]
life = clk[:, 5] - clk[:, 0]
nfin = ts[:, 7] >> 32
print(f"elements {len(ts)}  CTA lifetime cycles: mean {life.mean():.0f} p50 {np.median(life):.0f} p90 {np.percentile(life, 90):.0f}")
for i, nm in enumerate(names):
    print(f"  {nm:10s} mean {d[:, i].mean():8.0f}  p50 {np.median(d[:, i]):8.0f}  p90 {np.percentile(d[:, i], 90):8.0f}  share {d[:, i].sum() / life.sum():.3f}")
fin = nfin > 0
print(f"finalizing CTAs {fin.mean():.3f}  (nfin mean {nfin[fin].mean():.2f});  finalize cycles among them {d[fin, 4].mean():.0f}")
g0 = ts[:, 6]
print(f"kernel span (globaltimer) {(g0.max() - g0.min()) / 1e3:.1f} us from first to last CTA start")
f = ts[fin]
sub = np.stack([f[:, 8] - f[:, 4], f[:, 9] - f[:, 8], f[:, 10] - f[:, 9], f[:, 5] - f[:, 10]], 1)
for i, nm in enumerate(["fin-info", "fin-stage", "fin-items", "fin-discard"]):
    print(f"  {nm:12s} mean {sub[:, i].mean():8.0f}  p50 {np.median(sub[:, i]):8.0f}")
it = f[:, 11:15]
print("items iterations (cycles from items start):", [int(np.median(np.where(it[:, k] > 0, it[:, k] - it[:, 0], 0))) for k in range(4)])
