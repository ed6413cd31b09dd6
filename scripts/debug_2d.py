import sys
sys.path.insert(0, ".")
import numpy as np
from oracle import oracle as O
from paper_2210_12253_b200 import meshgen as mg
from paper_2210_12253_b200.lor import LOR
m = mg.box_mesh(2, (2, 1), 2)
ctx = LOR(m)
q = ctx.query("h1")
rp, col, val = ctx.assemble("h1", 1.0, 1.0, "vertex")
ctx.sync()
rp, col, val = rp.cpu().numpy(), col.cpu().numpy(), val.cpu().numpy()
ref = O.assemble(m, "h1", "vertex", 1.0, 1.0)
gm, gs = ctx.dof_map("h1")
print("map gpu", gm.cpu().numpy().tolist())
print("map orc", O.dof_map(m, "h1")[0].tolist())
print("rowptr gpu", rp.tolist())
print("rowptr orc", ref.row_ptr.tolist())
for r in range(min(q["n_local"], 6)):
    print(r, "gpu", col[rp[r]:rp[r+1]].tolist(), np.round(val[rp[r]:rp[r+1]], 4).tolist())
    print(r, "orc", ref.col[ref.row_ptr[r]:ref.row_ptr[r+1]].tolist(), np.round(ref.val[ref.row_ptr[r]:ref.row_ptr[r+1]], 4).tolist())
print("launches", ctx.launches(), "phases", ctx.phase_ms())

t = ctx.debug_dump(0, "h1").view(np.uint32).reshape(729, 9)
z = ctx.debug_dump(1, "h1").reshape(729, 27)
for rk in (20, 22, 2 + 9 * 5):
    print("rk", rk, [hex(w) for w in t[rk]], z[rk].tolist())
