"""Quick device timing of the post-assembly steps (ParCSR split, A4 elimination, coordinate vectors)."""
import sys, json
import torch
sys.path.insert(0, ".")
from paper_2210_12253_b200 import meshgen as mg
from paper_2210_12253_b200.lor import LOR

def t_ms(fn, st, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(reps):
        fn()
    e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps

for cfg in sys.argv[1:] or ["C2"]:
    m, form = mg.config_mesh(cfg)
    ctx = LOR(m)
    st = torch.cuda.current_stream()
    sp = form["space"]
    A = ctx.assemble(sp, 1.0, 1.0, "vertex")
    ctx.sync()
    P = ctx.parcsr(sp, A)
    ess = ctx.boundary_dofs(sp)
    import paper_2210_12253_b200.lor as L
    import ctypes as C
    a = ctx._csr(*A)
    pc = ctx._pcsr(P)
    fill = lambda: L.lib().lor_parcsr_fill(ctx.h, L.OPS[sp], C.byref(a), C.byref(pc))
    v = [C.c_int64() for _ in range(3)]
    import time
    t0 = time.perf_counter(); L.lib().lor_parcsr_prepare(ctx.h, L.OPS[sp], C.byref(a), *[C.byref(x) for x in v]); t1 = time.perf_counter()
    elim = lambda: L.lib().lor_eliminate_bc(ctx.h, L.OPS[sp], C.c_void_p(ess.data_ptr()), C.c_int64(ess.numel()), C.byref(pc))
    out = torch.empty((3, ctx.query("h1")["n_local"]), dtype=torch.float64, device="cuda")
    coords = lambda: L.lib().lor_coordinates(ctx.h, C.c_void_p(out.data_ptr()))
    q = ctx.query(sp)
    res = dict(cfg=cfg, n=q["n_local"], nnz=q["nnz"], n_ess=ess.numel(), prepare_wall_ms=(t1 - t0) * 1e3,
               fill_ms=t_ms(fill, st), elim_ms=t_ms(elim, st), coords_ms=t_ms(coords, st), n_h1=out.shape[1])
    print(json.dumps(res), flush=True)
    ctx.close()
