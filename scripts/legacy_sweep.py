"""p-sweep of the macro-element assembly (lor_assemble_h1, full call) against the unstructured
comparator (lor_legacy_assemble_h1) on Cartesian meshes of N^3 LOR cells (PAPER.md l.593-606 and
its Fig. "throughput-assembly": the unstructured algorithm is flat in p, the macro-element one rises
with p, equal at p = 2, > 2x at the highest p).  Device time per call (CUDA events, L2 flushed),
MDOF/s = rows / time.  usage: python scripts/legacy_sweep.py [N=96] > profiles/legacy_sweep_*.jsonl"""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2210_12253_b200 import meshgen as mg  # noqa: E402
from paper_2210_12253_b200.lor import LOR  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 96
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()


def t_ms(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    out = []
    for i in range(reps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return statistics.median(out)


for p in (1, 2, 3, 4, 6, 8):
    n = N // p
    m = mg.box_mesh(3, (n, n, n), p)
    t0 = time.perf_counter()
    ctx = LOR(m, stream=st)
    torch.cuda.synchronize()
    setup = (time.perf_counter() - t0) * 1e3
    q = ctx.query("h1")
    out = ctx.alloc(q["n_local"], q["nnz"])
    macro = t_ms(lambda: ctx.assemble("h1", 1.0, 1.0, "vertex", out=out))
    t0 = time.perf_counter()
    ctx.legacy_setup()
    torch.cuda.synchronize()
    lsetup = (time.perf_counter() - t0) * 1e3
    leg = t_ms(lambda: ctx.legacy_assemble(1.0, 1.0, out=out))
    ph = ctx.phase_ms()
    print(json.dumps(dict(p=p, elements=n ** 3, rows=q["n_local"], nnz=q["nnz"], macro_ms=macro, legacy_ms=leg,
                          macro_mdofs=q["n_local"] / macro / 1e3, legacy_mdofs=q["n_local"] / leg / 1e3,
                          speedup=leg / macro, macro_fill_path=ctx.fill_path("h1"), setup_ms=setup,
                          legacy_setup_ms=lsetup, legacy_phases_ms=ph)), flush=True)
    ctx.close()
    del out
    torch.cuda.empty_cache()
