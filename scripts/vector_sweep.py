"""p-sweep of the vector-space assembly (lor_assemble_nd / _rt, full calls) on Cartesian meshes of
N^3 LOR cells, one B200, CUDA events, L2 flushed -- the H(curl) / H(div) counterpart of the H1
p-sweep (throughput rises with p for the macro-element method).
usage: python scripts/vector_sweep.py [N=96] [spaces=nd,rt] [ps=1,2,3,4,6,8] > profiles/vector_sweep_*.jsonl"""
import json
import statistics
import sys

import torch

sys.path.insert(0, ".")
from paper_2210_12253_b200 import meshgen as mg  # noqa: E402
from paper_2210_12253_b200.lor import LOR  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 96
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
PEAK = 6551.4


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


SPACES = sys.argv[2].split(",") if len(sys.argv) > 2 else ["nd", "rt"]
PS = [int(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [1, 2, 3, 4, 6, 8]
for space in SPACES:
    for p in PS:
        n = N // p
        m = mg.box_mesh(3, (n, n, n), p)
        ctx = LOR(m, stream=st, spaces=(space,))
        q = ctx.query(space)
        out = ctx.alloc(q["n_local"], q["nnz"])
        t = t_ms(lambda: ctx.assemble(space, 1.0, 1.0, "vertex", out=out))
        ph = ctx.phase_ms()
        ndpe = {"nd": 3 * p * (p + 1) ** 2, "rt": 3 * p * p * (p + 1), "h1": (p + 1) ** 3}[space]
        B = 24 * (p + 1) ** 3 * m.nel + 5 * ndpe * m.nel + 8 * (q["n_local"] + 1) + 12 * q["nnz"]
        print(json.dumps(dict(space=space, p=p, elements=m.nel, rows=q["n_local"], nnz=q["nnz"], call_ms=t,
                              mdofs=q["n_local"] / t / 1e3, fill_path=ctx.fill_path(space), phases_ms=ph,
                              call_frac=B / (t * 1e-3) / 1e9 / PEAK)), flush=True)
        ctx.close()
        del out
        torch.cuda.empty_cache()
