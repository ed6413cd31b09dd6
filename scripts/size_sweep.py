"""S-n size sweep and the C3-L plateau: H1 full-call throughput (lor_assemble_h1:
symbolic pass + scan + fill) on Cartesian p = 4 and Kershaw p = 8 meshes from 10^5 to ~10^8 rows, one
B200, CUDA events, L2 flushed before every call.  usage: python scripts/size_sweep.py > profiles/size_sweep_*.jsonl"""
import json
import statistics
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2210_12253_b200 import meshgen as mg  # noqa: E402
from paper_2210_12253_b200.lor import LOR  # noqa: E402

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


cases = [("cartesian", 4, n) for n in (8, 12, 16, 24, 32, 48, 64)] + [("kershaw", 8, n) for n in (6, 12, 24, 36, 48)]
if len(sys.argv) > 1:  # e.g. "kershaw:8:48" -- selected cases only
    cases = [(c.split(":")[0], int(c.split(":")[1]), int(c.split(":")[2])) for c in sys.argv[1:]]
for kind, p, n in cases:
    m = mg.box_mesh(3, (n, n, n), p, kershaw=0.3 if kind == "kershaw" else None)
    t0 = time.perf_counter()
    ctx = LOR(m, stream=st, spaces=("h1",))
    torch.cuda.synchronize()
    setup = (time.perf_counter() - t0) * 1e3
    q = ctx.query("h1")
    out = ctx.alloc(q["n_local"], q["nnz"])
    t = t_ms(lambda: ctx.assemble("h1", 1.0, 1.0, "vertex", out=out))
    ph = ctx.phase_ms()
    B = 8 * 3 * (p + 1) ** 3 * m.nel + 4 * (p + 1) ** 3 * m.nel + 8 * (q["n_local"] + 1) + 12 * q["nnz"]
    print(json.dumps(dict(mesh=kind, p=p, n=n, elements=m.nel, rows=q["n_local"], nnz=q["nnz"], call_ms=t,
                          mdofs=q["n_local"] / t / 1e3, fill_ms=ph[1], fill_frac=B / (ph[1] * 1e-3) / 1e9 / PEAK,
                          call_frac=B / (t * 1e-3) / 1e9 / PEAK, setup_ms=setup, phases_ms=ph)), flush=True)
    ctx.close()
    del out
    torch.cuda.empty_cache()
