"""Emulated weak scaling on one GPU: the N ranks of a z-slab run (N x 32^3 elements for C2, N x 24^3
for C3) are set up as N contexts on the same device, and each rank's full assembly call is timed on
its own (CUDA events, L2 flushed before each) -- the per-GPU work of an N-GPU run, without the
other GPUs.  With the extended frame no data moves between ranks inside the call (ghost layer of
coordinates), so max-over-ranks of these times is the N-GPU step time up to NVLink/launch noise.
Prints one JSON line per N.  usage: python scripts/emulated_scaling.py [C2|C3] [N ...]"""
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2210_12253_b200 import meshgen as mg  # noqa: E402
from paper_2210_12253_b200.lor import LOR  # noqa: E402


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C2"
    ns = [int(v) for v in sys.argv[2:]] or [1, 2, 4, 8]
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    stream = torch.cuda.current_stream()
    t1 = None
    for n in ns:
        mesh, form = mg.config_mesh(cfg, gpus=n)
        per = []
        rows = 0
        for r in range(n):
            ctx = LOR(mesh, rank=r, nranks=n, stream=stream)
            sp = form["space"]
            q = ctx.query(sp)
            rows += q["n_local"]
            out = ctx.alloc(q["n_local"], q["nnz"])
            for _ in range(3):
                ctx.assemble(sp, form["alpha"], form["beta"], form["quad"], out=out)
            ctx.sync()
            ts = []
            for i in range(10):
                flush.fill_(float(i))
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                ctx.assemble(sp, form["alpha"], form["beta"], form["quad"], out=out)
                b.record(stream)
                b.synchronize()
                ts.append(a.elapsed_time(b))
            per.append(statistics.median(ts))
            path = ctx.fill_path(sp)
            ctx.close()
            del out
            torch.cuda.empty_cache()
        tmax = max(per)
        if n == 1:
            t1 = tmax
        print(json.dumps({"config": cfg, "ranks": n, "fill_path": path, "rows_global": rows,
                          "ms_per_rank": [round(v, 4) for v in per], "ms_max": tmax,
                          "MDOF_s_global": rows / (tmax * 1e-3) / 1e6,
                          "weak_efficiency_vs_1": (t1 / tmax) if t1 else None}), flush=True)


if __name__ == "__main__":
    main()
