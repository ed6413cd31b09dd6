"""Benchmark of the LOR assembly hot path (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--config C2] [--impl reference]

A "step" is one full assembly call lor_assemble_* through the C ABI: row counts, int64 scan,
fused element assembly (sub-cell matrices + CSR column/value fill + merge of shared rows) and,
for N > 1, the NCCL interface exchange + merge of interface rows (PAPER.md Step S1.2, A1-A3).
Workload at N = 1: BASELINE configs[1] = C2 (3D H1 diffusion+mass, 32^3 hexes, p = 4); at N > 1
the same per GPU (32 x 32 x 32N elements, z-slabs: weak scaling).  Inputs are resident in HBM
when the timed region starts; L2 is flushed (512 MiB write) before every timed step.

Reported: value = global rows / step time (MDOF/s, max over ranks); roofline of the dominant
kernel (k_assemble) against MEASURED_PEAKS.json hbm_gbs; the CPU oracle on a bounded sample
(cpu_baseline); e2e = the same call with the E-vector copied H2D from pinned host memory and
the CSR copied back D2H inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "LOR assembly MDOF/s and HBM GB/s (fp64) at 1/2/4/8 B200"
WORKLOADS = {
    "C2": "C2: 3D H1 diffusion+mass (alpha=beta=1), 32^3 hex per GPU, p=4, vertex rule, Cartesian",
    "C2-J": "C2-J: C2 with jittered interior vertices (seed 12253)",
    "C3": "C3: 3D H1 diffusion+mass, 24^3 hex per GPU, p=8, Kershaw eps=0.3",
    "C4": "C4: 3D H(curl) Nedelec LOR, 32^3 hex per GPU, p=4, curl-curl+mass",
    "C5": "C5: 3D H(div) Raviart-Thomas LOR, 32^3 hex per GPU, p=4, div-div+mass",
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap",
               0x80: "hw_power_brake_slowdown"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.002)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self.ok:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def algorithmic_bytes(mesh, q, dim, p, nel_local):
    """SURVEY 8(d) d.3 adapted to this design: coordinate E-vector +
    per-element topology records + row_ptr + col/val; the dominant kernel k_assemble reads the
    E-vector, the topology/space records and row_ptr, and writes col/val."""
    npts = (p + 1) ** dim
    coords = 8 * dim * npts * nel_local
    topo = (192 + 256) * nel_local
    rowptr = 8 * (q["n_local"] + 1)
    out = 12 * q["nnz"]
    return dict(call=coords + topo + rowptr + out, k_assemble=coords + topo + rowptr + out)


def cpu_baseline(cfg, space, form, sample_n):
    """The oracle as it stands (single-threaded C, test infrastructure) on a bounded sample."""
    from oracle import oracle as O
    from paper_2210_12253_b200 import meshgen as mg
    O.build()
    m, _ = mg.config_mesh(cfg, n=sample_n)
    t0 = time.perf_counter()
    A = O.assemble(m, space, form["quad"], form["alpha"], form["beta"])
    dt = time.perf_counter() - t0
    rows = A.row_ptr.shape[0] - 1
    return {"value": rows / dt / 1e6, "unit": "MDOF/s", "cores": 1, "kind": "oracle",
            "sample": f"{cfg} recipe at {sample_n}^3 elements ({rows} rows, {A.nnz} nnz), full oracle assembly, "
                      f"{dt:.2f} s"}


def run_reference(args):
    """--impl reference: the CPU oracle on a bounded sample of the workload, per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2210_12253_b200 import meshgen as mg
    O.build()
    cfg = args.config
    m, form = mg.config_mesh(cfg, n=args.ref_n)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        A = O.assemble(m, form["space"], form["quad"], form["alpha"], form["beta"])
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    rows = A.row_ptr.shape[0] - 1
    t = statistics.mean(times)
    v = rows / t / 1e6
    line = {"metric": METRIC, "value": v, "unit": "MDOF/s", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(cfg, cfg), "sample_elements": f"{args.ref_n}^3", "rows": rows,
                       "nnz": int(A.nnz)},
            "cpu_baseline": {"value": v, "unit": "MDOF/s", "cores": 1, "kind": "oracle",
                             "sample": f"{cfg} recipe at {args.ref_n}^3 elements per step"},
            "e2e": {"value": v, "unit": "MDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-n", type=int, default=20, help="elements per axis of the oracle cpu_baseline sample")
    ap.add_argument("--ref-n", type=int, default=12, help="elements per axis per reference-arm step")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import torch.distributed as dist

    from paper_2210_12253_b200 import meshgen as mg
    from paper_2210_12253_b200.lor import LOR, nccl_unique_id

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    dev = torch.device("cuda", local_rank)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream(dev)

    mesh, form = mg.config_mesh(args.config, gpus=world)
    nid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    ctx = LOR(mesh, rank=rank, nranks=world, nccl_id=nid, device=local_rank, stream=stream)
    space = form["space"]
    q = ctx.query(space)
    out = ctx.alloc(q["n_local"], q["nnz"])
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    def step():
        ctx.assemble(space, form["alpha"], form["beta"], form["quad"], out=out)

    for _ in range(max(args.warmup, 3)):
        step()
    ctx.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    phases = []
    l0 = ctx.launches()
    with ClockSampler(dev.index) as clk:
        for i in range(args.steps):
            flush.fill_(float(i))  # L2 flush outside the timed step
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
            ev[i][1].synchronize()
            phases.append(ctx.phase_ms())
    ctx.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = ctx.launches() - l0
    step_ms = [a.elapsed_time(b) for a, b in ev]
    t_ms = statistics.mean(step_ms)
    # the fill step: element pass k_assemble + merge pass k_merge_rows
    asm_ms = statistics.mean(p[1] + (p[2] if len(p) > 3 else 0.0) for p in phases)
    if world > 1:
        tt = torch.tensor([t_ms, asm_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, asm_ms = float(tt[0]), float(tt[1])
    value = q["n_global"] / (t_ms * 1e-3) / 1e6
    nel_local = ctx.n_elem_local
    B = algorithmic_bytes(mesh, q, mesh.dim, mesh.p, nel_local)
    peak, peak_kind = peaks()
    achieved = B["k_assemble"] / (asm_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(args.config, {}).get("fill_dram_bytes")
        except Exception:
            traffic = None

    # ---- e2e: pinned host E-vector H2D + assembly + CSR D2H, same public API ------------------
    e2e = None
    if not args.no_e2e:
        e0, e1 = ctx.elem_begin, ctx.elem_begin + nel_local
        Xh = torch.from_numpy(mesh.X[e0:e1].copy()).pin_memory()
        hrp = torch.empty(q["n_local"] + 1, dtype=torch.int64).pin_memory()
        hcol = torch.empty(max(q["nnz"], 1), dtype=torch.int32).pin_memory()
        hval = torch.empty(max(q["nnz"], 1), dtype=torch.float64).pin_memory()
        ne = max(3, min(args.steps, 10))
        times = []
        for i in range(ne + 2):
            flush.fill_(float(i))
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            ctx.update_coordinates(Xh)
            step()
            hrp.copy_(out[0], non_blocking=True)
            hcol.copy_(out[1], non_blocking=True)
            hval.copy_(out[2], non_blocking=True)
            b.record(stream)
            b.synchronize()
            if i >= 2:
                times.append(a.elapsed_time(b))
        te = statistics.mean(times)
        if world > 1:
            tt = torch.tensor([te], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            te = float(tt[0])
        e2e = {"value": q["n_global"] / (te * 1e-3) / 1e6, "unit": "MDOF/s", "ms_per_step": te,
               "h2d_bytes_per_step": int(Xh.numel() * 8),
               "d2h_bytes_per_step": int(hrp.numel() * 8 + hcol.numel() * 4 + hval.numel() * 8)}

    if rank == 0:
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(args.config, space, form, args.cpu_n)
        ph = [statistics.mean(p[i] for p in phases) for i in range(len(phases[0]))] if phases and phases[0] else []
        line = {
            "metric": METRIC, "value": value, "unit": "MDOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(args.config, args.config), "rows_global": q["n_global"],
                       "nnz_per_gpu": q["nnz"], "elements_per_gpu": nel_local, "p": mesh.p, "space": space,
                       "l2": "flushed (512 MiB write) before every timed step",
                       "parallelism": f"z-slab x{world}" if world > 1 else "single GPU"},
            "hbm_gbs": B["call"] / (t_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": ("fill step a6 = k_xh1_fill" if ctx.fill_path(space) == 1 else
                                                    "fill step a6 = k_assemble + k_merge_rows"), "achieved": achieved,
                         "peak": peak, "unit": "GB/s", "frac": achieved / peak, "peak_kind": peak_kind,
                         "traffic": traffic, "algorithmic_bytes_per_launch": B["k_assemble"], "avg_launch_ms": asm_ms},
            "phases_ms": dict(zip(["count+scan", "k_assemble", "k_merge_rows", "exchange+finalize"], ph)),
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
