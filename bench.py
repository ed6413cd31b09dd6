"""Benchmark of the LOR assembly hot path (BASELINE.json metric) -- one JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--config C2] [--impl reference]

A "step" is one full assembly call lor_assemble_<space> through the C ABI (SURVEY P-24, PAPER.md
l.306-374): the per-call symbolic pass (row lengths and column positions, A2), the int64 scan, the
fused element pass (sub-cell matrices + CSR column/value fill, A1-A2; + merge of shared rows on the
general path) and, for N > 1, the NCCL interface exchange + merge of interface rows (A3
replacement).  Configs C4-G / C5-C time the discrete gradient / curl instead (Algorithm 1,
l.417-445).  Workload at N = 1: BASELINE configs[1] = C2 (3D H1 diffusion+mass, 32^3 hexes,
p = 4); at N > 1 the same per GPU (32 x 32 x 32N elements, z-slabs: weak scaling).  Inputs are
resident in HBM when the timed region starts; L2 is flushed (512 MiB write) before every timed step.

Reported beside the headline: the numeric-only re-assembly (pattern reuse, l.543-546,
lor_reassemble_*), lor_setup time, the roofline of the dominant kernel against MEASURED_PEAKS.json,
the CPU oracle pinned to one core (cpu_baseline), and e2e = the same call with the E-vector copied
H2D from pinned host memory and the CSR copied back D2H inside the timed region.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
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
    "C4-J": "C4-J: C4 with jittered interior vertices (seed 12253)",
    "C5": "C5: 3D H(div) Raviart-Thomas LOR, 32^3 hex per GPU, p=4, div-div+mass",
    "C5-J": "C5-J: C5 with jittered interior vertices (seed 12253)",
    "C4-G": "C4-G: discrete gradient (ND rows x H1 cols) on the C4 mesh, 32^3 hex per GPU, p=4",
    "C5-C": "C5-C: discrete curl (RT rows x ND cols) on the C5 mesh, 32^3 hex per GPU, p=4",
    "C2-A4": "C2-A4: ParCSR split + A4 boundary elimination of the assembled C2 matrix (NEXT-1)",
    "C4-A4": "C4-A4: ParCSR split + A4 boundary elimination of the assembled C4 (ND) matrix (NEXT-1)",
    "C5-A4": "C5-A4: ParCSR split + A4 boundary elimination of the assembled C5 (RT) matrix (NEXT-1)",
    "C2-X": "C2-X: LOR vertex coordinate vectors of the C2 mesh (E-vector -> owned H1 dofs, NEXT-2)",
    "C2-L": "C2-L: the unstructured (legacy) comparator on the C2 workload: LOR mesh as an arbitrary hex mesh, "
            "dense 8x8 cell matrices, direct CSR assembly (PAPER.md l.593-606, NEXT-4)",
    "C2-V": "C2-V: C2 with variable coefficients alpha a(x), beta b(x) given as E-vectors at the LOR vertices (NEXT-3)",
    "C4-V": "C4-V: C4 (ND) with variable coefficients a(x), b(x) at the LOR vertices (NEXT-3)",
    "C5-V": "C5-V: C5 (RT) with variable coefficients a(x), b(x) at the LOR vertices (NEXT-3)",
}
DISCRETE = {"C4-G": ("C4", "grad"), "C5-C": ("C5", "curl")}
# steps after the assembly: A3 layout + A4, coordinate vectors (l.400-404)
AUX = {"C2-A4": ("C2", "a4"), "C4-A4": ("C4", "a4"), "C5-A4": ("C5", "a4"), "C2-X": ("C2", "coords")}
# the paper's own numbers for the discrete operators (context only; 1 V100)
PAPER_DISCRETE_GDOFS = {"grad": 12.0, "curl": 4.5}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, burst copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


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


def algorithmic_bytes(q, dim, p, nel_local, ndpe, space):
    """B_asm = coordinate E-vector + element->dof map (int32, + int8 signs for
    ND/RT) + row_ptr (int64) + col (int32) + val (fp64): what the method itself must move."""
    npts = (p + 1) ** dim
    return (8 * dim * npts * nel_local + (4 + (1 if space != "h1" else 0)) * ndpe * nel_local
            + 8 * (q["n_local"] + 1) + 12 * q["nnz"])


def discrete_bytes(which, nel_local, ndpe, n_rows):
    """B_G = (4 ndpe_H1 + 5 ndpe_ND) nel + 8 (n_ND + 1) + 24 n_ND (2 entries per
    row); B_C = (5 ndpe_ND + 5 ndpe_RT) nel + 8 (n_RT + 1) + 48 n_RT (4 entries per row)."""
    if which == "grad":
        return (4 * ndpe[0] + 5 * ndpe[1]) * nel_local + 8 * (n_rows + 1) + 24 * n_rows
    return (5 * ndpe[1] + 5 * ndpe[2]) * nel_local + 8 * (n_rows + 1) + 48 * n_rows


def host_info():
    info = {}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            if k.strip() in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core", "CPU(s)"):
                info[k.strip()] = v.strip()
        with open("/proc/meminfo") as f:
            info["MemTotal"] = f.readline().split(":")[1].strip()
    except Exception:
        pass
    return info


ORACLE_SNIPPET = r"""
import json, sys, time
import numpy as np
sys.path.insert(0, {root!r})
from oracle import oracle as O
from paper_2210_12253_b200 import meshgen as mg
O.build()
m, form = mg.config_mesh({cfg!r}, n={n})
t0 = time.perf_counter()
if {aux!r} == "coords":
    from oracle import bc
    t0 = time.perf_counter()
    xyz = bc.coordinates(m)
    A = O.Csr(row_ptr=np.zeros(xyz.shape[1] + 1, dtype=np.int64), row_id=None, col=np.zeros(0), val=None, n_cols=0)
elif {aux!r} == "a4":
    from oracle import bc
    A0 = O.assemble(m, form["space"], form["quad"], form["alpha"], form["beta"])
    t0 = time.perf_counter()
    ess = bc.boundary_dofs(m, form["space"])
    n0 = A0.row_ptr.shape[0] - 1
    P = bc.parcsr_split(bc.eliminate(A0, ess), 0, n0, 0, n0)
    A = A0
elif {which!r}:
    A = O.discrete(m, {which!r})
elif {vc!r}:
    xs = [m.X[:, d, :] for d in range(m.dim)]
    ca = 1.0 + 0.5 * np.sin(3.0 * xs[0]) * np.cos(2.0 * xs[1]) + xs[2] * xs[2]
    cb = 2.0 + np.cos(xs[0] + xs[1] + xs[2])
    t0 = time.perf_counter()
    A = O.assemble(m, form["space"], form["quad"], form["alpha"], form["beta"], coef=(ca, cb))
else:
    A = O.assemble(m, form["space"], form["quad"], form["alpha"], form["beta"])
dt = time.perf_counter() - t0
print(json.dumps(dict(rows=int(A.row_ptr.shape[0] - 1), nnz=int(A.nnz), seconds=dt)))
"""


def cpu_baseline(cfg, n):
    """The oracle as it stands (single-threaded C, test infrastructure), pinned to core 0
    (taskset -c 0), on the workload's recipe at n^3 elements (n = 32: the full C2/C4/C5 mesh)."""
    base, which = DISCRETE.get(cfg, (cfg, ""))
    base, aux = AUX.get(cfg, (base, ""))
    vc = cfg.endswith("-V")
    if vc or cfg.endswith("-L"):
        base = cfg[:-2]
    if aux:
        n = min(n, 8 if aux == "a4" else 16)
    code = ORACLE_SNIPPET.format(root=ROOT, cfg=base, n=n, which=which, aux=aux, vc=vc)
    cmd = [sys.executable, "-c", code]
    pinned = False
    try:
        subprocess.run(["taskset", "-c", "0", "true"], check=True, capture_output=True)
        cmd = ["taskset", "-c", "0"] + cmd
        pinned = True
    except Exception:
        pass
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        return {"value": None, "unit": "MDOF/s", "cores": 1, "kind": "oracle", "error": res.stderr[-300:]}
    d = json.loads(res.stdout.strip().splitlines()[-1])
    return {"value": d["rows"] / d["seconds"] / 1e6, "unit": "MDOF/s", "cores": 1, "kind": "oracle",
            "pinned": "taskset -c 0" if pinned else "unpinned",
            "sample": f"{base} recipe at {n}^3 elements{' (the full workload)' if n == 32 and base != 'C3' else ''}: "
                      f"{d['rows']} rows, {d['nnz']} nnz, "
                      f"{'discrete ' + which if which else ('oracle/bc ' + aux) if aux else 'full oracle assembly'} "
                      f"in {d['seconds']:.2f} s",
            "host": host_info()}


def run_reference(args):
    """--impl reference: the CPU oracle on a bounded sample of the workload, per step."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import oracle as O
    from paper_2210_12253_b200 import meshgen as mg
    O.build()
    cfg = args.config
    base, which = DISCRETE.get(cfg, (cfg, ""))
    m, form = mg.config_mesh(base, n=args.ref_n)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        A = O.discrete(m, which) if which else O.assemble(m, form["space"], form["quad"], form["alpha"], form["beta"])
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
                             "sample": f"{base} recipe at {args.ref_n}^3 elements per step"},
            "e2e": {"value": v, "unit": "MDOF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def self_launch(args):
    """--gpus N > 1 without a torchrun environment: re-run this script under torch.distributed.run
    with N ranks on 127.0.0.1 (one process per GPU)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def timed(stream, fn, steps, flush):
    """device time of `steps` calls of fn (CUDA events on the library stream, L2 flushed before each)."""
    import torch
    out = []
    for i in range(steps):
        flush.fill_(float(i))
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        fn()
        b.record(stream)
        b.synchronize()
        out.append(a.elapsed_time(b))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-reassembly", action="store_true")
    ap.add_argument("--cpu-n", type=int, default=None,
                    help="elements per axis of the oracle cpu_baseline run (default: the full mesh, 32; C3: 12)")
    ap.add_argument("--ref-n", type=int, default=12, help="elements per axis per reference-arm step")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(self_launch(args))

    import numpy as np
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

    cfg = args.config.upper()
    base, which = DISCRETE.get(cfg, (cfg, ""))
    base, aux = AUX.get(cfg, (base, ""))
    varcoef = cfg.endswith("-V")
    legacy = cfg.endswith("-L")
    if varcoef or legacy:
        base = cfg[:-2]
    mesh, form = mg.config_mesh(base, gpus=world)
    nid = None
    if world > 1:
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = LOR(mesh, rank=rank, nranks=world, nccl_id=nid, device=local_rank, stream=stream)
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    space = form["space"]
    nel_local = ctx.n_elem_local
    if varcoef:  # smooth coefficient fields sampled at the LOR vertices (the E-vector points)
        e0, e1 = ctx.elem_begin, ctx.elem_begin + nel_local
        xs = [mesh.X[e0:e1, d, :] for d in range(mesh.dim)]
        ca = 1.0 + 0.5 * np.sin(3.0 * xs[0]) * np.cos(2.0 * xs[1]) + xs[2] * xs[2]
        cb = 2.0 + np.cos(xs[0] + xs[1] + xs[2])
        ctx.set_coefficients(ca, cb)
    ndpe = (ctx.ndpe[0], ctx.ndpe[1], ctx.ndpe[2])
    flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)
    aux_bytes = None
    if aux:
        # the post-assembly step on the assembled operator: the matrix is assembled once (untimed), the
        # symbolic split (lor_parcsr_prepare, synchronous) is setup; a step = the numeric split + A4
        q = ctx.query(space)
        ng = q["n_global"]
        if aux == "coords":
            qh = ctx.query("h1")
            q = dict(n_local=qh["n_local"], nnz=0, n_global=qh["n_global"])
            xyz = torch.empty((mesh.dim, qh["n_local"]), dtype=torch.float64, device=dev)

            def step():
                ctx.coordinates(out=xyz)
            aux_bytes = 16 * mesh.dim * qh["n_local"] + 192 * nel_local
        else:
            A = ctx.assemble(space, form["alpha"], form["beta"], form["quad"])
            ctx.sync()
            P = ctx.parcsr(space, A)
            ess = ctx.boundary_dofs(space)
            ctx.sync()
            ep = A[0].cpu()
            ess_h = ess.cpu().long()
            nnz_e = int((ep[ess_h + 1] - ep[ess_h]).sum()) if ess_h.numel() else 0

            def step():
                ctx.parcsr(space, A, out=P, prepared=True)
                ctx.eliminate_bc(space, ess, P)
            aux_bytes = (24 * q["nnz"] + 32 * (q["n_local"] + 1) + q["n_local"] + 4 * ess.numel() + 24 * nnz_e)
        q = dict(n_local=q["n_local"], nnz=q["nnz"], n_global=q["n_global"])
    elif which:
        q = ctx.query_discrete(which)
        ng = q["n_local"]
        if world > 1:
            tt = torch.tensor([ng], dtype=torch.int64, device=dev)
            dist.all_reduce(tt)
            ng = int(tt[0])
        q = dict(n_local=q["n_local"], nnz=q["nnz"], n_global=ng)
        out = ctx.alloc(q["n_local"], q["nnz"])

        def step():
            ctx.discrete(which, out=out)
    elif legacy:
        q = ctx.query(space)
        out = ctx.alloc(q["n_local"], q["nnz"])
        t1 = time.perf_counter()
        ctx.legacy_setup()
        setup_ms += (time.perf_counter() - t1) * 1e3

        def step():
            ctx.legacy_assemble(form["alpha"], form["beta"], out=out)
    else:
        q = ctx.query(space)
        out = ctx.alloc(q["n_local"], q["nnz"])

        def step():
            ctx.assemble(space, form["alpha"], form["beta"], form["quad"], out=out)

    for _ in range(max(args.warmup, 3)):
        step()
    ctx.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    phases = []
    l0 = ctx.launches()
    with ClockSampler(dev.index) as clk:
        step_ms = []
        for i in range(args.steps):
            step_ms += timed(stream, step, 1, flush)
            phases.append(ctx.phase_ms())
    ctx.sync()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches = ctx.launches() - l0
    t_ms = statistics.mean(step_ms)
    if aux:
        fill_ms = t_ms
        kernel = ("k_coords (E-vector -> owned H1 dofs)" if aux == "coords" else
                  "ParCSR fill (k_pc_fill_flat) + A4 (k_bc_mark, k_bc_rows)")
        B = aux_bytes
    elif which:
        fill_ms = t_ms  # the discrete call: row_ptr stride kernel + k_discrete
        kernel = f"discrete {which} (k_discrete, a{8 if which == 'grad' else 9})"
        B = discrete_bytes(which, nel_local, ndpe, q["n_local"])
    elif legacy:
        fill_ms = t_ms
        kernel = "legacy comparator: k_leg_ea + k_leg_rows (count) + k_scan + k_leg_rows (fill)"
        ncell = nel_local * mesh.p ** 3  # broken LOR coordinates + LOR element restriction + CSR
        B = 192 * ncell + 32 * ncell + 8 * (q["n_local"] + 1) + 12 * q["nnz"]
    else:
        # phases: [symbolic + scan, element pass / fill, merge pass, exchange + finalize]
        fill_ms = statistics.mean(p[1] + (p[2] if len(p) > 3 else 0.0) for p in phases)
        kernel = (("fill step a6 = k_xh1_fill" if space == "h1" else "fill step a6 = k_xv_fill")
                  if ctx.fill_path(space) == 1 else "fill step a6 = k_assemble + k_merge_rows")
        B = algorithmic_bytes(q, mesh.dim, mesh.p, nel_local, ndpe[{"h1": 0, "nd": 1, "rt": 2}[space]], space)
        if varcoef:  # + the two coefficient E-vectors
            B += 2 * 8 * (mesh.p + 1) ** mesh.dim * nel_local
    if world > 1:
        tt = torch.tensor([t_ms, fill_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t_ms, fill_ms = float(tt[0]), float(tt[1])
    value = q["n_global"] / (t_ms * 1e-3) / 1e6
    peak, peak_kind = peaks()
    achieved = B / (fill_ms * 1e-3) / 1e9
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_summary.json")
    if os.path.exists(prof):
        try:
            with open(prof) as f:
                traffic = json.load(f).get(cfg, {}).get("fill_dram_bytes")
        except Exception:
            traffic = None

    # ---- numeric-only re-assembly (pattern reuse), same buffers ---------------------------------
    reasm = None
    if not which and not aux and not legacy and not args.no_reassembly:
        def restep():
            ctx.reassemble(space, form["alpha"], form["beta"], form["quad"], out=out)
        for _ in range(3):
            restep()
        ctx.sync()
        rt = statistics.mean(timed(stream, restep, args.steps, flush))
        rphase = ctx.phase_ms()
        if world > 1:
            tt = torch.tensor([rt], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            rt = float(tt[0])
        reasm = {"value": q["n_global"] / (rt * 1e-3) / 1e6, "unit": "MDOF/s", "ms_per_step": rt,
                 "what": "lor_reassemble_* (PAPER.md l.543-546): values only into the pattern of the last full call; "
                         "no symbolic pass, no scan" + ("; col not rewritten" if ctx.fill_path(space) == 1 else ""),
                 "phases_ms": rphase}

    # ---- e2e: pinned host E-vector H2D + the same call + CSR D2H, same public API ---------------
    e2e = None
    if not args.no_e2e and not aux and not legacy:
        e0, e1 = ctx.elem_begin, ctx.elem_begin + nel_local
        Xh = torch.from_numpy(mesh.X[e0:e1].copy()).pin_memory()
        hrp = torch.empty(q["n_local"] + 1, dtype=torch.int64).pin_memory()
        hcol = torch.empty(max(q["nnz"], 1), dtype=torch.int32).pin_memory()
        hval = torch.empty(max(q["nnz"], 1), dtype=torch.float64).pin_memory()

        def e2e_step():
            ctx.update_coordinates(Xh)
            step()
            hrp.copy_(out[0], non_blocking=True)
            hcol.copy_(out[1], non_blocking=True)
            hval.copy_(out[2], non_blocking=True)
        timed(stream, e2e_step, 2, flush)
        te = statistics.mean(timed(stream, e2e_step, max(3, min(args.steps, 10)), flush))
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
            cpu = cpu_baseline(cfg, args.cpu_n or (12 if base.startswith("C3") else 32))
        ph = [statistics.mean(p[i] for p in phases) for i in range(len(phases[0]))] if phases and phases[0] else []
        line = {
            "metric": METRIC, "value": value, "unit": "MDOF/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": t_ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOADS.get(cfg, cfg), "rows_global": q["n_global"],
                       "nnz_per_gpu": q["nnz"], "elements_per_gpu": nel_local, "p": mesh.p,
                       "space": which or space, "l2": "flushed (512 MiB write) before every timed step",
                       "parallelism": f"z-slab x{world}" if world > 1 else "single GPU",
                       "step": ("lor_legacy_assemble_h1 (unstructured comparator, full call)" if legacy else
                                "lor_coordinates" if aux == "coords" else
                                "lor_parcsr_fill + lor_eliminate_bc (boundary dofs of the whole domain)" if aux else
                                ("lor_discrete_" + which) if which else
                                "lor_assemble_" + space + ": symbolic pass + scan + fill (full call, SURVEY P-24)")},
            "hbm_gbs": B / (t_ms * 1e-3) / 1e9,
            "roofline": {"bound": "hbm", "kernel": kernel, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind, "traffic": traffic,
                         "algorithmic_bytes_per_launch": B, "avg_launch_ms": fill_ms,
                         "bytes_model": ("DESIGN.md 4 (B_L = 224 ncell + 8 (n+1) + 12 nnz)" if legacy else
                                         "DESIGN.md 4 (B_X = 16 dim n_H1 + 192 nel)" if aux == "coords" else
                                         "DESIGN.md 4 (B_A4 = 24 nnz + 32 (n+1) + n + 4 n_ess + 24 nnz_ess)" if aux else
                                         "SURVEY 8(d) d.3 (" + ("B_G" if which == "grad" else "B_C" if which else "B_asm") + ")")},
            "phases_ms": ({} if which or aux or legacy else dict(zip(["symbolic+scan", "fill (element pass)", "merge pass",
                                                     "exchange+finalize"], ph))),
            "setup_ms": setup_ms,
            "reassembly": reasm,
            "cpu_baseline": cpu, "e2e": e2e, "gpu_launches": int(launches), "clocks": clk.summary(),
        }
        if which:
            line["paper_context"] = {"value": PAPER_DISCRETE_GDOFS[which] * 1e3, "unit": "MDOF/s",
                                     "hardware": "1x V100 (PAPER.md l.663-664)", "note": "context only"}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
