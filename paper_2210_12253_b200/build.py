"""In-tree build of liblor_b200.so (sm_100a) -- the native library behind the C ABI include/lor.h.

The fused element kernel is instantiated per (dim, space, p); each instantiation is its own
generated translation unit so nvcc runs them in parallel.  Output:
paper_2210_12253_b200/liblor_b200.so (git-ignored, travels to the GPU box with the tree).

    python -m paper_2210_12253_b200.build          # incremental
    LOR_BUILD_P=2,4 python -m ...                   # dev: only some degrees (others -> UNSUPPORTED)
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(ROOT, "build", "lor")
LIB = os.path.join(HERE, "liblor_b200.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-std=c++17", "-O3", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-I", CSRC,
         "-Wno-deprecated-gpu-targets"]

COMBOS = [(2, 0), (3, 0), (3, 1), (3, 2)]  # (dim, space): H1 2D, H1 3D, ND, RT
SPACE_NAME = {0: "SP_H1", 1: "SP_ND", 2: "SP_RT"}


def _sources_hash() -> str:
    h = hashlib.sha256()
    for name in sorted(os.listdir(CSRC)):
        if name.endswith((".cu", ".cuh", ".h", ".cpp")):
            with open(os.path.join(CSRC, name), "rb") as f:
                h.update(name.encode() + f.read())
    with open(os.path.join(ROOT, "include", "lor.h"), "rb") as f:
        h.update(f.read())
    h.update(" ".join(FLAGS + ARCH).encode())
    h.update(os.environ.get("LOR_BUILD_P", "").encode())
    return h.hexdigest()[:16]


def _gen_units(plist):
    os.makedirs(BUILD, exist_ok=True)
    units = []
    for dim, sp in COMBOS:
        for p in range(1, 9):
            name = f"asm_{dim}_{sp}_{p}"
            path = os.path.join(BUILD, name + ".cu")
            if p in plist:
                body = (f'#include "lor_asm.cuh"\nnamespace lorb {{\n'
                        f"cudaError_t launch_asm_{dim}_{sp}_{p}(const AsmArgs &a, int quad, cudaStream_t st, int *smem_out) {{\n"
                        f"  return launch_asm_kz<{dim}, {SPACE_NAME[sp]}, {p}>(a, quad, st, smem_out);\n}}\n}}\n")
            else:
                body = (f'#include "lor_kernels.h"\nnamespace lorb {{\n'
                        f"cudaError_t launch_asm_{dim}_{sp}_{p}(const AsmArgs &, int, cudaStream_t, int *smem_out) {{\n"
                        f"  if (smem_out) *smem_out = 0;\n  return cudaErrorInvalidValue;\n}}\n}}\n")
            old = open(path).read() if os.path.exists(path) else None
            if old != body:
                with open(path, "w") as f:
                    f.write(body)
            units.append(path)
    return units


def _deps(path, seen=None) -> list:
    """Local headers a translation unit includes (transitively), from its #include "..." lines."""
    import re
    seen = set() if seen is None else seen
    for inc in re.findall(r'#include\s+"([^"]+)"', open(path).read()):
        cand = os.path.normpath(os.path.join(os.path.dirname(path), inc))
        if not os.path.exists(cand):
            cand = os.path.join(CSRC, os.path.basename(inc))
        if os.path.exists(cand) and cand not in seen:
            seen.add(cand)
            _deps(cand, seen)
    return sorted(seen)


def _unit_key(src) -> str:
    h = hashlib.sha256()
    for name in [src] + _deps(src):
        with open(name, "rb") as f:
            h.update(os.path.basename(name).encode() + f.read())
    h.update(" ".join(FLAGS + ARCH).encode())
    return h.hexdigest()[:16]


def _compile(src, obj, extra=()):
    key = _unit_key(src)
    kfile = obj + ".key"
    if os.path.exists(obj) and os.path.exists(kfile) and open(kfile).read() == key:
        return obj, False
    cmd = [NVCC] + FLAGS + ARCH + list(extra) + ["-c", src, "-o", obj]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    with open(kfile, "w") as f:
        f.write(key)
    return obj, True


def build(force: bool = False, verbose: bool = True) -> str:
    plist = [int(v) for v in os.environ.get("LOR_BUILD_P", "1,2,3,4,5,6,7,8").split(",") if v.strip()]
    stamp = os.path.join(BUILD, "stamp")
    key = _sources_hash()
    if not force and os.path.exists(LIB) and os.path.exists(stamp) and open(stamp).read() == key:
        return LIB
    units = _gen_units(plist)
    jobs = [(os.path.join(CSRC, "lor_kernels.cu"), os.path.join(BUILD, "lor_kernels.o")),
            (os.path.join(CSRC, "lor_parcsr.cu"), os.path.join(BUILD, "lor_parcsr.o")),
            (os.path.join(CSRC, "lor_legacy.cu"), os.path.join(BUILD, "lor_legacy.o")),
            (os.path.join(CSRC, "lor_vec2d.cu"), os.path.join(BUILD, "lor_vec2d.o")),
            (os.path.join(CSRC, "lor_capi.cu"), os.path.join(BUILD, "lor_capi.o")),
            (os.path.join(CSRC, "lor_plan.cpp"), os.path.join(BUILD, "lor_plan.o")),
            (os.path.join(CSRC, "lor_xframe.cpp"), os.path.join(BUILD, "lor_xframe.o")),
            (os.path.join(CSRC, "lor_xh1.cu"), os.path.join(BUILD, "lor_xh1.o")),
            (os.path.join(CSRC, "lor_xv_nd.cu"), os.path.join(BUILD, "lor_xv_nd.o")),
            (os.path.join(CSRC, "lor_xv_rt.cu"), os.path.join(BUILD, "lor_xv_rt.o"))]
    jobs += [(u, u[:-3] + ".o") for u in units]
    # largest first (ND / high p) for better packing
    jobs.sort(key=lambda j: (("_3_1_" in j[0]) * 10 + ("_3_0_" in j[0]) * 5 + int(j[0][-4]) if "asm_" in j[0]
                             else (200 if "lor_xv" in j[0] else 100)), reverse=True)
    nw = max(1, min(len(jobs), os.cpu_count() or 4))
    if verbose:
        print(f"[lor build] {len(jobs)} translation units on {nw} workers (p in {plist})", flush=True)
    with cf.ThreadPoolExecutor(nw) as ex:
        futs = [ex.submit(_compile, s, o) for s, o in jobs]
        res = [f.result() for f in futs]
    objs = [o for o, _ in res]
    if verbose:
        print(f"[lor build] recompiled {sum(r for _, r in res)} of {len(res)}", flush=True)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC] + ARCH + ["-shared", "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    with open(stamp, "w") as f:
        f.write(key)
    if verbose:
        print(f"[lor build] wrote {LIB}", flush=True)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
