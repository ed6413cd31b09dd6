"""Diagnostic sweep on a GPU box: every parity case in its own process (a device fault in one
case cannot poison the others).  Test infrastructure (imports the oracle).

    python scripts/gpu_check.py              # all cases
    python scripts/gpu_check.py --one NAME   # one case (used internally)
"""
import subprocess
import sys
import time
import traceback

sys.path.insert(0, ".")


def cases():
    from paper_2210_12253_b200 import meshgen as mg
    out = [("C1", lambda: mg.config_mesh("C1")[0], "h1", "vertex", 1.0, 0.0)]
    for p in (2, 3, 4):
        out.append((f"h1-2d-p{p}", (lambda p=p: mg.box_mesh(2, (3, 2), p)), "h1", "vertex", 1.0, 1.0))
    import os
    plist = [int(v) for v in os.environ.get("CHECK_P", "1,2,3,4,5,8").split(",")]
    for sp in ("h1", "nd", "rt"):
        for p in plist:
            out.append((f"{sp}-cart-p{p}", (lambda p=p: mg.box_mesh(3, (2, 2, 2), p)), sp, "vertex", 1.0, 1.0))
        out.append((f"{sp}-jitscr-p3", lambda: mg.box_mesh(3, (3, 2, 2), 3, jitter=True, scramble=True), sp, "vertex", 1.0, 1.0))
        out.append((f"{sp}-gauss2-p2", lambda: mg.box_mesh(3, (2, 2, 2), 2, jitter=True), sp, "gauss2", 1.0, 1.0))
    return out


def run_one(name):
    from oracle import oracle as O
    from paper_2210_12253_b200.lor import LOR
    from tests.parity import compare_full, to_host
    for nm, mk, space, quad, a, b in cases():
        if nm != name:
            continue
        t0 = time.time()
        mesh = mk()
        ctx = LOR(mesh)
        q = ctx.query(space)
        rp, col, val = ctx.assemble(space, a, b, quad)
        ctx.sync()
        ref = O.assemble(mesh, space, quad, a, b)
        if q["nnz"] != ref.nnz:
            print(f"  nnz gpu {q['nnz']} oracle {ref.nnz}")
        r = compare_full(to_host(rp), to_host(col), to_host(val), ref, 0, q["n_local"], name)
        print(f"PASS {name}: rows {q['n_local']} nnz {q['nnz']} max_rel {r['max_rel']:.2e} ({time.time()-t0:.1f}s)")
        return


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "--one":
        try:
            run_one(sys.argv[2])
        except Exception as ex:
            print(f"FAIL {sys.argv[2]}: {str(ex)[:600]}")
            traceback.print_exc(limit=3)
            sys.exit(1)
        sys.exit(0)
    from oracle import oracle as O
    O.build()
    san = "--sanitize" in sys.argv
    for nm, *_ in cases():
        cmd = [sys.executable, __file__, "--one", nm]
        if san:
            cmd = ["compute-sanitizer", "--tool", "memcheck", "--print-limit", "5"] + cmd
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=300)
        lines = [l for l in (r.stdout + r.stderr).splitlines() if l.strip()]
        head = [l for l in lines if l.startswith(("PASS", "FAIL", "  nnz", "========="))][:8]
        print("\n".join(head) if head else f"?? {nm}: rc={r.returncode} {lines[-3:]}", flush=True)
        if r.returncode != 0 and not san and "--no-san" not in sys.argv:
            r2 = subprocess.run(["compute-sanitizer", "--tool", "memcheck", "--print-limit", "3"]
                                + [sys.executable, __file__, "--one", nm], capture_output=True, text=True, timeout=600)
            sl = [l for l in (r2.stdout + r2.stderr).splitlines() if l.startswith("=========")][:14]
            print("    " + "\n    ".join(sl), flush=True)
