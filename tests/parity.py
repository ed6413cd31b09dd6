"""Parity helpers shared by the GPU tests (compare the CUDA path with the CPU oracle).

Tolerance rule (reading P-10): entry (i,k) passes iff
    |g - o| <= 1e-12 * max(|o|, 1e-3 * max_k |o_ik|)
patterns (row_ptr, col), dof maps and the discrete operators must be bit-exact.
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-12
FLOOR = 1e-3


def to_host(t):
    return t.detach().cpu().numpy()


def compare_rows(rp, col, val, ref, row_begin=0, rows=None, what=""):
    """rp/col/val: numpy arrays of the GPU CSR (local rows). ref: oracle Csr (global row ids).
    rows: optional list of oracle row positions to check (default: all rows in ref).
    Returns dict with max errors; raises AssertionError with a description on mismatch."""
    ref_rows = ref.row_id
    idx = range(len(ref_rows)) if rows is None else rows
    max_rel = 0.0
    n_checked = 0
    for i in idx:
        g = int(ref_rows[i])
        lr = g - row_begin
        s, e = int(rp[lr]), int(rp[lr + 1])
        os_, oe = int(ref.row_ptr[i]), int(ref.row_ptr[i + 1])
        gc, oc = col[s:e], ref.col[os_:oe]
        if gc.shape != oc.shape or not np.array_equal(gc, oc):
            raise AssertionError(f"{what}: column mismatch in row {g}: gpu {gc.tolist()} oracle {oc.tolist()}")
        gv, ov = val[s:e], ref.val[os_:oe]
        scale = np.maximum(np.abs(ov), FLOOR * np.abs(ov).max(initial=0.0))
        err = np.abs(gv - ov)
        bad = err > RTOL * scale
        if bad.any():
            k = int(np.flatnonzero(bad)[0])
            raise AssertionError(f"{what}: value mismatch row {g} col {oc[k]}: gpu {gv[k]!r} oracle {ov[k]!r} "
                                 f"(rel {err[k] / max(scale[k], 1e-300):.3e})")
        with np.errstate(divide="ignore", invalid="ignore"):
            r = np.where(scale > 0, err / scale, 0.0)
        max_rel = max(max_rel, float(r.max(initial=0.0)))
        n_checked += 1
    return dict(max_rel=max_rel, rows=n_checked)


def compare_full(rp, col, val, ref, row_begin, n_local, what=""):
    """all local rows: row_ptr must match exactly, then every row."""
    sel = np.flatnonzero((ref.row_id >= row_begin) & (ref.row_id < row_begin + n_local))
    assert len(sel) == n_local, f"{what}: oracle has {len(sel)} rows in range, gpu {n_local}"
    ref_rp = ref.row_ptr[sel[0]:sel[-1] + 2] - ref.row_ptr[sel[0]] if n_local else np.zeros(1, np.int64)
    if not np.array_equal(rp[:n_local + 1], ref_rp):
        bad = int(np.flatnonzero(rp[:n_local + 1] != ref_rp)[0])
        raise AssertionError(f"{what}: row_ptr mismatch at local row {bad}: gpu {rp[max(bad-1,0):bad+2]} "
                             f"oracle {ref_rp[max(bad-1,0):bad+2]}")
    return compare_rows(rp, col, val, ref, row_begin, rows=sel, what=what)
