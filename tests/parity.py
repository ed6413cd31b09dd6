"""Parity helpers shared by the GPU tests (compare the CUDA path with the CPU oracle).

Tolerance rule (reading P-10, amended in round 2 as P-10b): entry (i,k) passes iff
    |g - o| <= max(1e-12 * |o|,  64 u * max_k |o_ik|),    u = 2^-53
i.e. 1e-12 relative, except for entries so small against their row (below ~7e-3 of the row max)
that the rounding of the row's large terms dominates them: those are held to the a-priori error
bound of the computation (a sum of <= 8 cells x 8 points of terms bounded by the row max, rounded
independently on both sides; gamma_64 = 64 u).  Patterns (row_ptr, col), dof maps and the discrete
operators must be bit-exact.
"""
from __future__ import annotations

import numpy as np

RTOL = 1e-12
ABS_ROW = 64.0 * 2.0 ** -53          # absolute bound relative to the row max (P-10b)
FLOOR = ABS_ROW / RTOL               # |o| below FLOOR * rowmax: the absolute bound applies


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


def compare_csr_arrays(rp, col, val, ref, row_begin, n_local, what=""):
    """Vectorised compare_full for large matrices: row_ptr and col bit-exact, every value under the
    P-10 rule.  Also reports the entries below the floor (|o| < 1e-3 row max) separately: their
    largest error relative to the row max ("floor_abs") and relative to themselves ("floor_rel",
    informational: cancellation-small entries carry rounding of the row's large terms)."""
    sel = np.flatnonzero((ref.row_id >= row_begin) & (ref.row_id < row_begin + n_local))
    assert len(sel) == n_local, f"{what}: oracle has {len(sel)} rows in range, gpu {n_local}"
    if n_local == 0:
        return dict(max_rel=0.0, rows=0, floor_abs=0.0, floor_rel=0.0)
    assert np.array_equal(ref.row_id[sel], np.arange(row_begin, row_begin + n_local)), \
        f"{what}: oracle rows not the contiguous range"
    assert np.array_equal(sel, np.arange(sel[0], sel[0] + n_local)), f"{what}: oracle rows not stored contiguously"
    s0 = int(ref.row_ptr[sel[0]])
    ref_rp = ref.row_ptr[sel[0]:sel[-1] + 2] - s0
    rp = np.asarray(rp[:n_local + 1])
    if not np.array_equal(rp, ref_rp):
        bad = int(np.flatnonzero(rp != ref_rp)[0])
        raise AssertionError(f"{what}: row_ptr mismatch at local row {bad}: gpu {rp[max(bad-1,0):bad+2]} "
                             f"oracle {ref_rp[max(bad-1,0):bad+2]}")
    nnz = int(ref_rp[-1])
    oc, ov = ref.col[s0:s0 + nnz], ref.val[s0:s0 + nnz]
    gc, gv = np.asarray(col[:nnz]), np.asarray(val[:nnz])
    if not np.array_equal(gc, oc):
        k = int(np.flatnonzero(gc != oc)[0])
        r = int(np.searchsorted(ref_rp, k, side="right") - 1)
        raise AssertionError(f"{what}: column mismatch in local row {r}: gpu {gc[ref_rp[r]:ref_rp[r+1]].tolist()} "
                             f"oracle {oc[ref_rp[r]:ref_rp[r+1]].tolist()}")
    lens = np.diff(ref_rp)
    ao = np.abs(ov)
    rowmax = np.zeros(n_local)
    nz = lens > 0
    rowmax[nz] = np.maximum.reduceat(ao, ref_rp[:-1][nz])
    rm = np.repeat(rowmax, lens)
    scale = np.maximum(ao, FLOOR * rm)
    err = np.abs(gv - ov)
    bad = err > RTOL * scale
    if bad.any():
        k = int(np.flatnonzero(bad)[0])
        r = int(np.searchsorted(ref_rp, k, side="right") - 1)
        raise AssertionError(f"{what}: value mismatch local row {r} col {oc[k]}: gpu {gv[k]!r} oracle {ov[k]!r} "
                             f"(rel {err[k] / max(scale[k], 1e-300):.3e})")
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(scale > 0, err / scale, 0.0)
        fl = ao < FLOOR * rm
        floor_abs = float(np.max(np.where(fl & (rm > 0), err / np.where(rm > 0, rm, 1.0), 0.0), initial=0.0))
        floor_rel = float(np.max(np.where(fl & (ao > 0), err / np.where(ao > 0, ao, 1.0), 0.0), initial=0.0))
    return dict(max_rel=float(rel.max(initial=0.0)), rows=n_local, floor_abs=floor_abs, floor_rel=floor_rel)
