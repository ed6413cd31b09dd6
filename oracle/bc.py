"""Oracle for the steps after the local assembly -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s cpu_baseline / --impl reference legs
may import this module; the product path never does.  Plain numpy definitions, written from the
paper and DESIGN.md readings P-26..P-28, no blocking or reordering:

* ``boundary_dofs``   the essential dofs of a trace condition on the whole domain boundary: the dofs
                      whose LOR entity lies on a boundary facet (a face of exactly one element; an
                      edge in 2D), found from each element's own local lattice (H1: points with
                      x_n in {0, p}; ND: edges along s != n with x_n in {0, p}; RT: faces normal to
                      n with x_n in {0, p}), mapped through the oracle's own dof map.
* ``eliminate``       Step A4 (l.376-380): rows and columns of the essential dofs eliminated, the
                      diagonal entry replaced by 1, the pattern kept.
* ``parcsr_split``    the ParCSR layout (l.369-370): diag block (columns owned by the rank, local
                      ids, diagonal first then ascending for square operators -- hypre's
                      convention, reading P-26) and offd block (col_map_offd = ascending distinct
                      off-rank columns, offd column = index into it).
* ``coordinates``     the LOR vertex coordinate vectors (l.400-404): the E-vector value of every H1
                      dof, taken from the minimal element containing it (reading P-27).
"""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def _facet_keys(mesh):
    """(element, axis n, side) -> sorted vertex tuple of the element's local facet."""
    dim = mesh.dim
    nc = 1 << dim
    keys = {}
    for e in range(mesh.nel):
        for n in range(dim):
            for side in (0, 1):
                corners = [v for v in range(nc) if ((v >> n) & 1) == side]
                keys[(e, n, side)] = tuple(sorted(int(mesh.elem[e, v]) for v in corners))
    return keys


def _local_on_facet(dim, p, space, n, side):
    """macro-element local dofs lying on the local facet (axis n, side) -- App. A.3 local orders."""
    xn = side * p
    out = []
    if space == "h1":
        ext = [p + 1] * dim
        for l in range(int(np.prod(ext))):
            x = [(l // int(np.prod(ext[:a]))) % ext[a] for a in range(dim)]
            if x[n] == xn:
                out.append(l)
        return out
    # vector spaces: family a, extents (ND: p along a, p+1 elsewhere; RT: p+1 along a, p elsewhere)
    off = 0
    for a in range(dim):
        ext = [(p if b == a else p + 1) if space == "nd" else (p + 1 if b == a else p) for b in range(dim)]
        tangential = (a != n) if space == "nd" else (a == n)
        for r in range(int(np.prod(ext))):
            x = [r % ext[0], (r // ext[0]) % ext[1]] + ([r // (ext[0] * ext[1])] if dim == 3 else [])
            if tangential and x[n] == xn:
                out.append(off + r)
        off += int(np.prod(ext))
    return out


def boundary_dofs(mesh, space="h1", nranks=None) -> np.ndarray:
    """Global (rank-major) ids of the dofs on the domain boundary, ascending."""
    keys = _facet_keys(mesh)
    count = {}
    for k in keys.values():
        count[k] = count.get(k, 0) + 1
    m, _ = O.dof_map(mesh, space, nranks)
    ids = set()
    for (e, n, side), k in keys.items():
        if count[k] == 1:
            for l in _local_on_facet(mesh.dim, mesh.p, space, n, side):
                ids.add(int(m[e, l]))
    return np.array(sorted(ids), dtype=np.int64)


def eliminate(A: O.Csr, ess) -> O.Csr:
    """A4: for essential j, row j -> unit row (1 on the diagonal, explicit 0 elsewhere) and column j
    -> 0 in every other row.  A holds global rows ``A.row_id`` with global columns."""
    ess = np.zeros(A.n_cols, dtype=bool) if len(ess) == 0 else np.isin(np.arange(A.n_cols), ess)
    rows = np.repeat(A.row_id, np.diff(A.row_ptr))
    val = A.val.copy()
    kill = ess[rows] | ess[A.col]
    val[kill] = 0.0
    val[ess[rows] & (A.col == rows)] = 1.0
    return O.Csr(row_ptr=A.row_ptr.copy(), row_id=A.row_id.copy(), col=A.col.copy(), val=val, n_cols=A.n_cols)


def parcsr_split(A: O.Csr, row_begin, n_local, col_begin, col_end, square=True) -> dict:
    """ParCSR blocks of global rows [row_begin, row_begin + n_local) of A."""
    sel = np.nonzero((A.row_id >= row_begin) & (A.row_id < row_begin + n_local))[0]
    assert np.array_equal(A.row_id[sel], np.arange(row_begin, row_begin + n_local))
    dr, dc, dv, orr, oc, ov = [0], [], [], [0], [], []
    offd_cols = set()
    for i in sel:
        s, e = A.row_ptr[i], A.row_ptr[i + 1]
        for c in A.col[s:e]:
            if not (col_begin <= c < col_end):
                offd_cols.add(int(c))
    col_map = np.array(sorted(offd_cols), dtype=np.int64)
    where = {int(c): k for k, c in enumerate(col_map)}
    for i in sel:
        g = int(A.row_id[i])
        s, e = A.row_ptr[i], A.row_ptr[i + 1]
        d = [(int(c) - col_begin, float(v)) for c, v in zip(A.col[s:e], A.val[s:e]) if col_begin <= c < col_end]
        if square:
            d = [x for x in d if x[0] == g - col_begin] + [x for x in d if x[0] != g - col_begin]
        dc += [x[0] for x in d]
        dv += [x[1] for x in d]
        dr.append(len(dc))
        o = [(where[int(c)], float(v)) for c, v in zip(A.col[s:e], A.val[s:e]) if not (col_begin <= c < col_end)]
        oc += [x[0] for x in o]
        ov += [x[1] for x in o]
        orr.append(len(oc))
    return dict(diag_row_ptr=np.array(dr, dtype=np.int64), diag_col=np.array(dc, dtype=np.int32),
                diag_val=np.array(dv, dtype=np.float64), offd_row_ptr=np.array(orr, dtype=np.int64),
                offd_col=np.array(oc, dtype=np.int32), offd_val=np.array(ov, dtype=np.float64), col_map_offd=col_map)


def coordinates(mesh, nranks=None) -> np.ndarray:
    """[dim, n_global] LOR vertex coordinates: for every H1 dof the E-vector value in the minimal
    element containing it."""
    m, _ = O.dof_map(mesh, "h1", nranks)
    n = int(m.max()) + 1
    out = np.full((mesh.dim, n), np.nan)
    done = np.zeros(n, dtype=bool)
    for e in range(mesh.nel):
        for l in range(m.shape[1]):
            g = m[e, l]
            if not done[g]:
                out[:, g] = mesh.X[e, :, l]
                done[g] = True
    return out
