"""Python (ctypes) front end of the CPU oracle -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this module.  The product path (``paper_2210_12253_b200``)
never imports it; the two share only the seeded input generator ``meshgen``.

The arithmetic lives in ``lor_oracle.c`` (plain C, fp64, ``-ffp-contract=off``); this file only
marshals numpy arrays.  See that file's header for what is computed and which passage of
PAPER.md / which SURVEY reading each step follows.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "lor_oracle.c")
LIB = os.path.join(HERE, "liblor_oracle.so")

SPACES = {"h1": 0, "nd": 1, "rt": 2}
QUADS = {"vertex": 0, "gauss2": 1}


def build(force: bool = False) -> str:
    """Compile the oracle (gcc, fp64, no FMA contraction)."""
    if force or not os.path.exists(LIB) or os.path.getmtime(LIB) < os.path.getmtime(SRC):
        tmp = LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fPIC", "-shared", "-o", tmp, SRC,
                               "-lm"])
        os.replace(tmp, LIB)
    return LIB


class _Mesh(C.Structure):
    _fields_ = [("dim", C.c_int), ("p", C.c_int), ("nv", C.c_int64), ("nel", C.c_int64),
                ("elem", C.POINTER(C.c_int64)), ("X", C.POINTER(C.c_double)), ("nranks", C.c_int),
                ("erb", C.POINTER(C.c_int64)), ("ca", C.POINTER(C.c_double)), ("cb", C.POINTER(C.c_double))]


class _Csr(C.Structure):
    _fields_ = [("n_rows", C.c_int64), ("n_cols", C.c_int64), ("nnz", C.c_int64),
                ("row_ptr", C.POINTER(C.c_int64)), ("row_id", C.POINTER(C.c_int64)),
                ("col", C.POINTER(C.c_int32)), ("val", C.POINTER(C.c_double))]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_last_error.restype = C.c_char_p
    return _lib


@dataclass
class Csr:
    row_ptr: np.ndarray   # int64 [n_rows+1]
    row_id: np.ndarray    # int64 [n_rows] global id of each stored row
    col: np.ndarray       # int32
    val: np.ndarray       # float64
    n_cols: int

    @property
    def nnz(self):
        return int(self.col.shape[0])

    def dense(self, n_rows=None):
        n_rows = n_rows if n_rows is not None else int(self.row_id.max()) + 1
        A = np.zeros((n_rows, self.n_cols))
        for r in range(self.row_id.shape[0]):
            s, e = self.row_ptr[r], self.row_ptr[r + 1]
            A[self.row_id[r], self.col[s:e]] = self.val[s:e]
        return A


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError(f"oracle rc={rc}: {lib().orc_last_error().decode()}")


class OracleMesh:
    """Keeps numpy buffers alive while the C struct points into them."""

    def __init__(self, mesh, nranks: int | None = None, coef=None):
        self.dim = mesh.dim
        self.p = mesh.p
        self.elem = np.ascontiguousarray(mesh.elem, dtype=np.int64)
        self.X = np.ascontiguousarray(mesh.X, dtype=np.float64)
        erb = mesh.elem_rank_begin if nranks is None or nranks > 1 else np.array([0, mesh.nel])
        if erb is None:
            erb = np.array([0, mesh.nel])
        self.erb = np.ascontiguousarray(erb, dtype=np.int64)
        self.nranks = len(self.erb) - 1
        # variable coefficients: (a, b) E-vectors [nel][(p+1)^dim] (reading P-28), None = constants
        self.coef = None if coef is None else tuple(np.ascontiguousarray(c, dtype=np.float64) for c in coef)
        ptr = (lambda a: a.ctypes.data_as(C.POINTER(C.c_double))) if coef is not None else None
        self.s = _Mesh(mesh.dim, mesh.p, mesh.nv, mesh.nel, self.elem.ctypes.data_as(C.POINTER(C.c_int64)),
                       self.X.ctypes.data_as(C.POINTER(C.c_double)), self.nranks,
                       self.erb.ctypes.data_as(C.POINTER(C.c_int64)),
                       ptr(self.coef[0]) if coef is not None else None,
                       ptr(self.coef[1]) if coef is not None else None)


def _take(c: _Csr) -> Csr:
    nr, nnz = c.n_rows, c.nnz
    out = Csr(row_ptr=np.ctypeslib.as_array(c.row_ptr, (nr + 1,)).copy(),
              row_id=np.ctypeslib.as_array(c.row_id, (max(nr, 1),)).copy()[:nr],
              col=np.ctypeslib.as_array(c.col, (max(nnz, 1),)).copy()[:nnz],
              val=np.ctypeslib.as_array(c.val, (max(nnz, 1),)).copy()[:nnz], n_cols=int(c.n_cols))
    lib().orc_free(C.byref(c))
    return out


def assemble(mesh, space="h1", quad="vertex", alpha=1.0, beta=1.0, nranks=None, coef=None) -> Csr:
    """O2-O6: the full LOR matrix, all global rows, rank-major ids.  coef = (a, b) coefficient
    E-vectors (variable coefficients alpha a(x), beta b(x)) or None."""
    om = OracleMesh(mesh, nranks, coef)
    c = _Csr()
    _check(lib().orc_assemble(C.byref(om.s), SPACES[space], QUADS[quad], C.c_double(alpha), C.c_double(beta),
                              C.byref(c)))
    return _take(c)


def assemble_rows(mesh, rows, space="h1", quad="vertex", alpha=1.0, beta=1.0, nranks=None, coef=None) -> Csr:
    """O10: the requested global rows only (any size; cost ~ number of rows)."""
    om = OracleMesh(mesh, nranks, coef)
    r = np.ascontiguousarray(np.unique(np.asarray(rows, dtype=np.int64)))
    c = _Csr()
    _check(lib().orc_assemble_rows(C.byref(om.s), SPACES[space], QUADS[quad], C.c_double(alpha), C.c_double(beta),
                                   C.c_int64(r.shape[0]), r.ctypes.data_as(C.POINTER(C.c_int64)), C.byref(c)))
    return _take(c)


def discrete(mesh, which="grad", nranks=None) -> Csr:
    """O7: discrete gradient (ND x H1), curl (RT x ND, 3D) or 2D rotated gradient (RT x H1), all rows."""
    om = OracleMesh(mesh, nranks)
    c = _Csr()
    _check(lib().orc_discrete(C.byref(om.s), {"grad": 0, "curl": 1, "rotgrad": 2}[which], C.byref(c)))
    return _take(c)


def space_size(mesh, space="h1", nranks=None):
    om = OracleMesh(mesh, nranks)
    n = C.c_int64()
    ndpe = C.c_int()
    off = np.zeros(om.nranks + 1, dtype=np.int64)
    _check(lib().orc_space_size(C.byref(om.s), SPACES[space], C.byref(n), C.byref(ndpe),
                                off.ctypes.data_as(C.POINTER(C.c_int64))))
    return int(n.value), int(ndpe.value), off


def dof_map(mesh, space="h1", nranks=None):
    om = OracleMesh(mesh, nranks)
    n, ndpe, _ = space_size(mesh, space, nranks)
    m = np.zeros((mesh.nel, ndpe), dtype=np.int32)
    s = np.zeros((mesh.nel, ndpe), dtype=np.int8)
    _check(lib().orc_dof_map(C.byref(om.s), SPACES[space], m.ctypes.data_as(C.POINTER(C.c_int32)),
                             s.ctypes.data_as(C.POINTER(C.c_int8))))
    return m, s


def topology_counts(mesh):
    om = OracleMesh(mesh)
    cnt = np.zeros(3, dtype=np.int64)
    _check(lib().orc_topology_counts(C.byref(om.s), cnt.ctypes.data_as(C.POINTER(C.c_int64))))
    return tuple(int(v) for v in cnt)


def local_matrix(dim, space, quad, alpha, beta, corners, ca8=None, cb8=None) -> np.ndarray:
    """O4 on one cell: corners [2^dim, dim] in local order a + 2b + 4c; ca8 / cb8 = corner values of the
    variable coefficients (None: constants)."""
    n = {"h1": 1 << dim, "nd": 12 if dim == 3 else 4, "rt": 6 if dim == 3 else 4}[space]
    A = np.zeros((n, n))
    cr = np.ascontiguousarray(corners, dtype=np.float64)
    ap = None if ca8 is None else np.ascontiguousarray(ca8, dtype=np.float64)
    bp = None if cb8 is None else np.ascontiguousarray(cb8, dtype=np.float64)
    dp = lambda a: None if a is None else a.ctypes.data_as(C.POINTER(C.c_double))  # noqa: E731
    _check(lib().orc_local_matrix_vc(C.c_int(dim), SPACES[space], QUADS[quad], C.c_double(alpha), C.c_double(beta),
                                     cr.ctypes.data_as(C.POINTER(C.c_double)), dp(ap), dp(bp),
                                     A.ctypes.data_as(C.POINTER(C.c_double))))
    return A


def gll(p: int):
    x = np.zeros(p + 1)
    w = np.zeros(p + 1)
    lib().orc_gll(C.c_int(p), x.ctypes.data_as(C.POINTER(C.c_double)), w.ctypes.data_as(C.POINTER(C.c_double)))
    return x, w
