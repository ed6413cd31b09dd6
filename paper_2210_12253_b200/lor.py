"""Thin Python binding of the C ABI in include/lor.h (argument marshalling only).

Every step of the assembly runs in liblor_b200.so (hand-written sm_100a kernels).  There is no
CPU or PyTorch fallback: if the library or a GPU is missing, constructing ``LOR`` raises.
PyTorch provides device memory (the caller-owned output buffers) and the CUDA stream.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liblor_b200.so")

H1, ND, RT = 0, 1, 2
SPACES = {"h1": H1, "nd": ND, "rt": RT}
QUADS = {"vertex": 0, "gauss2": 1}
STATUS = {0: "OK", 1: "INVALID_ARGUMENT", 2: "DEGENERATE_GEOMETRY", 3: "OUT_OF_MEMORY", 4: "CUDA", 5: "NCCL",
          6: "UNSUPPORTED", 7: "BUFFER_TOO_SMALL"}


class LorError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"lor error {STATUS.get(code, code)}: {msg}")
        self.code = code


class _SetupArgs(C.Structure):
    _fields_ = [("dim", C.c_int), ("p", C.c_int), ("n_vert", C.c_int64), ("vert_xyz", C.c_void_p),
                ("n_elem", C.c_int64), ("elem_vert", C.c_void_p), ("elem_nodes", C.c_void_p), ("rank", C.c_int),
                ("nranks", C.c_int), ("elem_rank_begin", C.c_void_p), ("nccl_unique_id", C.c_void_p),
                ("cuda_stream", C.c_void_p), ("device", C.c_int), ("space_mask", C.c_int)]


class _Csr(C.Structure):
    _fields_ = [("row_ptr", C.c_void_p), ("col", C.c_void_p), ("val", C.c_void_p), ("cap_nnz", C.c_int64)]


class _ParCsr(C.Structure):
    _fields_ = [("diag_row_ptr", C.c_void_p), ("diag_col", C.c_void_p), ("diag_val", C.c_void_p),
                ("cap_diag", C.c_int64), ("offd_row_ptr", C.c_void_p), ("offd_col", C.c_void_p),
                ("offd_val", C.c_void_p), ("cap_offd", C.c_int64), ("col_map_offd", C.c_void_p),
                ("cap_col_map", C.c_int64)]


OPS = {"h1": 0, "nd": 1, "rt": 2, "grad": 3, "curl": 4, "rotgrad": 5}


_lib = None


def lib():
    """Load liblor_b200.so from the package directory (never a fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise LorError(-1, f"{LIB_PATH} not built; run python -m paper_2210_12253_b200.build")
        L = C.CDLL(LIB_PATH)
        L.lor_last_error.restype = C.c_char_p
        L.lor_kernel_launches.restype = C.c_int64
        L.lor_setup.argtypes = [C.POINTER(_SetupArgs), C.POINTER(C.c_void_p)]
        for name in ("lor_destroy", "lor_sync"):
            getattr(L, name).argtypes = [C.c_void_p]
        L.lor_last_error.argtypes = [C.c_void_p]
        L.lor_kernel_launches.argtypes = [C.c_void_p]
        L.lor_query.argtypes = [C.c_void_p, C.c_int] + [C.POINTER(C.c_int64)] * 4
        L.lor_query_discrete.argtypes = [C.c_void_p, C.c_int] + [C.POINTER(C.c_int64)] * 3
        for name in ("lor_assemble_h1", "lor_assemble_nd", "lor_assemble_rt", "lor_reassemble_h1", "lor_reassemble_nd",
                     "lor_reassemble_rt"):
            getattr(L, name).argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_int, C.POINTER(_Csr)]
        L.lor_discrete_grad.argtypes = [C.c_void_p, C.POINTER(_Csr)]
        L.lor_discrete_curl.argtypes = [C.c_void_p, C.POINTER(_Csr)]
        L.lor_discrete_rotgrad.argtypes = [C.c_void_p, C.POINTER(_Csr)]
        L.lor_dof_map.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.lor_query_elements.argtypes = [C.c_void_p, C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                         C.POINTER(C.c_int), C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.lor_nccl_get_unique_id.argtypes = [C.c_void_p]
        L.lor_set_exchange.argtypes = [C.c_void_p, C.c_int]
        L.lor_exchange_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.lor_assemble_finish.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Csr)]
        L.lor_plan_dry_run.argtypes = [C.POINTER(_SetupArgs), C.c_void_p, C.c_void_p, C.c_void_p]
        L.lor_xframe_dry_run.argtypes = [C.POINTER(_SetupArgs), C.c_void_p, C.c_void_p, C.c_void_p]
        L.lor_debug_dump.restype = C.c_int64
        L.lor_debug_dump.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int64]
        L.lor_update_coordinates.argtypes = [C.c_void_p, C.c_void_p]
        L.lor_last_phase_ms.argtypes = [C.c_void_p, C.POINTER(C.c_float), C.c_int]
        L.lor_fill_path.argtypes = [C.c_void_p, C.c_int]
        L.lor_query_transpose.argtypes = [C.c_void_p, C.c_int, C.POINTER(C.c_int64)]
        L.lor_dof_transpose.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int64]
        L.lor_parcsr_prepare.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Csr)] + [C.POINTER(C.c_int64)] * 3
        L.lor_parcsr_fill.argtypes = [C.c_void_p, C.c_int, C.POINTER(_Csr), C.POINTER(_ParCsr)]
        L.lor_boundary_dofs.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        L.lor_eliminate_bc.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, C.POINTER(_ParCsr)]
        L.lor_bc_exchange_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_int]
        L.lor_eliminate_bc_finish.argtypes = [C.c_void_p, C.c_int, C.POINTER(_ParCsr)]
        L.lor_parcsr_exchange_counts.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
        L.lor_coordinates.argtypes = [C.c_void_p, C.c_void_p]
        L.lor_set_coefficients.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.lor_set_coefficients_global.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.lor_legacy_setup.argtypes = [C.c_void_p]
        L.lor_legacy_assemble_h1.argtypes = [C.c_void_p, C.c_double, C.c_double, C.POINTER(_Csr)]
        _lib = L
    return _lib


def nccl_unique_id() -> bytes:
    buf = (C.c_char * 128)()
    rc = lib().lor_nccl_get_unique_id(buf)
    if rc:
        raise LorError(rc, "ncclGetUniqueId")
    return bytes(buf)


def plan_dry_run(mesh, rank=0, nranks=1, elem_rank_begin=None):
    """Host-only plan of one rank (no GPU): returns (info[3][8], send[3][nranks], recv[3][nranks])."""
    vert = np.ascontiguousarray(mesh.vert, dtype=np.float64)
    elem = np.ascontiguousarray(mesh.elem, dtype=np.int64)
    erb = elem_rank_begin if elem_rank_begin is not None else mesh.elem_rank_begin
    erb = np.ascontiguousarray(erb if nranks > 1 else [0, elem.shape[0]], dtype=np.int64)
    a = _SetupArgs()
    a.dim, a.p = int(mesh.dim), int(mesh.p)
    a.n_vert, a.vert_xyz = vert.shape[0], vert.ctypes.data
    a.n_elem, a.elem_vert = elem.shape[0], elem.ctypes.data
    a.elem_nodes = None
    a.rank, a.nranks = rank, nranks
    a.elem_rank_begin = erb.ctypes.data
    info = np.zeros((3, 8), dtype=np.int64)
    send = np.zeros((3, nranks), dtype=np.int64)
    recv = np.zeros((3, nranks), dtype=np.int64)
    rc = lib().lor_plan_dry_run(C.byref(a), info.ctypes.data, send.ctypes.data, recv.ctypes.data)
    if rc:
        raise LorError(rc, lib().lor_last_error(None).decode())
    return info, send, recv


def xframe_dry_run(mesh, rank=0, nranks=1):
    """Host-only extended-frame plan of one rank (no GPU): (info[4], send[nranks], recv[nranks]) --
    lor_xframe_dry_run: regular neighbourhood, ghost layer size, largest cell box, local elements."""
    vert = np.ascontiguousarray(mesh.vert, dtype=np.float64)
    elem = np.ascontiguousarray(mesh.elem, dtype=np.int64)
    erb = np.ascontiguousarray(mesh.elem_rank_begin if nranks > 1 else [0, elem.shape[0]], dtype=np.int64)
    a = _SetupArgs()
    a.dim, a.p = int(mesh.dim), int(mesh.p)
    a.n_vert, a.vert_xyz = vert.shape[0], vert.ctypes.data
    a.n_elem, a.elem_vert = elem.shape[0], elem.ctypes.data
    a.elem_nodes = None
    a.rank, a.nranks = rank, nranks
    a.elem_rank_begin = erb.ctypes.data
    info = np.zeros(4, dtype=np.int64)
    send = np.zeros(nranks, dtype=np.int64)
    recv = np.zeros(nranks, dtype=np.int64)
    rc = lib().lor_xframe_dry_run(C.byref(a), info.ctypes.data, send.ctypes.data, recv.ctypes.data)
    if rc:
        raise LorError(rc, lib().lor_last_error(None).decode())
    return info, send, recv


class LOR:
    """One context per rank/GPU.  ``mesh`` provides ``dim, p, vert, elem, X`` (numpy)."""

    def __init__(self, mesh, *, rank=0, nranks=1, elem_rank_begin=None, nccl_id: bytes | None = None,
                 stream=None, device=None, use_evector=True, spaces=None):
        import torch
        if not torch.cuda.is_available():
            raise LorError(4, "no CUDA device: the LOR library has no CPU path")
        self.torch = torch
        self.device = torch.device("cuda", device if device is not None else torch.cuda.current_device())
        self.stream = stream if stream is not None else torch.cuda.current_stream(self.device)
        self.dim, self.p = int(mesh.dim), int(mesh.p)
        self._vert = np.ascontiguousarray(mesh.vert, dtype=np.float64)
        self._elem = np.ascontiguousarray(mesh.elem, dtype=np.int64)
        self._X = np.ascontiguousarray(mesh.X, dtype=np.float64) if use_evector else None
        erb = elem_rank_begin if elem_rank_begin is not None else (
            mesh.elem_rank_begin if (nranks > 1 and getattr(mesh, "elem_rank_begin", None) is not None) else None)
        self._erb = np.ascontiguousarray(erb, dtype=np.int64) if erb is not None else None
        self._nccl = C.create_string_buffer(nccl_id, 128) if nccl_id is not None else None
        a = _SetupArgs()
        a.dim, a.p = self.dim, self.p
        a.n_vert = self._vert.shape[0]
        a.vert_xyz = self._vert.ctypes.data
        a.n_elem = self._elem.shape[0]
        a.elem_vert = self._elem.ctypes.data
        a.elem_nodes = self._X.ctypes.data if self._X is not None else None
        a.rank, a.nranks = rank, nranks
        a.elem_rank_begin = self._erb.ctypes.data if self._erb is not None else None
        a.nccl_unique_id = C.cast(self._nccl, C.c_void_p) if self._nccl is not None else None
        a.cuda_stream = self.stream.cuda_stream
        a.device = self.device.index
        # spaces to set up (None: all); H1 always (its frame records serve the vector spaces)
        a.space_mask = 0 if spaces is None else sum(1 << SPACES[x] for x in set(spaces) | {"h1"})
        h = C.c_void_p()
        rc = lib().lor_setup(C.byref(a), C.byref(h))
        if rc:
            raise LorError(rc, lib().lor_last_error(None).decode())
        self.h = h
        self.rank, self.nranks = rank, nranks
        eb, ne = C.c_int64(), C.c_int64()
        n1, n2, n3 = C.c_int(), C.c_int(), C.c_int()
        self._check(lib().lor_query_elements(self.h, C.byref(eb), C.byref(ne), C.byref(n1), C.byref(n2), C.byref(n3)))
        self.elem_begin, self.n_elem_local = eb.value, ne.value
        self.ndpe = {H1: n1.value, ND: n2.value, RT: n3.value}

    # ------------------------------------------------------------------ plumbing
    def _check(self, rc):
        if rc:
            raise LorError(rc, lib().lor_last_error(self.h).decode())

    def close(self):
        if getattr(self, "h", None):
            lib().lor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def sync(self):
        self._check(lib().lor_sync(self.h))

    def launches(self) -> int:
        return int(lib().lor_kernel_launches(self.h))

    def fill_path(self, space="h1") -> int:
        """1: extended-frame single-pass fill, 0: element pass + merge pass, 2: per-row path (3D, p = 1,
        one rank, every space) -- lor_fill_path."""
        return int(lib().lor_fill_path(self.h, SPACES[space]))

    def phase_ms(self):
        buf = (C.c_float * 8)()
        n = lib().lor_last_phase_ms(self.h, buf, 8)
        return [buf[i] for i in range(n)]

    def update_coordinates(self, X_local):
        """X_local: this rank's E-vector slice, a torch tensor (pinned host or device) or numpy array."""
        ptr = X_local.data_ptr() if hasattr(X_local, "data_ptr") else X_local.ctypes.data
        self._check(lib().lor_update_coordinates(self.h, C.c_void_p(ptr)))

    def debug_dump(self, what, space="h1", cap=1 << 26):
        buf = np.zeros(cap, dtype=np.uint8)
        n = lib().lor_debug_dump(self.h, what, SPACES.get(space, space), buf.ctypes.data, cap)
        return buf[:n]

    def set_exchange(self, mode: int):
        self._check(lib().lor_set_exchange(self.h, mode))

    # ------------------------------------------------------------------ queries
    def query(self, space):
        sp = SPACES.get(space, space)
        v = [C.c_int64() for _ in range(4)]
        self._check(lib().lor_query(self.h, sp, *[C.byref(x) for x in v]))
        return dict(n_local=v[0].value, row_begin=v[1].value, n_global=v[2].value, nnz=v[3].value)

    def query_discrete(self, which):
        w = {"grad": 0, "curl": 1, "rotgrad": 2}.get(which, which)
        v = [C.c_int64() for _ in range(3)]
        self._check(lib().lor_query_discrete(self.h, w, *[C.byref(x) for x in v]))
        return dict(n_local=v[0].value, nnz=v[1].value, n_cols=v[2].value)

    # ------------------------------------------------------------------ outputs
    def alloc(self, n_rows, nnz):
        t = self.torch
        return (t.empty(n_rows + 1, dtype=t.int64, device=self.device), t.empty(max(nnz, 1), dtype=t.int32, device=self.device),
                t.empty(max(nnz, 1), dtype=t.float64, device=self.device))

    @staticmethod
    def _csr(rp, col, val):
        c = _Csr()
        c.row_ptr, c.col, c.val = rp.data_ptr(), col.data_ptr(), val.data_ptr()
        c.cap_nnz = col.numel()
        return c

    def assemble(self, space="h1", alpha=1.0, beta=1.0, quad="vertex", out=None):
        """Enqueue LOR assembly on the context stream; returns (row_ptr, col, val) device tensors."""
        sp = SPACES.get(space, space)
        q = self.query(sp)
        if out is None:
            out = self.alloc(q["n_local"], q["nnz"])
        fn = (lib().lor_assemble_h1, lib().lor_assemble_nd, lib().lor_assemble_rt)[sp]
        self._check(fn(self.h, C.c_double(alpha), C.c_double(beta), QUADS.get(quad, quad), C.byref(self._csr(*out))))
        return out

    def reassemble(self, space="h1", alpha=1.0, beta=1.0, quad="vertex", out=None):
        """Numeric-only re-assembly into ``out`` = the buffers of an earlier ``assemble`` of the same
        space and rule (pattern reuse, lor_reassemble_*): values from the current coordinates."""
        sp = SPACES.get(space, space)
        fn = (lib().lor_reassemble_h1, lib().lor_reassemble_nd, lib().lor_reassemble_rt)[sp]
        self._check(fn(self.h, C.c_double(alpha), C.c_double(beta), QUADS.get(quad, quad), C.byref(self._csr(*out))))
        return out

    def exchange_copy_from(self, src: "LOR", space):
        self._check(lib().lor_exchange_copy(self.h, src.h, SPACES.get(space, space)))

    def assemble_finish(self, space, out):
        self._check(lib().lor_assemble_finish(self.h, SPACES.get(space, space), C.byref(self._csr(*out))))

    def discrete(self, which="grad", out=None):
        q = self.query_discrete(which)
        if out is None:
            out = self.alloc(q["n_local"], q["nnz"])
        fn = {"grad": lib().lor_discrete_grad, 0: lib().lor_discrete_grad, "curl": lib().lor_discrete_curl,
              1: lib().lor_discrete_curl, "rotgrad": lib().lor_discrete_rotgrad, 2: lib().lor_discrete_rotgrad}[which]
        self._check(fn(self.h, C.byref(self._csr(*out))))
        return out

    def dof_transpose(self, space="h1"):
        """(offsets[n_local+1] int64, entries int32) device tensors: per owned row the ascending
        local element * ndpe + local dof pairs of this rank's elements (lor_dof_transpose)."""
        t = self.torch
        sp = SPACES.get(space, space)
        n = C.c_int64()
        self._check(lib().lor_query_transpose(self.h, sp, C.byref(n)))
        q = self.query(sp)
        off = t.empty(q["n_local"] + 1, dtype=t.int64, device=self.device)
        ent = t.empty(max(n.value, 1), dtype=t.int32, device=self.device)
        self._check(lib().lor_dof_transpose(self.h, sp, C.c_void_p(off.data_ptr()), C.c_void_p(ent.data_ptr()),
                                            C.c_int64(ent.numel())))
        return off, ent[:n.value]

    def dof_map(self, space="h1"):
        t = self.torch
        sp = SPACES.get(space, space)
        n = self.ndpe[sp]
        m = t.empty((self.n_elem_local, n), dtype=t.int32, device=self.device)
        s = t.empty((self.n_elem_local, n), dtype=t.int8, device=self.device)
        self._check(lib().lor_dof_map(self.h, sp, C.c_void_p(m.data_ptr()), C.c_void_p(s.data_ptr())))
        return m, s

    # ------------------------------------------------------------------ A3 layout / A4 (NEXT-1)
    def parcsr(self, op, A, out=None, prepared=False):
        """hypre-style split of the assembled operator ``A`` = (row_ptr, col, val) of ``op`` ("h1", "nd",
        "rt", "grad", "curl"): lor_parcsr_prepare (synchronous sizes) + lor_parcsr_fill.  Returns a
        dict of device tensors diag_row_ptr, diag_col, diag_val, offd_row_ptr, offd_col, offd_val,
        col_map_offd (``out`` = such a dict to reuse)."""
        t = self.torch
        o = OPS.get(op, op)
        a = self._csr(*A)
        if prepared and out is not None:  # numeric part only (same operator, same pattern)
            self._check(lib().lor_parcsr_fill(self.h, o, C.byref(a), C.byref(self._pcsr(out))))
            return out
        v = [C.c_int64() for _ in range(3)]
        self._check(lib().lor_parcsr_prepare(self.h, o, C.byref(a), *[C.byref(x) for x in v]))
        nd, no, nc = (x.value for x in v)
        n = A[0].numel() - 1
        if out is None:
            out = dict(diag_row_ptr=t.empty(n + 1, dtype=t.int64, device=self.device),
                       diag_col=t.empty(max(nd, 1), dtype=t.int32, device=self.device),
                       diag_val=t.empty(max(nd, 1), dtype=t.float64, device=self.device),
                       offd_row_ptr=t.empty(n + 1, dtype=t.int64, device=self.device),
                       offd_col=t.empty(max(no, 1), dtype=t.int32, device=self.device),
                       offd_val=t.empty(max(no, 1), dtype=t.float64, device=self.device),
                       col_map_offd=t.empty(max(nc, 1), dtype=t.int64, device=self.device))
        out["sizes"] = (nd, no, nc)
        self._check(lib().lor_parcsr_fill(self.h, o, C.byref(a), C.byref(self._pcsr(out))))
        return out

    @staticmethod
    def _pcsr(M):
        m = _ParCsr()
        m.diag_row_ptr, m.diag_col, m.diag_val = (M[k].data_ptr() for k in ("diag_row_ptr", "diag_col", "diag_val"))
        m.offd_row_ptr, m.offd_col, m.offd_val = (M[k].data_ptr() for k in ("offd_row_ptr", "offd_col", "offd_val"))
        m.col_map_offd = M["col_map_offd"].data_ptr()
        m.cap_diag, m.cap_offd, m.cap_col_map = M["diag_col"].numel(), M["offd_col"].numel(), M["col_map_offd"].numel()
        return m

    def boundary_dofs(self, space="h1"):
        """int32 device tensor: local rows of the owned dofs on the domain boundary (lor_boundary_dofs)."""
        t = self.torch
        sp = SPACES.get(space, space)
        n = C.c_int64()
        self._check(lib().lor_boundary_dofs(self.h, sp, None, 0, C.byref(n)))
        rows = t.empty(max(n.value, 1), dtype=t.int32, device=self.device)
        self._check(lib().lor_boundary_dofs(self.h, sp, C.c_void_p(rows.data_ptr()), C.c_int64(rows.numel()),
                                            C.byref(n)))
        return rows[:n.value]

    def eliminate_bc(self, space, ess, M):
        """Step A4 on the ParCSR ``M`` of ``space`` (lor_eliminate_bc); ``ess`` = int32 device tensor."""
        self._check(lib().lor_eliminate_bc(self.h, SPACES.get(space, space), C.c_void_p(ess.data_ptr()),
                                           C.c_int64(ess.numel()), C.byref(self._pcsr(M))))

    def bc_exchange_copy_from(self, src: "LOR", space):
        self._check(lib().lor_bc_exchange_copy(self.h, src.h, SPACES.get(space, space)))

    def eliminate_bc_finish(self, space, M):
        self._check(lib().lor_eliminate_bc_finish(self.h, SPACES.get(space, space), C.byref(self._pcsr(M))))

    def parcsr_exchange_counts(self, space):
        s = np.zeros(self.nranks, dtype=np.int64)
        r = np.zeros(self.nranks, dtype=np.int64)
        self._check(lib().lor_parcsr_exchange_counts(self.h, SPACES.get(space, space), s.ctypes.data, r.ctypes.data))
        return s, r

    def coordinates(self, out=None):
        """LOR vertex coordinate vectors of the owned H1 dofs: device tensor [dim, n_local] (lor_coordinates)."""
        t = self.torch
        q = self.query("h1")
        if out is None:
            out = t.empty((self.dim, max(q["n_local"], 1)), dtype=t.float64, device=self.device)
        self._check(lib().lor_coordinates(self.h, C.c_void_p(out.data_ptr())))
        return out[:, :q["n_local"]]

    # ------------------------------------------------------------------ variable coefficients (NEXT-3)
    def set_coefficients(self, a=None, b=None):
        """Coefficient E-vectors a(x), b(x) [n_elem_local, (p+1)^dim] of this rank's elements (numpy or
        torch, host or device) multiplying alpha / beta in later assemblies; None, None = constants."""
        if a is None and b is None:
            self._check(lib().lor_set_coefficients(self.h, None, None))
            self._coef = None
            return
        t = self.torch
        conv = lambda x: (x if isinstance(x, t.Tensor) else t.from_numpy(np.ascontiguousarray(x, dtype=np.float64))  # noqa: E731
                          ).to(dtype=t.float64).contiguous()
        a, b = conv(a), conv(b)
        self._coef = (a, b)  # keep alive until the copy on the context stream has run
        self._check(lib().lor_set_coefficients(self.h, C.c_void_p(a.data_ptr()), C.c_void_p(b.data_ptr())))
        self.sync()

    def set_coefficients_global(self, a, b):
        """Coefficient E-vectors of the WHOLE mesh [n_elem, (p+1)^dim] (host numpy): the context keeps its
        local elements' and its ghost layer's (extended frames across ranks)."""
        a = np.ascontiguousarray(a, dtype=np.float64)
        b = np.ascontiguousarray(b, dtype=np.float64)
        self._check(lib().lor_set_coefficients_global(self.h, a.ctypes.data, b.ctypes.data))

    # ------------------------------------------------------------------ unstructured comparator (NEXT-4)
    def legacy_setup(self):
        """LOR mesh as an unstructured mesh: element restriction, broken coordinates, transpose."""
        self._check(lib().lor_legacy_setup(self.h))

    def legacy_assemble(self, alpha=1.0, beta=1.0, out=None):
        """The unstructured comparator's H1 assembly (lor_legacy_assemble_h1, vertex rule)."""
        q = self.query("h1")
        if out is None:
            out = self.alloc(q["n_local"], q["nnz"])
        self._check(lib().lor_legacy_assemble_h1(self.h, C.c_double(alpha), C.c_double(beta), C.byref(self._csr(*out))))
        return out
