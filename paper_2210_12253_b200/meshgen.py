"""Seeded synthetic mesh generator -- the ONE module shared by the oracle and the CUDA path.

It produces the *inputs* of the LOR assembly problem and nothing else:

* a coarse tensor-product (quad/hex) mesh: vertex coordinates and element-to-vertex
  connectivity with the local corner order ``a + 2b (+ 4c)``;
* the high-order coordinate **E-vector** ``X[nel][dim][(p+1)^dim]`` -- the mesh nodes at the
  tensor Gauss--Lobatto points of each element, stored contiguously per element
  (Step A1: "the mesh coordinates are represented as high-order
  E-vectors, where all the coordinates corresponding to a macro element are stored
  contiguously").  The LOR vertices are these points (Sec. 2.1).

It holds none of the method's arithmetic (no numbering, no local matrices, no assembly).
The Gauss--Lobatto points used to *place* the geometry nodes are computed here with numpy's
Legendre routines; the oracle has its own, independently pinned GLL routine, and both the
oracle and the GPU library consume the *same* E-vector bytes (SURVEY P-9: parity is
ill-conditioned w.r.t. coordinate rounding, so both sides must read identical coordinates).

Recipes:
  * Cartesian box ``[0,1]^d`` (or ``[0,1]^2 x [0,G]`` for slab meshes), lexicographic ids,
    x fastest.
  * ``jitter``: interior coarse vertices moved by U(-0.1,0.1)*h per coordinate,
    ``numpy.random.default_rng(12253)`` in vertex-id order.
  * ``kershaw``: the Kershaw/CEED map with eps_y = eps_z = eps applied per unit z-slab.
  * ``scramble``: each element's local corner order rotated by one of the 24 proper cube
    rotations, ``default_rng(2210).integers(24)`` per element in element order.
"""
from __future__ import annotations

import itertools
from dataclasses import dataclass, field

import numpy as np

JITTER_SEED = 12253
SCRAMBLE_SEED = 2210


@dataclass
class Mesh:
    dim: int
    p: int
    vert: np.ndarray          # [nv, dim] float64
    elem: np.ndarray          # [nel, 2^dim] int64, local corner order a + 2b + 4c
    X: np.ndarray             # [nel, dim, (p+1)^dim] float64 E-vector at GLL points
    shape: tuple              # elements per axis
    elem_rank_begin: np.ndarray = field(default=None)  # [nranks+1] int64 (z-slabs)
    name: str = ""

    @property
    def nel(self) -> int:
        return int(self.elem.shape[0])

    @property
    def nv(self) -> int:
        return int(self.vert.shape[0])


def gll_points_01(p: int) -> np.ndarray:
    """Gauss--Lobatto points mapped to [0,1] (roots of (1-x^2) P_p'(x)), ascending."""
    if p < 1:
        raise ValueError("p >= 1 required")
    if p == 1:
        x = np.array([-1.0, 1.0])
    else:
        c = np.zeros(p + 1)
        c[p] = 1.0
        inner = np.polynomial.legendre.legroots(np.polynomial.legendre.legder(c))
        # polish with Newton on P_p'(x) in long double-free fp64 (a few steps)
        d1 = np.polynomial.legendre.legder(c)
        d2 = np.polynomial.legendre.legder(d1)
        for _ in range(3):
            inner = inner - np.polynomial.legendre.legval(inner, d1) / np.polynomial.legendre.legval(inner, d2)
        inner = np.sort(inner)
        x = np.concatenate([[-1.0], inner, [1.0]])
        # enforce exact symmetry
        x = 0.5 * (x - x[::-1])
    return (x + 1.0) / 2.0


# --------------------------------------------------------------------------- structured meshes
def _box(dim, n, lo, hi):
    axes = [np.linspace(lo[d], hi[d], n[d] + 1) for d in range(dim)]
    if dim == 2:
        Y, Xc = np.meshgrid(axes[1], axes[0], indexing="ij")
        vert = np.stack([Xc.ravel(), Y.ravel()], axis=1)
    else:
        Z, Y, Xc = np.meshgrid(axes[2], axes[1], axes[0], indexing="ij")
        vert = np.stack([Xc.ravel(), Y.ravel(), Z.ravel()], axis=1)
    return vert


def _connectivity(dim, n):
    if dim == 2:
        nx, ny = n
        j, i = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
        base = (i + (nx + 1) * j).ravel()
        offs = [0, 1, nx + 1, nx + 2]  # a + 2b
        return np.stack([base + o for o in offs], axis=1).astype(np.int64)
    nx, ny, nz = n
    k, j, i = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    sx, sy = 1, nx + 1
    sz = (nx + 1) * (ny + 1)
    base = (i * sx + j * sy + k * sz).ravel()
    offs = [a * sx + b * sy + c * sz for c in (0, 1) for b in (0, 1) for a in (0, 1)]
    return np.stack([base + o for o in offs], axis=1).astype(np.int64)


def _kershaw_right(eps, t):
    return np.where(t <= 0.5, (2.0 - eps) * t, 1.0 + eps * (t - 1.0))


def _kershaw_left(eps, t):
    return 1.0 - _kershaw_right(eps, 1.0 - t)


def _kershaw_step(a, b, lam):
    return a + (b - a) * np.clip(lam, 0.0, 1.0)


def kershaw_map(xyz: np.ndarray, eps_y: float, eps_z: float) -> np.ndarray:
    """Kershaw (JCP 1981) / CEED-benchmark map of the unit cube."""
    x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    layer = np.minimum(np.floor(6.0 * x), 5).astype(np.int64)
    lam = 6.0 * x - layer
    Ly, Ry = _kershaw_left(eps_y, y), _kershaw_right(eps_y, y)
    Lz, Rz = _kershaw_left(eps_z, z), _kershaw_right(eps_z, z)
    Y = np.empty_like(y)
    Z = np.empty_like(z)
    for L in range(6):
        m = layer == L
        if L == 0:
            Y[m], Z[m] = Ly[m], Lz[m]
        elif L in (1, 4):
            Y[m] = _kershaw_step(Ly[m], Ry[m], lam[m])
            Z[m] = _kershaw_step(Lz[m], Rz[m], lam[m])
        elif L == 2:
            Y[m] = _kershaw_step(Ry[m], Ly[m], lam[m] / 2)
            Z[m] = _kershaw_step(Rz[m], Lz[m], lam[m] / 2)
        elif L == 3:
            Y[m] = _kershaw_step(Ry[m], Ly[m], (1 + lam[m]) / 2)
            Z[m] = _kershaw_step(Rz[m], Lz[m], (1 + lam[m]) / 2)
        else:
            Y[m], Z[m] = Ry[m], Rz[m]
    return np.stack([x, Y, Z], axis=1)


def cube_rotations():
    """The 24 proper rotations of the cube, in the order SURVEY App. B fixes."""
    rots = []
    for perm in itertools.permutations(range(3)):
        for s in itertools.product((1, -1), repeat=3):
            M = np.zeros((3, 3), dtype=np.int64)
            for i in range(3):
                M[i, perm[i]] = s[i]
            if round(np.linalg.det(M)) == 1:
                rots.append(M)
    assert len(rots) == 24
    return rots


def _scramble(elem: np.ndarray, dim: int) -> np.ndarray:
    rng = np.random.default_rng(SCRAMBLE_SEED)
    out = elem.copy()
    if dim == 3:
        rots = cube_rotations()
        choice = rng.integers(24, size=elem.shape[0])
        corners = np.array([[a, b, c] for c in (0, 1) for b in (0, 1) for a in (0, 1)])
        perms = []
        for M in rots:
            perm = np.empty(8, dtype=np.int64)
            for q in range(8):
                old = (M @ (2 * corners[q] - 1) + 1) // 2
                perm[q] = old[0] + 2 * old[1] + 4 * old[2]
            perms.append(perm)
        perms = np.array(perms)
    else:
        # the 4 proper rotations of the square
        choice = rng.integers(4, size=elem.shape[0])
        corners = np.array([[a, b] for b in (0, 1) for a in (0, 1)])
        perms = []
        for r in range(4):
            th = r * np.pi / 2
            M = np.rint(np.array([[np.cos(th), -np.sin(th)], [np.sin(th), np.cos(th)]])).astype(np.int64)
            perm = np.empty(4, dtype=np.int64)
            for q in range(4):
                old = (M @ (2 * corners[q] - 1) + 1) // 2
                perm[q] = old[0] + 2 * old[1]
            perms.append(perm)
        perms = np.array(perms)
    for e in range(elem.shape[0]):
        out[e] = elem[e][perms[choice[e]]]
    return out


def evector(dim: int, p: int, vert: np.ndarray, elem: np.ndarray) -> np.ndarray:
    """Trilinear (bilinear) interpolation of each element's corners at the tensor GLL points.

    X_e[d][k][j][i] = sum_{abc} n_a(s_i) n_b(s_j) n_c(s_k) V[E[e][a+2b+4c]][d],
    n_0 = 1-s, n_1 = s, s = GLL points on [0,1].
    """
    s = gll_points_01(p)
    n = np.stack([1.0 - s, s], axis=0)  # [2, p+1]
    C = vert[elem]  # [nel, 2^dim, dim]
    nel = elem.shape[0]
    if dim == 2:
        C = C.reshape(nel, 2, 2, dim)  # [e, b, a, d]
        X = np.einsum("bj,ai,ebad->edji", n, n, C, optimize=True)
        return np.ascontiguousarray(X.reshape(nel, dim, (p + 1) ** 2))
    C = C.reshape(nel, 2, 2, 2, dim)  # [e, c, b, a, d]
    X = np.einsum("ck,bj,ai,ecbad->edkji", n, n, n, C, optimize=True)
    return np.ascontiguousarray(X.reshape(nel, dim, (p + 1) ** 3))


def box_mesh(dim: int, n, p: int, *, lo=None, hi=None, jitter: bool = False, kershaw: float | None = None,
             scramble: bool = False, nranks: int = 1, name: str = "") -> Mesh:
    """Structured box mesh with optional jitter / per-slab Kershaw / orientation scramble.

    For slab meshes (``nranks`` > 1) the z extent is split into ``nranks`` contiguous element
    slabs (``elem_rank_begin[r] = r * nel / nranks``); the caller picks n_z divisible by nranks.
    """
    n = tuple(int(v) for v in n)
    assert len(n) == dim
    lo = tuple(lo) if lo is not None else (0.0,) * dim
    hi = tuple(hi) if hi is not None else (1.0,) * dim
    vert = _box(dim, n, lo, hi)
    elem = _connectivity(dim, n)
    nv = vert.shape[0]
    if jitter:
        rng = np.random.default_rng(JITTER_SEED)
        h = np.array([(hi[d] - lo[d]) / n[d] for d in range(dim)])
        idx = np.stack(np.unravel_index(np.arange(nv), tuple(v + 1 for v in n[::-1])), axis=1)[:, ::-1]
        interior = np.all((idx > 0) & (idx < np.array(n)), axis=1)
        delta = rng.uniform(-0.1, 0.1, size=(nv, dim)) * h
        vert = vert + np.where(interior[:, None], delta, 0.0)
    if kershaw is not None:
        assert dim == 3
        z0 = np.floor(vert[:, 2] - lo[2] + 1e-12)
        z0 = np.clip(z0, 0, max(hi[2] - lo[2] - 1, 0))
        loc = vert.copy()
        loc[:, 2] = vert[:, 2] - lo[2] - z0
        loc[:, 0] = (vert[:, 0] - lo[0]) / (hi[0] - lo[0])
        loc[:, 1] = (vert[:, 1] - lo[1]) / (hi[1] - lo[1])
        m = kershaw_map(loc, kershaw, kershaw)
        vert = np.stack([lo[0] + m[:, 0] * (hi[0] - lo[0]), lo[1] + m[:, 1] * (hi[1] - lo[1]),
                         lo[2] + z0 + m[:, 2]], axis=1)
    if scramble:
        elem = _scramble(elem, dim)
    X = evector(dim, p, vert, elem)
    nel = elem.shape[0]
    erb = np.array([r * nel // nranks for r in range(nranks + 1)], dtype=np.int64)
    return Mesh(dim=dim, p=p, vert=np.ascontiguousarray(vert), elem=np.ascontiguousarray(elem), X=X,
                shape=n, elem_rank_begin=erb, name=name)


# --------------------------------------------------------------------------- named workloads
def config_mesh(cfg: str, *, gpus: int = 1, p: int | None = None, n: int | None = None) -> tuple[Mesh, dict]:
    """The BASELINE.json configurations as concrete synthetic inputs.

    Returns (mesh, form) where form = {"space", "alpha", "beta", "quad"}.
    Slab configs (C3, C5, and C2 in weak-scaling mode) stack ``gpus`` unit slabs in z.
    """
    cfg = cfg.upper()
    if cfg == "C1":
        return box_mesh(2, (4, 4), p or 2, name="C1"), dict(space="h1", alpha=1.0, beta=0.0, quad="vertex")
    if cfg in ("C2", "C2-J"):
        nn = n or 32
        m = box_mesh(3, (nn, nn, nn * gpus), p or 4, hi=(1.0, 1.0, float(gpus)), jitter=cfg.endswith("J"),
                     nranks=gpus, name=cfg)
        return m, dict(space="h1", alpha=1.0, beta=1.0, quad="vertex")
    if cfg in ("C3", "C3-L"):
        nn = n or (48 if cfg == "C3-L" else 24)
        m = box_mesh(3, (nn, nn, nn * gpus), p or 8, hi=(1.0, 1.0, float(gpus)), kershaw=0.3, nranks=gpus,
                     name=cfg)
        return m, dict(space="h1", alpha=1.0, beta=1.0, quad="vertex")
    if cfg in ("C4", "C4-J"):
        nn = n or 32
        m = box_mesh(3, (nn, nn, nn * gpus), p or 4, hi=(1.0, 1.0, float(gpus)), jitter=cfg.endswith("J"),
                     nranks=gpus, name=cfg)
        return m, dict(space="nd", alpha=1.0, beta=1.0, quad="vertex")
    if cfg in ("C5", "C5-J"):
        nn = n or 32
        m = box_mesh(3, (nn, nn, nn * gpus), p or 4, hi=(1.0, 1.0, float(gpus)), jitter=cfg.endswith("J"),
                     nranks=gpus, name=cfg)
        return m, dict(space="rt", alpha=1.0, beta=1.0, quad="vertex")
    raise ValueError(f"unknown config {cfg}")
