"""Pins of oracle/bc.py (A4 elimination, ParCSR layout, boundary dofs, coordinate vectors) against
what the paper and the mathematics fix -- not against the oracle itself:

* boundary-dof counts: closed forms of the LOR surface lattice of a box (points / edges / faces on
  the boundary of an N_x x N_y x N_z cell grid), invariant under orientation scrambling;
* boundary dofs are exactly the dofs whose geometric support (LOR vertex; both end points of an
  edge via the discrete gradient; all corners of a face via C and G) lies on one boundary plane;
* A4: the eliminated Dirichlet problem of the Laplacian (alpha = 1, beta = 0,
  Cartesian) with linear boundary data reproduces the linear function exactly (Q1 / LOR-Q1 on
  affine cells contains the linears and the vertex rule integrates c . grad v exactly);
  symmetry kept; identity on the essential block;
* ParCSR (l.369-370): for a z-slab split of a Cartesian H1 matrix the off-rank column count is one
  (N_x+1)(N_y+1) plane per neighbour slab and the offd nonzeros one (3N_x+1)(3N_y+1) 9-point
  plane stencil per neighbour; the diag block starts every row with the diagonal;
* coordinates (l.400-404): on a Cartesian box the set of LOR vertex coordinates is the tensor
  lattice of the GLL points of every element; every E-vector copy of a shared vertex agrees with
  the deduplicated value to rounding.
"""
import numpy as np
import pytest
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from oracle import bc
from paper_2210_12253_b200 import meshgen as mg


def _cells(m):
    return [s * m.p for s in m.shape]


@pytest.mark.parametrize("scramble", [False, True])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_boundary_counts_closed_form(oracle_lib, p, scramble):
    m = mg.box_mesh(3, (2, 3, 2), p, jitter=True, scramble=scramble)
    Nx, Ny, Nz = _cells(m)
    h1 = (Nx + 1) * (Ny + 1) * (Nz + 1) - (Nx - 1) * (Ny - 1) * (Nz - 1)
    nd = (Nx * ((Ny + 1) * (Nz + 1) - (Ny - 1) * (Nz - 1)) + Ny * ((Nx + 1) * (Nz + 1) - (Nx - 1) * (Nz - 1)) +
          Nz * ((Nx + 1) * (Ny + 1) - (Nx - 1) * (Ny - 1)))
    rt = 2 * (Nx * Ny + Ny * Nz + Nx * Nz)
    assert len(bc.boundary_dofs(m, "h1")) == h1
    assert len(bc.boundary_dofs(m, "nd")) == nd
    assert len(bc.boundary_dofs(m, "rt")) == rt
    m2 = mg.box_mesh(2, (3, 2), p, scramble=scramble)
    Nx, Ny = _cells(m2)
    assert len(bc.boundary_dofs(m2, "h1")) == (Nx + 1) * (Ny + 1) - (Nx - 1) * (Ny - 1)


def _on_plane(xyz, tol=1e-12):
    """bit mask per point: which of the 6 boundary planes of [0,1]^3 it lies on"""
    bits = np.zeros(xyz.shape[1], dtype=np.int64)
    for a in range(3):
        bits |= (np.abs(xyz[a]) < tol).astype(np.int64) << (2 * a)
        bits |= (np.abs(xyz[a] - 1.0) < tol).astype(np.int64) << (2 * a + 1)
    return bits


@pytest.mark.parametrize("p", [1, 2, 3])
def test_boundary_dofs_geometric(oracle_lib, p):
    """a dof is essential iff its support lies on one boundary plane (jittered interior, scrambled)"""
    m = mg.box_mesh(3, (2, 2, 3), p, jitter=True, scramble=True)
    xyz = bc.coordinates(m)
    vb = _on_plane(xyz)
    n_h1 = xyz.shape[1]
    ess = np.zeros(n_h1, dtype=bool)
    ess[bc.boundary_dofs(m, "h1")] = True
    assert np.array_equal(ess, vb != 0)
    G = oracle_lib.discrete(m, "grad")
    ends = G.col.reshape(-1, 2)
    nd_geo = (vb[ends[:, 0]] & vb[ends[:, 1]]) != 0
    ess_nd = np.zeros(ends.shape[0], dtype=bool)
    ess_nd[bc.boundary_dofs(m, "nd")] = True
    assert np.array_equal(ess_nd, nd_geo)
    C = oracle_lib.discrete(m, "curl")
    edges = C.col.reshape(-1, 4)
    corner_bits = np.full(edges.shape[0], -1, dtype=np.int64)
    for k in range(4):
        corner_bits &= vb[ends[edges[:, k], 0]] & vb[ends[edges[:, k], 1]]
    ess_rt = np.zeros(edges.shape[0], dtype=bool)
    ess_rt[bc.boundary_dofs(m, "rt")] = True
    assert np.array_equal(ess_rt, corner_bits != 0)


def _to_scipy(A, n):
    rows = np.repeat(A.row_id, np.diff(A.row_ptr))
    return sp.csr_matrix((A.val, (rows, A.col)), shape=(n, n))


@pytest.mark.parametrize("dim,p", [(2, 1), (2, 3), (3, 1), (3, 2), (3, 4)])
def test_eliminate_reproduces_linear_dirichlet(oracle_lib, dim, p):
    shape = (3, 2) if dim == 2 else (2, 2, 2)
    m = mg.box_mesh(dim, shape, p, scramble=True)
    A = oracle_lib.assemble(m, "h1", "vertex", 1.0, 0.0)
    n = A.row_ptr.shape[0] - 1
    xyz = bc.coordinates(m)
    coef = np.array([0.3, -1.7, 2.2][:dim])
    u = 0.75 + coef @ xyz
    ess = bc.boundary_dofs(m, "h1")
    K = _to_scipy(bc.eliminate(A, ess), n)
    A0 = _to_scipy(A, n)
    mask = np.zeros(n, dtype=bool)
    mask[ess] = True
    g = np.where(mask, u, 0.0)
    b = -(A0 @ g)
    b[mask] = u[mask]
    x = spla.spsolve(K.tocsc(), b)
    assert np.max(np.abs(x - u)) < 1e-10 * np.max(np.abs(u))
    # structure: symmetric, unit rows / columns on the essential block
    assert abs(K - K.T).max() == 0.0
    Kd = K.toarray()
    assert np.array_equal(Kd[np.ix_(mask, mask)], np.eye(mask.sum()))
    assert not Kd[np.ix_(mask, ~mask)].any() and not Kd[np.ix_(~mask, mask)].any()
    assert np.array_equal(Kd[np.ix_(~mask, ~mask)], A0.toarray()[np.ix_(~mask, ~mask)])


@pytest.mark.parametrize("nranks", [2, 3])
def test_parcsr_slab_closed_form(oracle_lib, nranks):
    p = 2
    m = mg.box_mesh(3, (2, 3, 2 * nranks), p, nranks=nranks)
    A = oracle_lib.assemble(m, "h1", "vertex", 1.0, 1.0, nranks=nranks)
    _, _, off = oracle_lib.space_size(m, "h1", nranks)
    Nx, Ny, _ = _cells(m)
    for r in range(nranks):
        P = bc.parcsr_split(A, off[r], off[r + 1] - off[r], off[r], off[r + 1], square=True)
        nb = (r > 0) + (r < nranks - 1)
        assert len(P["col_map_offd"]) == nb * (Nx + 1) * (Ny + 1)
        assert len(P["offd_col"]) == nb * (3 * Nx + 1) * (3 * Ny + 1)
        assert np.all(np.diff(P["col_map_offd"]) > 0)
        assert not np.any((P["col_map_offd"] >= off[r]) & (P["col_map_offd"] < off[r + 1]))
        # the diagonal first: local column == local row
        d0 = P["diag_col"][P["diag_row_ptr"][:-1]]
        assert np.array_equal(d0, np.arange(off[r + 1] - off[r]))
        assert P["diag_row_ptr"][-1] + P["offd_row_ptr"][-1] == A.row_ptr[off[r + 1]] - A.row_ptr[off[r]]


@pytest.mark.parametrize("dim,p", [(2, 3), (3, 1), (3, 4)])
def test_coordinates_cartesian_lattice(oracle_lib, dim, p):
    shape = (3, 2) if dim == 2 else (2, 3, 2)
    m = mg.box_mesh(dim, shape, p, scramble=True)
    xyz = bc.coordinates(m)
    x1 = mg.gll_points_01(p)
    axes = []
    for a in range(dim):
        pts = sorted({(e + t) / shape[a] for e in range(shape[a]) for t in x1})
        axes.append(np.array(pts))
    # every coordinate equals a lattice point to rounding, and the lattice is covered exactly once
    key = []
    for a in range(dim):
        idx = np.abs(xyz[a][:, None] - axes[a][None, :]).argmin(axis=1)
        assert np.max(np.abs(xyz[a] - axes[a][idx])) < 1e-14
        key.append(idx)
    key = np.ravel_multi_index(tuple(key), tuple(len(v) for v in axes))
    assert len(np.unique(key)) == key.shape[0] == int(np.prod([len(v) for v in axes]))


def test_coordinates_copies_agree(oracle_lib):
    m = mg.box_mesh(3, (2, 2, 2), 3, kershaw=0.3, scramble=True)
    xyz = bc.coordinates(m)
    mp, _ = oracle_lib.dof_map(m, "h1")
    for e in range(m.nel):
        assert np.max(np.abs(m.X[e] - xyz[:, mp[e]])) < 1e-15
