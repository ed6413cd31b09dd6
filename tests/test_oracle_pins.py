"""Pins of the CPU oracle to what the paper and mathematics fix.

None of these re-types the oracle's formulas: they compare it with printed numbers
(tests/golden/*.json, each cited), textbook element matrices, closed forms (Kronecker
products of 1D matrices, finite-difference stencils, pattern-count formulas), invariants of the
discrete de Rham complex, a geometric (Stokes) identity, brute-force dense eigenvalues
against independently built high-order matrices, and independent re-derivations (row oracle
vs full oracle, rank split vs single rank, orientation-scrambled vs plain mesh).
"""
import json
import os

import numpy as np
import pytest
import scipy.sparse as sp

from paper_2210_12253_b200 import meshgen as mg

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def gold(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


def to_sparse(A):
    n_rows = int(A.row_id.max()) + 1
    rows = np.repeat(A.row_id, np.diff(A.row_ptr))
    return sp.csr_matrix((A.val, (rows, A.col.astype(np.int64))), shape=(n_rows, A.n_cols))


def unit_corners(dim, h=1.0):
    if dim == 2:
        return np.array([[a, b] for b in (0, 1) for a in (0, 1)], float) * h
    return np.array([[a, b, c] for c in (0, 1) for b in (0, 1) for a in (0, 1)], float) * h


def random_hex(rng):
    """a random trilinear hex with positive Jacobian at every point (perturbed unit cube)"""
    return unit_corners(3) + rng.uniform(-0.15, 0.15, size=(8, 3))


# ------------------------------------------------------------------------------- GLL (C.1)
def test_gll_closed_forms(oracle_lib):
    O = oracle_lib
    x, w = O.gll(2)
    np.testing.assert_allclose(x, [-1, 0, 1], atol=1e-15)
    np.testing.assert_allclose(w, [1 / 3, 4 / 3, 1 / 3], rtol=1e-14)
    x, _ = O.gll(3)
    np.testing.assert_allclose(x, [-1, -1 / np.sqrt(5), 1 / np.sqrt(5), 1], atol=1e-15)
    x, w = O.gll(4)
    np.testing.assert_allclose(x, [-1, -np.sqrt(3 / 7), 0, np.sqrt(3 / 7), 1], atol=1e-15)
    np.testing.assert_allclose(w, [1 / 10, 49 / 90, 32 / 45, 49 / 90, 1 / 10], rtol=1e-14)
    x, _ = O.gll(5)
    r = np.sqrt([1 / 3 - 2 * np.sqrt(7) / 21, 1 / 3 + 2 * np.sqrt(7) / 21])
    np.testing.assert_allclose(x, [-1, -r[1], -r[0], r[0], r[1], 1], atol=1e-15)


@pytest.mark.parametrize("p", range(1, 10))
def test_gll_exactness(oracle_lib, p):
    x, w = oracle_lib.gll(p)
    assert abs(w.sum() - 2) < 1e-14
    for k in range(2 * p):  # exact through degree 2p-1
        exact = 0.0 if k % 2 else 2.0 / (k + 1)
        assert abs((w * x ** k).sum() - exact) < 1e-13


# ------------------------------------------------------------ textbook p=1 cells (C.4, l.150)
def test_textbook_h1_cells(oracle_lib):
    O, g = oracle_lib, gold("textbook_cell_rows.json")
    r2 = g["h1_2d_unit_square_row0"]
    K = O.local_matrix(2, "h1", "vertex", 1, 0, unit_corners(2))
    np.testing.assert_allclose(K[0], r2["vertex_stiffness"], atol=1e-15)
    M = O.local_matrix(2, "h1", "vertex", 0, 1, unit_corners(2))
    np.testing.assert_allclose(M, np.eye(4) * r2["vertex_mass_diag"], atol=1e-16)
    K = O.local_matrix(2, "h1", "gauss2", 1, 0, unit_corners(2))
    np.testing.assert_allclose(6 * K[0], r2["exact_stiffness_x6"], atol=1e-14)
    M = O.local_matrix(2, "h1", "gauss2", 0, 1, unit_corners(2))
    np.testing.assert_allclose(36 * M[0], r2["exact_mass_x36"], atol=1e-14)
    r3 = g["h1_3d_unit_cube_row0"]
    K = O.local_matrix(3, "h1", "vertex", 1, 0, unit_corners(3))
    np.testing.assert_allclose(4 * K[0], r3["vertex_stiffness_x4"], atol=1e-15)
    M = O.local_matrix(3, "h1", "vertex", 0, 1, unit_corners(3))
    np.testing.assert_allclose(M, np.eye(8) * r3["vertex_mass_diag"], atol=1e-16)
    K = O.local_matrix(3, "h1", "gauss2", 1, 0, unit_corners(3))
    np.testing.assert_allclose(12 * K[0], r3["exact_stiffness_x12"], atol=1e-14)
    M = O.local_matrix(3, "h1", "gauss2", 0, 1, unit_corners(3))
    np.testing.assert_allclose(216 * M[0], r3["exact_mass_x216"], atol=1e-13)


def test_textbook_nd_rt_cells(oracle_lib):
    O, g = oracle_lib, gold("textbook_cell_rows.json")
    nd = g["nd_unit_cube_row_xedge00"]
    c = unit_corners(3)
    np.testing.assert_allclose(O.local_matrix(3, "nd", "vertex", 0, 1, c), np.eye(12) * nd["vertex_mass_diag"],
                               atol=1e-16)
    np.testing.assert_allclose(2 * O.local_matrix(3, "nd", "vertex", 1, 0, c)[0], nd["vertex_curlcurl_x2"], atol=1e-15)
    np.testing.assert_allclose(36 * O.local_matrix(3, "nd", "gauss2", 0, 1, c)[0], nd["exact_mass_x36"], atol=1e-13)
    np.testing.assert_allclose(6 * O.local_matrix(3, "nd", "gauss2", 1, 0, c)[0], nd["exact_curlcurl_x6"], atol=1e-13)
    rt = g["rt_unit_cube_row_x0"]
    np.testing.assert_allclose(O.local_matrix(3, "rt", "vertex", 0, 1, c), np.eye(6) * rt["vertex_mass_diag"],
                               atol=1e-16)
    np.testing.assert_allclose(6 * O.local_matrix(3, "rt", "gauss2", 0, 1, c)[0], rt["exact_mass_x6"], atol=1e-14)
    for quad in ("vertex", "gauss2"):
        np.testing.assert_allclose(O.local_matrix(3, "rt", quad, 1, 0, c)[0], rt["divdiv"], atol=1e-14)


def _cell_incidence():
    """cell-level G (12x8: edge tail -1, head +1) and C (6x12: right-hand circulation), from the
    reference-cell geometry alone (edge/face positions), not from the oracle."""
    corners = unit_corners(3).astype(int)
    edges = []
    for a in range(3):
        u, v = [d for d in range(3) if d != a]
        for b2 in (0, 1):
            for b1 in (0, 1):
                t = np.zeros(3, int)
                t[u], t[v] = b1, b2
                h = t.copy()
                h[a] = 1
                edges.append((a, t, h))
    G = np.zeros((12, 8))
    for i, (a, t, h) in enumerate(edges):
        G[i, [int(np.flatnonzero((corners == t).all(1))[0])]] = -1
        G[i, [int(np.flatnonzero((corners == h).all(1))[0])]] = 1
    Cm = np.zeros((6, 12))
    for f in range(6):
        d, side = f // 2, f % 2
        normal = np.zeros(3)
        normal[d] = 1
        center = np.full(3, 0.5)
        center[d] = side
        for i, (a, t, h) in enumerate(edges):
            if t[d] != side or h[d] != side:
                continue
            mid = (t + h) / 2.0
            tang = (h - t).astype(float)
            # circulation sign: (normal x (mid - center)) . tangent
            Cm[f, i] = np.sign(np.dot(np.cross(normal, mid - center), tang))
    return G, Cm


def test_cell_derham_factorizations(oracle_lib):
    """K_H1 = G^T M_ND G, K_ND = C^T M_RT C, K_RT = (sum w a/det) d d^T on a random trilinear hex
    (SURVEY C.6): a cross-check of the oracle's three element routines against each other, with
    the cell incidences built from reference geometry in this test."""
    O = oracle_lib
    rng = np.random.default_rng(7)
    G, Cm = _cell_incidence()
    assert np.abs(Cm @ G).max() == 0
    for quad in ("vertex", "gauss2"):
        for _ in range(3):
            c = random_hex(rng)
            KH = O.local_matrix(3, "h1", quad, 1.0, 0.0, c)
            MN = O.local_matrix(3, "nd", quad, 0.0, 1.0, c)
            np.testing.assert_allclose(KH, G.T @ MN @ G, atol=2e-14)
            KN = O.local_matrix(3, "nd", quad, 1.0, 0.0, c)
            MR = O.local_matrix(3, "rt", quad, 0.0, 1.0, c)
            np.testing.assert_allclose(KN, Cm.T @ MR @ Cm, atol=2e-14)
            KR = O.local_matrix(3, "rt", quad, 1.0, 0.0, c)
            assert np.linalg.matrix_rank(KR, tol=1e-12) == 1
            d = np.array([-1, 1, -1, 1, -1, 1.0])
            np.testing.assert_allclose(KR, KR[1, 1] * np.outer(d, d), atol=1e-14)


def test_vertex_rule_body_diagonal_is_zero(oracle_lib):
    """C.5: under the vertex rule the 3D H1 body-diagonal entries vanish for ANY geometry."""
    rng = np.random.default_rng(3)
    for _ in range(5):
        K = oracle_lib.local_matrix(3, "h1", "vertex", 1.0, 0.0, random_hex(rng))
        for q in range(8):
            assert K[q, 7 - q] == 0.0


# -------------------------------------------------------------- FD stencils at p=1 (C.4)
def test_p1_uniform_grid_is_fd_laplacian(oracle_lib):
    h = 0.25
    m2 = mg.box_mesh(2, (4, 4), 1)
    A = to_sparse(oracle_lib.assemble(m2, "h1", "vertex", 1.0, 0.0)).toarray()
    c = 2 + 5 * 2  # interior vertex (2,2)
    row = A[c]
    assert abs(row[c] - 4) < 1e-14
    for nb in (c - 1, c + 1, c - 5, c + 5):
        assert abs(row[nb] + 1) < 1e-14
    assert abs(np.abs(row).sum() - 8) < 1e-13
    m3 = mg.box_mesh(3, (4, 4, 4), 1)
    A = to_sparse(oracle_lib.assemble(m3, "h1", "vertex", 1.0, 0.0)).toarray()
    c = 2 + 5 * 2 + 25 * 2
    row = A[c]
    assert abs(row[c] - 6 * h) < 1e-14
    for nb in (c - 1, c + 1, c - 5, c + 5, c - 25, c + 25):
        assert abs(row[nb] + h) < 1e-14
    assert abs(np.abs(row).sum() - 12 * h) < 1e-13


# ---------------------------------------------------------- Kronecker form (C.3), Cartesian
def _grid_1d(n, p):
    s = mg.gll_points_01(p)
    x = np.concatenate([[0.0]] + [(i + s[1:]) / n for i in range(n)])
    return x


def _kmats(x, quad):
    N = len(x) - 1
    K = np.zeros((N + 1, N + 1))
    M = np.zeros((N + 1, N + 1))
    for j in range(N):
        hj = x[j + 1] - x[j]
        K[np.ix_([j, j + 1], [j, j + 1])] += np.array([[1, -1], [-1, 1]]) / hj
        if quad == "vertex":
            M[j, j] += hj / 2
            M[j + 1, j + 1] += hj / 2
        else:
            M[np.ix_([j, j + 1], [j, j + 1])] += hj * np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    return K, M


def _h1_coords(oracle_lib, mesh):
    """coordinate of every H1 dof, read from the E-vector through the oracle's map"""
    mp, _ = oracle_lib.dof_map(mesh, "h1")
    n = mp.max() + 1
    xyz = np.zeros((n, mesh.dim))
    for d in range(mesh.dim):
        xyz[mp.ravel(), d] = mesh.X[:, d, :].ravel()
    return xyz


@pytest.mark.parametrize("dim,shape,p", [(2, (3, 2), 4), (3, (2, 1, 2), 3), (3, (1, 2, 1), 5)])
@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
def test_kronecker_closed_form(oracle_lib, dim, shape, p, quad):
    alpha, beta = 1.3, 0.7
    m = mg.box_mesh(dim, shape, p)
    A = to_sparse(oracle_lib.assemble(m, "h1", quad, alpha, beta)).toarray()
    xs = [_grid_1d(shape[d], p) for d in range(dim)]
    KM = [_kmats(x, quad) for x in xs]
    if dim == 2:
        (Kx, Mx), (Ky, My) = KM
        Ak = alpha * (np.kron(My, Kx) + np.kron(Ky, Mx)) + beta * np.kron(My, Mx)
    else:
        (Kx, Mx), (Ky, My), (Kz, Mz) = KM
        Ak = alpha * (np.kron(Mz, np.kron(My, Kx)) + np.kron(Mz, np.kron(Ky, Mx)) + np.kron(Kz, np.kron(My, Mx))) \
            + beta * np.kron(Mz, np.kron(My, Mx))
    # permutation oracle-id -> lexicographic grid index, from the dof coordinates
    xyz = _h1_coords(oracle_lib, m)
    idx = np.zeros(len(xyz), dtype=np.int64)
    stride = 1
    for d in range(dim):
        ii = np.searchsorted(xs[d], xyz[:, d] - 1e-12)
        assert np.allclose(xs[d][ii], xyz[:, d], atol=1e-14)
        idx += ii * stride
        stride *= len(xs[d])
    assert len(np.unique(idx)) == len(idx)
    Ap = np.zeros_like(A)
    Ap[np.ix_(idx, idx)] = A
    assert np.abs(Ap - Ak).max() <= 1e-13 * np.abs(Ak).max()


# ------------------------------------------------------------------ pattern counts (C.2)
def _t(N):
    return 3 * N + 1


@pytest.mark.parametrize("shape,p", [((1, 1, 1), 1), ((2, 3, 4), 2), ((2, 1, 3), 3), ((1, 2, 1), 4)])
def test_pattern_closed_forms_3d(oracle_lib, shape, p):
    m = mg.box_mesh(3, shape, p, jitter=True)
    Nx, Ny, Nz = (s * p for s in shape)
    h1 = oracle_lib.assemble(m, "h1")
    assert h1.row_ptr.shape[0] - 1 == (Nx + 1) * (Ny + 1) * (Nz + 1)
    assert h1.nnz == _t(Nx) * _t(Ny) * _t(Nz)
    nd = oracle_lib.assemble(m, "nd")
    n_nd = Nx * (Ny + 1) * (Nz + 1) + (Nx + 1) * Ny * (Nz + 1) + (Nx + 1) * (Ny + 1) * Nz
    assert nd.row_ptr.shape[0] - 1 == n_nd
    assert nd.nnz == (Nx * _t(Ny) * _t(Nz) + _t(Nx) * Ny * _t(Nz) + _t(Nx) * _t(Ny) * Nz
                      + 8 * (Nx * Ny * _t(Nz) + Nx * Nz * _t(Ny) + Ny * Nz * _t(Nx)))
    rt = oracle_lib.assemble(m, "rt")
    assert rt.row_ptr.shape[0] - 1 == (Nx + 1) * Ny * Nz + Nx * (Ny + 1) * Nz + Nx * Ny * (Nz + 1)
    assert rt.nnz == _t(Nx) * Ny * Nz + Nx * _t(Ny) * Nz + Nx * Ny * _t(Nz) + 24 * Nx * Ny * Nz
    # interior row counts: 27 / 33 / 11 (C.2)
    assert np.diff(h1.row_ptr).max() <= 27 and np.diff(nd.row_ptr).max() <= 33 and np.diff(rt.row_ptr).max() <= 11
    if min(Nx, Ny, Nz) >= 3:
        assert np.diff(h1.row_ptr).max() == 27 and np.diff(nd.row_ptr).max() == 33
        assert np.diff(rt.row_ptr).max() == 11


@pytest.mark.parametrize("shape,p", [((1, 1), 1), ((3, 5), 2), ((2, 2), 4)])
def test_pattern_closed_forms_2d(oracle_lib, shape, p):
    m = mg.box_mesh(2, shape, p)
    Nx, Ny = (s * p for s in shape)
    A = oracle_lib.assemble(m, "h1", alpha=1.0, beta=0.0)
    assert A.row_ptr.shape[0] - 1 == (Nx + 1) * (Ny + 1)
    assert A.nnz == _t(Nx) * _t(Ny)
    assert np.diff(A.row_ptr).max() <= 9


def test_paper_printed_counts(oracle_lib):
    """dof counts from the oracle's numbering on the paper's meshes, and
    the nnz closed form (pinned above against the oracle) at those sizes."""
    g = gold("paper_pins.json")
    for key in ("h1_2d_p6_262144el", "h1_3d_p6_32768el"):
        e = g[key]
        dim, p, n = e["dim"], e["p"], e["elems_per_axis"]
        N = n * p
        assert (N + 1) ** dim == e["rows"]
        assert _t(N) ** dim == e["nnz"]
    m = mg.box_mesh(2, (512, 512), 6)
    assert oracle_lib.space_size(m, "h1")[0] == g["h1_2d_p6_262144el"]["rows"]
    m = mg.box_mesh(3, (32, 32, 32), 6)
    assert oracle_lib.space_size(m, "h1")[0] == g["h1_3d_p6_32768el"]["rows"]


def test_sharing_multiplicity(oracle_lib):
    """RT shared by <= 2 elements, ND by 4, H1 by 8 on a Cartesian mesh."""
    g = gold("paper_pins.json")["sharing_multiplicity"]
    m = mg.box_mesh(3, (3, 3, 3), 3)
    for sp_, k in (("h1", g["h1"]), ("nd", g["nd"]), ("rt", g["rt"])):
        mp, sg = oracle_lib.dof_map(m, sp_)
        cnt = np.bincount(mp.ravel())
        assert cnt.max() == k
        # each element map is injective
        for e in range(m.nel):
            assert len(np.unique(mp[e])) == mp.shape[1]
        assert set(np.unique(sg)) <= {-1, 1}


def test_unscrambled_signs(oracle_lib):
    """App. A.4: on unscrambled structured meshes the only sigma = -1 are RT dofs on coarse y-faces;
    all ND signs are +1 (edges run min->max vertex id = +axis)."""
    p = 3
    m = mg.box_mesh(3, (2, 2, 2), p)
    _, s = oracle_lib.dof_map(m, "nd")
    assert (s == 1).all()
    _, s = oracle_lib.dof_map(m, "rt")
    blk = (p + 1) * p * p
    assert (s[:, :blk] == 1).all() and (s[:, 2 * blk:] == 1).all()
    yb = s[:, blk:2 * blk].reshape(m.nel, p, p + 1, p)  # [cz][vy][cx]
    assert (yb[:, :, 0, :] == -1).all() and (yb[:, :, p, :] == -1).all() and (yb[:, :, 1:p, :] == 1).all()


# ---------------------------------------------------------------- invariants, any geometry
MESHES = [
    ("jitter", lambda p: mg.box_mesh(3, (2, 2, 2), p, jitter=True)),
    ("kershaw", lambda p: mg.box_mesh(3, (6, 2, 2), p, kershaw=0.3)),
    ("scramble", lambda p: mg.box_mesh(3, (2, 3, 2), p, jitter=True, scramble=True)),
]


@pytest.mark.parametrize("name,mk", MESHES)
@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
def test_rowsums_and_symmetry(oracle_lib, name, mk, quad):
    m = mk(3)
    A = to_sparse(oracle_lib.assemble(m, "h1", quad, 1.0, 0.0))
    rs = np.abs(np.asarray(A.sum(axis=1))).max()
    assert rs <= 1e-13 * abs(A).max()
    for sp_ in ("h1", "nd", "rt"):
        B = to_sparse(oracle_lib.assemble(m, sp_, quad, 1.0, 1.0))
        assert abs(B - B.T).max() <= 1e-14 * abs(B).max()
        assert (B.diagonal() > 0).all()


@pytest.mark.parametrize("name,mk", MESHES)
def test_discrete_complex(oracle_lib, name, mk):
    m = mk(2)
    G = oracle_lib.discrete(m, "grad")
    Cc = oracle_lib.discrete(m, "curl")
    assert (np.diff(G.row_ptr) == 2).all() and (np.diff(Cc.row_ptr) == 4).all()
    assert set(np.unique(G.val)) == {-1.0, 1.0} and set(np.unique(Cc.val)) == {-1.0, 1.0}
    Gs, Cs = to_sparse(G), to_sparse(Cc)
    assert abs(Cs @ Gs).max() == 0  # curl grad = 0, exact integer product
    assert np.abs(Gs @ np.ones(Gs.shape[1])).max() == 0
    for quad in ("vertex", "gauss2"):
        Knd = to_sparse(oracle_lib.assemble(m, "nd", quad, 1.0, 0.0))
        assert abs(Knd @ Gs).max() <= 1e-13 * abs(Knd).max()
        Krt = to_sparse(oracle_lib.assemble(m, "rt", quad, 1.0, 0.0))
        assert abs(Krt @ Cs).max() <= 1e-13 * abs(Krt).max()


def _edge_values_per_element(m, mp, sg, field_line_integral):
    """global ND dof values of a field, computed independently in every element from its local
    (+axis) edge geometry times sigma; returns {gid: [values from each element]}."""
    p = m.p
    vals = {}
    np_ = (p + 1) ** 3
    for e in range(m.nel):
        Xe = m.X[e].reshape(3, p + 1, p + 1, p + 1)  # [d][k][j][i]
        for a in range(3):
            ext = [p + 1] * 3
            ext[a] = p
            for z in range(ext[2]):
                for y in range(ext[1]):
                    for x in range(ext[0]):
                        c = [x, y, z]
                        l = a * p * (p + 1) ** 2 + x + ext[0] * (y + ext[1] * z)
                        t = np.array([Xe[d][c[2], c[1], c[0]] for d in range(3)])
                        h = list(c)
                        h[a] += 1
                        hd = np.array([Xe[d][h[2], h[1], h[0]] for d in range(3)])
                        v = sg[e, l] * field_line_integral(t, hd)
                        vals.setdefault(int(mp[e, l]), []).append(v)
    return vals


def _face_values_per_element(m, mp, sg, flux):
    p = m.p
    vals = {}
    for e in range(m.nel):
        Xe = m.X[e].reshape(3, p + 1, p + 1, p + 1)
        for a in range(3):
            up, vp = (a + 1) % 3, (a + 2) % 3
            ext = [p] * 3
            ext[a] = p + 1
            for z in range(ext[2]):
                for y in range(ext[1]):
                    for x in range(ext[0]):
                        c = [x, y, z]
                        l = a * (p + 1) * p * p + x + ext[0] * (y + ext[1] * z)

                        def P(du, dv):
                            q = list(c)
                            q[up] += du
                            q[vp] += dv
                            return np.array([Xe[d][q[2], q[1], q[0]] for d in range(3)])
                        d1 = P(1, 1) - P(0, 0)
                        d2 = P(0, 1) - P(1, 0)
                        v = sg[e, l] * flux(0.5 * np.cross(d1, d2))
                        vals.setdefault(int(mp[e, l]), []).append(v)
    return vals


@pytest.mark.parametrize("name,mk", MESHES)
def test_geometric_signs_stokes(oracle_lib, name, mk):
    """Signs pinned geometrically: every element sharing an ND/RT dof computes the
    same signed value of a field from its own local geometry, and C . ND(a x X / 2) = RT(a),
    G . phi = ND(grad phi) for a linear phi."""
    m = mk(2)
    a = np.array([0.3, -1.1, 0.7])
    b = np.array([1.7, 0.4, -0.9])
    mpn, sgn = oracle_lib.dof_map(m, "nd")
    mpr, sgr = oracle_lib.dof_map(m, "rt")
    nd_u = _edge_values_per_element(m, mpn, sgn, lambda P, Q: 0.5 * np.dot(np.cross(a, P), Q - P))
    nd_g = _edge_values_per_element(m, mpn, sgn, lambda P, Q: np.dot(b, Q - P))
    rt_a = _face_values_per_element(m, mpr, sgr, lambda S: np.dot(a, S))
    for dct in (nd_u, nd_g, rt_a):
        for v in dct.values():
            assert max(v) - min(v) <= 1e-15 * (1 + abs(v[0]))
    ndu = np.array([nd_u[i][0] for i in range(len(nd_u))])
    ndg = np.array([nd_g[i][0] for i in range(len(nd_g))])
    rta = np.array([rt_a[i][0] for i in range(len(rt_a))])
    Cs = to_sparse(oracle_lib.discrete(m, "curl"))
    Gs = to_sparse(oracle_lib.discrete(m, "grad"))
    assert np.abs(Cs @ ndu - rta).max() <= 1e-15
    xyz = _h1_coords(oracle_lib, m)
    assert np.abs(Gs @ (xyz @ b) - ndg).max() <= 1e-14


def test_lumped_mass_is_volume(oracle_lib):
    """affine (sheared) mesh: the vertex-rule H1 mass is diagonal and sums to the domain volume"""
    m = mg.box_mesh(3, (2, 2, 2), 3)
    S = np.array([[1.0, 0.2, 0.1], [0.0, 0.9, 0.3], [0.0, 0.0, 1.1]])
    m.vert = m.vert @ S.T
    m.X = np.einsum("kd,edn->ekn", S, m.X)
    M = to_sparse(oracle_lib.assemble(m, "h1", "vertex", 0.0, 1.0))
    off = M - sp.diags(M.diagonal())
    assert abs(off).max() <= 1e-16
    assert abs(M.sum() - np.linalg.det(S)) <= 1e-14


# ------------------------------------------------------------- independent re-derivations
@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
def test_row_oracle_matches_full(oracle_lib, space):
    m = mg.box_mesh(3, (2, 2, 3), 3, jitter=True, scramble=True)
    A = oracle_lib.assemble(m, space, "vertex", 1.0, 1.0)
    rng = np.random.default_rng(0)
    n = A.row_ptr.shape[0] - 1
    rows = np.unique(rng.integers(0, n, 40))
    R = oracle_lib.assemble_rows(m, rows, space, "vertex", 1.0, 1.0)
    for i, g in enumerate(R.row_id):
        s, e = A.row_ptr[g], A.row_ptr[g + 1]
        rs, re_ = R.row_ptr[i], R.row_ptr[i + 1]
        np.testing.assert_array_equal(A.col[s:e], R.col[rs:re_])
        np.testing.assert_allclose(A.val[s:e], R.val[rs:re_], rtol=0, atol=1e-15 * np.abs(A.val[s:e]).max())


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
def test_rank_split_is_symmetric_permutation(oracle_lib, space):
    """App. A.6: rank-major renumbering is a permutation of the single-rank numbering; each
    rank's owned rows are a contiguous range; the matrix is P A P^T."""
    m1 = mg.box_mesh(3, (2, 2, 4), 2, jitter=True)
    m2 = mg.box_mesh(3, (2, 2, 4), 2, jitter=True, nranks=2)
    A1 = to_sparse(oracle_lib.assemble(m1, space)).toarray()
    A2 = to_sparse(oracle_lib.assemble(m2, space)).toarray()
    mp1, s1 = oracle_lib.dof_map(m1, space)
    mp2, s2 = oracle_lib.dof_map(m2, space)
    np.testing.assert_array_equal(s1, s2)
    perm = np.zeros(mp1.max() + 1, dtype=np.int64)
    perm[mp1.ravel()] = mp2.ravel()
    assert len(np.unique(perm)) == len(perm)
    B = np.zeros_like(A1)
    B[np.ix_(perm, perm)] = A1
    np.testing.assert_array_equal(B, A2)
    n, _, off = oracle_lib.space_size(m2, space)
    assert off[0] == 0 and off[-1] == n and off[1] > 0
    # rank 0 owns exactly the dofs whose minimal element is in slab 0
    half = m2.nel // 2
    owned0 = set(np.unique(mp2[:half]).tolist())
    only1 = set(np.unique(mp2[half:]).tolist()) - owned0
    assert all(g < off[1] for g in owned0) and all(g >= off[1] for g in only1)


def test_scramble_is_a_permutation_h1(oracle_lib):
    """Rotating each element's local frame (App. B) leaves the geometry unchanged: the H1 matrix
    is the same up to a permutation recovered from dof coordinates."""
    p = 3
    ma = mg.box_mesh(3, (2, 2, 2), p, jitter=True)
    mb = mg.box_mesh(3, (2, 2, 2), p, jitter=True, scramble=True)
    Aa = to_sparse(oracle_lib.assemble(ma, "h1", "vertex", 1.0, 1.0)).toarray()
    Ab = to_sparse(oracle_lib.assemble(mb, "h1", "vertex", 1.0, 1.0)).toarray()
    xa, xb = _h1_coords(oracle_lib, ma), _h1_coords(oracle_lib, mb)
    ka = np.lexsort(np.round(xa, 12).T)
    kb = np.lexsort(np.round(xb, 12).T)
    np.testing.assert_allclose(xa[ka], xb[kb], atol=1e-15)
    Pa = Aa[np.ix_(ka, ka)]
    Pb = Ab[np.ix_(kb, kb)]
    assert np.abs(Pa - Pb).max() <= 1e-14 * np.abs(Pa).max()


# ----------------------------------------------------- spectral equivalence (l.131, l.138)
@pytest.mark.parametrize("dim,shape,ps,bound", [(2, (2, 2), range(1, 9), 6.0), (3, (2, 2, 2), range(1, 6), 20.0)])
def test_spectral_equivalence_h1(oracle_lib, dim, shape, ps, bound):
    from oracle import ho
    import scipy.linalg as sla
    kappas = []
    for p in ps:
        m = mg.box_mesh(dim, shape, p, jitter=True)
        mp, _ = oracle_lib.dof_map(m, "h1")
        A_lor = to_sparse(oracle_lib.assemble(m, "h1", "vertex", 1.0, 1.0)).toarray()
        x, _ = oracle_lib.gll(p)
        A_ho = ho.ho_h1_matrix(m, (x + 1) / 2, mp, A_lor.shape[0], 1.0, 1.0)
        ev = sla.eigh(A_ho, A_lor, eigvals_only=True)
        kappas.append(ev.max() / ev.min())
    print(f"H1 {dim}D kappa(A_LOR^-1 A_HO), p = {list(ps)}: {[round(k, 3) for k in kappas]}")
    assert max(kappas) <= bound, kappas
    if dim == 2:
        assert kappas[-1] <= 1.2 * kappas[len(kappas) // 2]  # bounded as p grows, no blow-up


# ------------------------------------ interpolation--histopolation ND / RT (l.142-150, reading P-13)
@pytest.mark.parametrize("p", range(1, 9))
def test_histopolation_delta_and_derivative(oracle_lib, p):
    """h_j = -sum_{k<j} l_k' (SPEC closed form): unit mean over its own GLL sub-interval and zero
    over the others; the derivative of any degree-p nodal polynomial has the nodal differences
    u_j - u_{j-1} as its histopolation coefficients (the 1D root of the discrete gradient)."""
    from oracle import ho
    x, _ = oracle_lib.gll(p)
    s = (x + 1) / 2
    xg, wg = ho.gauss(p + 2)
    for i in range(1, p + 1):
        a, b = s[i - 1], s[i]
        H = ho.histopolation_1d(s, a + (b - a) * xg)
        np.testing.assert_allclose((b - a) * (wg @ H), np.eye(p)[i - 1], atol=1e-12)
    u = np.random.default_rng(p).standard_normal(p + 1)
    t = np.linspace(0.0, 1.0, 17)
    _, D = ho.lagrange_1d(s, t)
    np.testing.assert_allclose(D @ u, ho.histopolation_1d(s, t) @ np.diff(u), atol=1e-9 * np.abs(D @ u).max())


def _ho_vec(oracle_lib, m, space, alpha, beta):
    from oracle import ho
    vm, vs = oracle_lib.dof_map(m, space)
    n, _, _ = oracle_lib.space_size(m, space)
    x, _ = oracle_lib.gll(m.p)
    return ho.ho_vector_matrix(m, space, (x + 1) / 2, vm, vs, n, alpha, beta)


@pytest.mark.parametrize("space", ["nd", "rt"])
def test_ho_vector_p1_is_lowest_order(oracle_lib, space):
    """l.150: 'the lowest-order case of the interpolation--histopolation bases reduces exactly to
    the standard lowest-order Nedelec and Raviart-Thomas elements' -- p = 1 HO matrix (q = 3 Gauss)
    equals the oracle's textbook lowest-order matrix under the Gauss-2 rule, which is exact on a
    Cartesian mesh."""
    m = mg.box_mesh(3, (2, 2, 2), 1)
    A_lor = to_sparse(oracle_lib.assemble(m, space, "gauss2", 1.3, 0.7)).toarray()
    A_ho = _ho_vec(oracle_lib, m, space, 1.3, 0.7)
    assert np.abs(A_ho - A_lor).max() <= 1e-14 * np.abs(A_lor).max()


@pytest.mark.parametrize("space,p", [("nd", 2), ("nd", 3), ("rt", 2), ("rt", 3)])
def test_ho_vector_commuting(oracle_lib, space, p):
    """In the interpolation--histopolation basis the discrete gradient / curl (purely topological,
    l.395-445) map into the kernel of the HO curl-curl / div-div operators: K_ND(alpha) G = 0,
    K_RT(alpha) C = 0 on a warped mesh (exactness of the high-order de Rham sequence)."""
    m = mg.box_mesh(3, (2, 2, 2), p, jitter=True)
    K = _ho_vec(oracle_lib, m, space, 1.0, 0.0)
    D = to_sparse(oracle_lib.discrete(m, "grad" if space == "nd" else "curl")).toarray()
    assert np.abs(K @ D).max() <= 1e-13 * np.abs(K).max()
    assert np.abs(K - K.T).max() <= 1e-14 * np.abs(K).max()


@pytest.mark.parametrize("space,bound", [("nd", 30.0), ("rt", 20.0)])
def test_spectral_equivalence_nd_rt(oracle_lib, space, bound):
    """l.145-148: with the interpolation--histopolation HO basis 'spectral equivalence of the
    high-order and low-order-refined stiffness matrices (and mass matrices) are recovered for
    vector finite element spaces'.  kappa(A_LOR^-1 A_HO) for curl-curl + mass (ND) and div-div +
    mass (RT), LOR under the vertex rule (reading P-1), warped 2x2x2 mesh, p = 1..4; SURVEY c.4
    bounds 30 / 20.  Measured: ND 9.01, 16.44, 18.65, 19.74; RT 3.00, 5.80, 8.84, 10.73."""
    import scipy.linalg as sla
    kappas = []
    for p in range(1, 5):
        m = mg.box_mesh(3, (2, 2, 2), p, jitter=True)
        A_lor = to_sparse(oracle_lib.assemble(m, space, "vertex", 1.0, 1.0)).toarray()
        A_ho = _ho_vec(oracle_lib, m, space, 1.0, 1.0)
        ev = sla.eigh(A_ho, A_lor, eigvals_only=True)
        kappas.append(ev.max() / ev.min())
    print(f"{space} kappa(A_LOR^-1 A_HO), p = 1..4: {[round(k, 3) for k in kappas]}")
    assert max(kappas) <= bound, kappas
    # bounded as p grows: the increments shrink (no blow-up)
    assert kappas[3] - kappas[2] <= kappas[1] - kappas[0]
