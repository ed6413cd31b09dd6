"""Pins of the oracle's 2D H(curl) / H(div) LOR matrices and the 2D discrete / rotated gradient
(conventions: DESIGN.md reading P-29) against what the paper and
the mathematics fix:

* p = 1 unit square: the textbook lowest-order Nedelec / Raviart-Thomas cell matrices (vertex rule:
  mass I/2, curl-curl c c^T with c = (1, -1, -1, 1), div-div d d^T with d = (-1, 1, -1, 1); Gauss-2:
  mass blocks [1/3 1/6; 1/6 1/3]) (the lowest-order case is the standard element);
* exact sequence: curl-curl(ND) G = 0 and div-div(RT) G_perp = 0 on jittered, scrambled meshes;
* de Rham factorisations: K_H1(alpha) = G^T M_ND(alpha) G = G_perp^T M_RT(alpha) G_perp (the
  gradient and the rotated gradient of Q1 lie in the lowest-order spaces);
* geometry of the signs: the dofs of a constant field c (ND: c.(Q - P) along each edge P -> Q of G;
  RT: c.rot90(Q - P) along the tau of G_perp) give u^T M u = |c|^2 * area;
* counts: n = n_edges p + n_el 2p(p-1), nnz = the number of dof pairs sharing a LOR cell (brute
  force over the cells)."""
import numpy as np
import pytest

from oracle import bc
from paper_2210_12253_b200 import meshgen as mg

SQ = np.array([[0.0, 0.0], [1.0, 0.0], [0.0, 1.0], [1.0, 1.0]])


def test_unit_square_textbook(oracle_lib):
    O = oracle_lib
    c = np.array([1.0, -1.0, -1.0, 1.0])
    d = np.array([-1.0, 1.0, -1.0, 1.0])
    assert np.array_equal(O.local_matrix(2, "nd", "vertex", 1.0, 0.0, SQ), np.outer(c, c))
    assert np.array_equal(O.local_matrix(2, "rt", "vertex", 1.0, 0.0, SQ), np.outer(d, d))
    for sp in ("nd", "rt"):
        assert np.array_equal(O.local_matrix(2, sp, "vertex", 0.0, 1.0, SQ), 0.5 * np.eye(4))
        g = O.local_matrix(2, sp, "gauss2", 0.0, 1.0, SQ)
        blk = np.array([[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
        ref = np.zeros((4, 4))
        ref[:2, :2] = ref[2:, 2:] = blk
        assert np.max(np.abs(g - ref)) < 1e-15


def _dense(A):
    return A.dense(A.row_ptr.shape[0] - 1)


@pytest.mark.parametrize("p", [1, 2, 3, 4])
@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
def test_exact_sequence_and_de_rham(oracle_lib, p, quad):
    O = oracle_lib
    m = mg.box_mesh(2, (3, 2), p, jitter=True, scramble=True)
    G = _dense(O.discrete(m, "grad"))
    Gp = _dense(O.discrete(m, "rotgrad"))
    Knd = _dense(O.assemble(m, "nd", quad, 1.3, 0.0))
    Krt = _dense(O.assemble(m, "rt", quad, 1.3, 0.0))
    assert np.abs(Knd @ G).max() < 1e-13 * np.abs(Knd).max()
    assert np.abs(Krt @ Gp).max() < 1e-13 * np.abs(Krt).max()
    Kh1 = _dense(O.assemble(m, "h1", quad, 1.3, 0.0))
    Mnd = _dense(O.assemble(m, "nd", quad, 0.0, 1.3))
    Mrt = _dense(O.assemble(m, "rt", quad, 0.0, 1.3))
    assert np.abs(G.T @ Mnd @ G - Kh1).max() < 1e-13 * np.abs(Kh1).max()
    assert np.abs(Gp.T @ Mrt @ Gp - Kh1).max() < 1e-13 * np.abs(Kh1).max()


def _ends(O, m, which):
    D = O.discrete(m, which)
    xy = bc.coordinates(m).T
    cols, vals = D.col.reshape(-1, 2), D.val.reshape(-1, 2)
    tail = np.where(vals[:, 0] < 0, cols[:, 0], cols[:, 1])
    head = np.where(vals[:, 0] < 0, cols[:, 1], cols[:, 0])
    return xy[tail], xy[head]


@pytest.mark.parametrize("p", [1, 2, 3])
def test_constant_field_energy(oracle_lib, p):
    O = oracle_lib
    m = mg.box_mesh(2, (3, 2), p, jitter=True, scramble=True)
    c = np.array([0.7, -1.9])
    P, Q = _ends(O, m, "grad")
    u = (Q - P) @ c
    M = _dense(O.assemble(m, "nd", "vertex", 0.0, 1.0))
    assert abs(u @ M @ u - c @ c) < 1e-12 * (c @ c)
    P, Q = _ends(O, m, "rotgrad")
    t = Q - P
    u = np.stack([-t[:, 1], t[:, 0]], axis=1) @ c
    M = _dense(O.assemble(m, "rt", "vertex", 0.0, 1.0))
    assert abs(u @ M @ u - c @ c) < 1e-12 * (c @ c)


@pytest.mark.parametrize("space", ["nd", "rt"])
@pytest.mark.parametrize("p", [1, 2, 4])
def test_counts_brute_force(oracle_lib, space, p):
    O = oracle_lib
    nx, ny = 3, 2
    m = mg.box_mesh(2, (nx, ny), p, scramble=True)
    ne = nx * (ny + 1) + ny * (nx + 1)
    A = O.assemble(m, space, "vertex", 1.0, 1.0)
    n = A.row_ptr.shape[0] - 1
    assert n == ne * p + m.nel * 2 * p * (p - 1)
    mp, sg = O.dof_map(m, space)
    assert set(np.unique(sg)) <= {-1, 1}
    pairs = set()
    for e in range(m.nel):
        for ky in range(p):
            for kx in range(p):
                loc = []
                for i in range(4):
                    fam, off = i // 2, i & 1
                    x = [kx, ky]
                    if space == "nd":
                        x[1 - fam] += off
                    else:
                        x[fam] += off
                    ext0 = (p if fam == 0 else p + 1) if space == "nd" else (p + 1 if fam == 0 else p)
                    loc.append(mp[e, fam * p * (p + 1) + x[0] + ext0 * x[1]])
                pairs.update((a, b) for a in loc for b in loc)
    assert A.nnz == len(pairs)


def _ho2(O, m, space, alpha, beta):
    from oracle import ho
    vm, vs = O.dof_map(m, space)
    n = int(vm.max()) + 1
    x, _ = O.gll(m.p)
    return ho.ho_vector_matrix_2d(m, space, (x + 1) / 2, vm, vs, n, alpha, beta)


@pytest.mark.parametrize("space", ["nd", "rt"])
def test_ho2d_p1_is_lowest_order(oracle_lib, space):
    """the p = 1 interpolation-histopolation matrix (q = 3 Gauss) equals the lowest-order
    matrix under the Gauss-2 rule (exact on a Cartesian mesh)"""
    m = mg.box_mesh(2, (3, 2), 1)
    A_lor = _dense(oracle_lib.assemble(m, space, "gauss2", 1.3, 0.7))
    A_ho = _ho2(oracle_lib, m, space, 1.3, 0.7)
    assert np.abs(A_ho - A_lor).max() <= 1e-14 * np.abs(A_lor).max()


@pytest.mark.parametrize("space,p", [("nd", 2), ("nd", 4), ("rt", 2), ("rt", 4)])
def test_ho2d_commuting(oracle_lib, space, p):
    """the topological G / G_perp map into the kernels of the HO curl-curl / div-div (exact sequence)"""
    m = mg.box_mesh(2, (3, 2), p, jitter=True)
    K = _ho2(oracle_lib, m, space, 1.0, 0.0)
    D = _dense(oracle_lib.discrete(m, "grad" if space == "nd" else "rotgrad"))
    assert np.abs(K @ D).max() <= 1e-12 * np.abs(K).max()


@pytest.mark.parametrize("space", ["nd", "rt"])
def test_spectral_equivalence_2d(oracle_lib, space):
    """kappa(A_LOR^-1 A_HO) bounded in p for the 2D vector spaces (curl-curl / div-div +
    mass, vertex-rule LOR, warped 3x2 mesh, p = 1..6; SURVEY c.4 bound 12 for 2D ND)"""
    import scipy.linalg as sla
    kappas = []
    for p in range(1, 7):
        m = mg.box_mesh(2, (3, 2), p, jitter=True)
        A_lor = _dense(oracle_lib.assemble(m, space, "vertex", 1.0, 1.0))
        A_ho = _ho2(oracle_lib, m, space, 1.0, 1.0)
        ev = sla.eigh(A_ho, A_lor, eigvals_only=True)
        kappas.append(ev.max() / ev.min())
    print(f"2D {space} kappa(A_LOR^-1 A_HO), p = 1..6: {[round(k, 3) for k in kappas]}")
    assert max(kappas) <= 12.0, kappas
    assert kappas[5] - kappas[4] <= kappas[1] - kappas[0]  # increments shrink: no blow-up
