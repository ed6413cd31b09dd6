"""Pins of the oracle's variable coefficients (DESIGN.md
reading P-28: alpha a(x), beta b(x) with a, b given at the LOR vertices as E-vectors and interpolated
multilinearly inside each LOR cell) against what the mathematics fixes:

* a = b = 1 reproduces the constant-coefficient matrices: bit for bit under the vertex rule (the
  interpolation weights at a corner are exactly 0 / 1), to rounding under Gauss-2 (the eight
  weights sum to 1 up to a few ulps);
* mass with a multilinear b on a Cartesian box: the sum of all H1 mass entries is the exact
  integral of b (both rules integrate multilinear functions exactly on boxes);
* H1 energy of a linear u = c.x with a multilinear a: u^T K u = |c|^2 int a;
* ND curl energy of the interpolant of u = 1/2 a x x (dofs = line integrals 1/2 (a x P).(Q - P) along
  the edges P -> Q given by the discrete gradient): u^T K u = |a|^2 int alpha-coefficient;
* RT div energy of u = x (dofs = fluxes x_c . A_f, vector area A_f = 1/2 sum_e C_fe (P_e x Q_e) from
  the discrete curl and gradient): u^T K u = 9 int a.
The oracle's ND/RT dof geometry comes from its own G and C, which are pinned independently
(test_oracle_pins.py: Stokes / vector-area identities)."""
import numpy as np
import pytest

from oracle import bc
from paper_2210_12253_b200 import meshgen as mg


def _evec(m, f):
    """scalar E-vector of f sampled at the coordinate E-vector points"""
    return np.ascontiguousarray(f(*[m.X[:, d, :] for d in range(m.dim)]))


def _lin3(x, y, z):
    return 1.0 + x + 2.0 * y + 3.0 * z + 4.0 * x * y * z


INT_LIN3 = 1.0 + 0.5 + 1.0 + 1.5 + 0.5  # integral of _lin3 over [0,1]^3


def _dense(A):
    return A.dense(A.row_ptr.shape[0] - 1)


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
def test_unit_coefficients_bitwise(oracle_lib, space, quad):
    m = mg.box_mesh(3, (2, 2, 2), 2, jitter=True, scramble=True)
    one = np.ones((m.nel, (m.p + 1) ** 3))
    A0 = oracle_lib.assemble(m, space, quad, 1.3, 0.7)
    A1 = oracle_lib.assemble(m, space, quad, 1.3, 0.7, coef=(one, one))
    assert np.array_equal(A0.col, A1.col)
    if quad == "vertex":
        assert np.array_equal(A0.val, A1.val)
    else:
        assert np.max(np.abs(A0.val - A1.val)) <= 8 * 2.0 ** -53 * np.abs(A0.val).max()


@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
@pytest.mark.parametrize("p", [1, 2, 3])
def test_mass_integral_multilinear(oracle_lib, quad, p):
    m = mg.box_mesh(3, (2, 3, 2), p, scramble=True)
    b = _evec(m, _lin3)
    A = oracle_lib.assemble(m, "h1", quad, 0.0, 1.0, coef=(np.ones_like(b), b))
    assert abs(A.val.sum() - INT_LIN3) < 1e-12 * INT_LIN3


@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
@pytest.mark.parametrize("p", [1, 3])
def test_h1_energy_linear(oracle_lib, quad, p):
    m = mg.box_mesh(3, (2, 2, 3), p, scramble=True)
    a = _evec(m, _lin3)
    A = oracle_lib.assemble(m, "h1", quad, 1.0, 0.0, coef=(a, np.ones_like(a)))
    c = np.array([0.3, -1.1, 0.7])
    u = c @ bc.coordinates(m)
    e = u @ (_dense(A) @ u)
    assert abs(e - (c @ c) * INT_LIN3) < 1e-11 * (c @ c) * INT_LIN3


def _edges(O, m):
    G = O.discrete(m, "grad")
    xyz = bc.coordinates(m).T
    cols, vals = G.col.reshape(-1, 2), G.val.reshape(-1, 2)
    tail = np.where(vals[:, 0] < 0, cols[:, 0], cols[:, 1])
    head = np.where(vals[:, 0] < 0, cols[:, 1], cols[:, 0])
    return xyz[tail], xyz[head]


@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
@pytest.mark.parametrize("p", [1, 2])
def test_nd_curl_energy(oracle_lib, quad, p):
    m = mg.box_mesh(3, (2, 2, 2), p, scramble=True)
    a = _evec(m, _lin3)
    A = oracle_lib.assemble(m, "nd", quad, 1.0, 0.0, coef=(a, np.ones_like(a)))
    P, Q = _edges(oracle_lib, m)
    av = np.array([0.4, -0.9, 1.3])
    u = 0.5 * np.einsum("ij,ij->i", np.cross(av, P), Q - P)
    e = u @ (_dense(A) @ u)
    assert abs(e - (av @ av) * INT_LIN3) < 1e-11 * (av @ av) * INT_LIN3


@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
@pytest.mark.parametrize("p", [1, 2])
def test_rt_div_energy(oracle_lib, quad, p):
    m = mg.box_mesh(3, (2, 2, 2), p, scramble=True)
    a = _evec(m, _lin3)
    A = oracle_lib.assemble(m, "rt", quad, 1.0, 0.0, coef=(a, np.ones_like(a)))
    P, Q = _edges(oracle_lib, m)
    Cc = oracle_lib.discrete(m, "curl")
    ce, cv = Cc.col.reshape(-1, 4), Cc.val.reshape(-1, 4)
    area = 0.5 * np.einsum("fk,fkd->fd", cv, np.cross(P[ce], Q[ce]))
    centroid = 0.25 * (P[ce] + Q[ce]).sum(axis=1) / 2.0
    u = np.einsum("fd,fd->f", centroid, area)
    e = u @ (_dense(A) @ u)
    assert abs(e - 9.0 * INT_LIN3) < 1e-11 * 9.0 * INT_LIN3
