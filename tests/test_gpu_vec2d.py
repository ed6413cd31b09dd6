"""GPU parity of the 2D H(curl) / H(div) LOR matrices and the 2D discrete / rotated gradient (SURVEY
8(f) NEXT-2; reading P-29) through the C ABI against the oracle:
element restrictions and signs bit-exact, pattern bit-exact, values within the P-10b rule, G and
G_perp bit-exact; every p, both rules, jittered and orientation-scrambled quads, variable
coefficients, boundary dofs."""
import numpy as np
import pytest

from paper_2210_12253_b200 import meshgen as mg
from tests.parity import compare_full, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


@pytest.mark.parametrize("space", ["nd", "rt"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
def test_vec2d_parity(torch_cuda, oracle_lib, space, p, quad):
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(2, (3, 4), p, jitter=True, scramble=True)
    ctx = LOR(m)
    mp, sg = ctx.dof_map(space)
    rm, rs = oracle_lib.dof_map(m, space)
    assert np.array_equal(to_host(mp), rm) and np.array_equal(to_host(sg), rs), "element restriction"
    rp, col, val = ctx.assemble(space, 1.3, 0.7, quad)
    ctx.sync()
    q = ctx.query(space)
    ref = oracle_lib.assemble(m, space, quad, 1.3, 0.7)
    assert q["nnz"] == ref.nnz
    compare_full(to_host(rp), to_host(col), to_host(val), ref, 0, q["n_local"], f"2D {space} p={p} {quad}")


@pytest.mark.parametrize("which", ["grad", "rotgrad"])
@pytest.mark.parametrize("p", [1, 2, 5, 8])
def test_vec2d_discrete(torch_cuda, oracle_lib, which, p):
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(2, (3, 4), p, jitter=True, scramble=True)
    ctx = LOR(m)
    rp, col, val = ctx.discrete(which)
    ctx.sync()
    ref = oracle_lib.discrete(m, which)
    assert np.array_equal(to_host(rp), ref.row_ptr)
    assert np.array_equal(to_host(col), ref.col) and np.array_equal(to_host(val), ref.val), which


def test_vec2d_coefficients_and_boundary(torch_cuda, oracle_lib):
    from oracle import bc
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(2, (4, 3), 3, jitter=True, scramble=True)
    a = np.ascontiguousarray(1.0 + 0.5 * np.sin(3.0 * m.X[:, 0, :]) * np.cos(2.0 * m.X[:, 1, :]))
    b = np.ascontiguousarray(2.0 + np.cos(m.X[:, 0, :] + m.X[:, 1, :]))
    ctx = LOR(m)
    ctx.set_coefficients(a, b)
    for space in ("nd", "rt"):
        rp, col, val = ctx.assemble(space, 1.3, 0.7, "vertex")
        ctx.sync()
        q = ctx.query(space)
        compare_full(to_host(rp), to_host(col), to_host(val),
                     oracle_lib.assemble(m, space, "vertex", 1.3, 0.7, coef=(a, b)), 0, q["n_local"], f"2D coef {space}")
        assert np.array_equal(to_host(ctx.boundary_dofs(space)).astype(np.int64), bc.boundary_dofs(m, space))


@pytest.mark.parametrize("space", ["nd", "rt"])
def test_vec2d_parcsr_and_a4(torch_cuda, oracle_lib, space):
    """NEXT-1 on the 2D vector spaces: ParCSR split (one rank: diag block = the matrix with the
    diagonal first) and A4 with the boundary dofs, against oracle/bc.py; the 2D gradient / rotated
    gradient split (all ascending)"""
    from oracle import bc
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(2, (4, 3), 3, jitter=True, scramble=True)
    ctx = LOR(m)
    A = ctx.assemble(space, 1.3, 0.7, "vertex")
    ctx.sync()
    P = ctx.parcsr(space, A)
    ess = ctx.boundary_dofs(space)
    ctx.eliminate_bc(space, ess, P)
    ctx.sync()
    ref = oracle_lib.assemble(m, space, "vertex", 1.3, 0.7)
    n = ref.row_ptr.shape[0] - 1
    R = bc.parcsr_split(bc.eliminate(ref, bc.boundary_dofs(m, space)), 0, n, 0, n)
    assert np.array_equal(to_host(P["diag_row_ptr"]), R["diag_row_ptr"])
    nd = len(R["diag_col"])
    assert np.array_equal(to_host(P["diag_col"])[:nd], R["diag_col"])
    dv = to_host(P["diag_val"])[:nd]
    mark = np.zeros(n, dtype=bool)
    mark[bc.boundary_dofs(m, space)] = True
    rows = np.repeat(np.arange(n), np.diff(R["diag_row_ptr"]))
    k = mark[rows] | mark[R["diag_col"]]
    assert np.array_equal(dv[k], R["diag_val"][k])
    assert np.allclose(dv[~k], R["diag_val"][~k], rtol=1e-12, atol=1e-14 * np.abs(ref.val).max())
    which = "grad" if space == "nd" else "rotgrad"
    D = ctx.discrete(which)
    ctx.sync()
    PD = ctx.parcsr(which, D)
    ctx.sync()
    RD = bc.parcsr_split(oracle_lib.discrete(m, which), 0, n, 0, int(oracle_lib.space_size(m, "h1")[0]), square=False)
    for key in ("diag_row_ptr", "diag_col", "diag_val"):
        assert np.array_equal(to_host(PD[key])[:len(RD[key])], RD[key]), key
