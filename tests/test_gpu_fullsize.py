"""GPU parity at (and near) the BASELINE sizes, whole matrices, in the launch configuration
bench.py times ("full matrices at C1/C2/C4 and single-GPU C3/C5" instead of 2-3 k sampled
rows).  Every row_ptr / col entry bit-exact, every value under the P-10 rule (tests/parity.py).

* C2 (32^3, p = 4, H1) in full: 2,146,689 rows, 57,066,625 nnz (oracle: ~137 M triplets);
* C4 / C5 recipes (ND / RT, p = 4) at 16^3, and C2-J (jittered) / C3 (Kershaw, p = 8) at 12^3;
* the discrete gradient at C4 size and the discrete curl at C5 size (32^3, p = 4), bit-exact,
  plus G / C at p = 8 and through a 3-rank split;
* the 3D Gauss-2 rule at every p = 1..8 for H1, ND and RT.
"""
import numpy as np
import pytest

from paper_2210_12253_b200 import meshgen as mg
from tests.parity import compare_csr_arrays, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def full_case(O, m, form, what):
    from paper_2210_12253_b200.lor import LOR
    ctx = LOR(m)
    sp = form["space"]
    q = ctx.query(sp)
    rp, col, val = ctx.assemble(sp, form["alpha"], form["beta"], form["quad"])
    ctx.sync()
    rp, col, val = to_host(rp), to_host(col), to_host(val)
    path = ctx.fill_path(sp)
    ctx.close()
    ref = O.assemble(m, sp, form["quad"], form["alpha"], form["beta"])
    assert q["nnz"] == ref.nnz
    res = compare_csr_arrays(rp, col, val, ref, 0, q["n_local"], what)
    print(f"{what}: path {path}, rows {res['rows']}, max_rel {res['max_rel']:.2e}, "
          f"sub-floor err/rowmax {res['floor_abs']:.2e}")
    return res


def test_c2_full_matrix(torch_cuda, oracle_lib):
    m, form = mg.config_mesh("C2")
    res = full_case(oracle_lib, m, form, "C2 full")
    assert res["rows"] == 2146689


@pytest.mark.parametrize("cfg,n", [("C4", 16), ("C5", 16), ("C2-J", 12), ("C3", 12)])
def test_config_recipe_full_matrix(torch_cuda, oracle_lib, cfg, n):
    m, form = mg.config_mesh(cfg, n=n)
    full_case(oracle_lib, m, form, f"{cfg}@{n}^3 full")


@pytest.mark.parametrize("which,cfg", [("grad", "C4"), ("curl", "C5"), ("grad", "C5")])
def test_discrete_full_size(torch_cuda, oracle_lib, which, cfg):
    from paper_2210_12253_b200.lor import LOR
    m, _ = mg.config_mesh(cfg)
    ctx = LOR(m)
    rp, col, val = ctx.discrete(which)
    ctx.sync()
    ref = oracle_lib.discrete(m, which)
    np.testing.assert_array_equal(to_host(rp), ref.row_ptr)
    np.testing.assert_array_equal(to_host(col), ref.col)
    np.testing.assert_array_equal(to_host(val), ref.val)
    ctx.close()


@pytest.mark.parametrize("which", ["grad", "curl"])
@pytest.mark.parametrize("p", [7, 8])
def test_discrete_high_p(torch_cuda, oracle_lib, which, p):
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(3, (2, 2, 3), p, jitter=True, scramble=True)
    ctx = LOR(m)
    rp, col, val = ctx.discrete(which)
    ctx.sync()
    ref = oracle_lib.discrete(m, which)
    np.testing.assert_array_equal(to_host(rp), ref.row_ptr)
    np.testing.assert_array_equal(to_host(col), ref.col)
    np.testing.assert_array_equal(to_host(val), ref.val)


@pytest.mark.parametrize("which", ["grad", "curl"])
def test_discrete_per_rank(torch_cuda, oracle_lib, which):
    """rows owned by each of 3 ranks (no communication): their union in rank
    order is the oracle's rank-major operator"""
    from paper_2210_12253_b200.lor import LOR
    nranks = 3
    m = mg.box_mesh(3, (2, 3, 2 * nranks), 4, jitter=True, scramble=True, nranks=nranks)
    ref = oracle_lib.discrete(m, which, nranks=nranks)
    w = 2 if which == "grad" else 4
    row_sp = "nd" if which == "grad" else "rt"
    for r in range(nranks):
        ctx = LOR(m, rank=r, nranks=nranks)
        q = ctx.query(row_sp)
        rp, col, val = ctx.discrete(which)
        ctx.sync()
        b, n = q["row_begin"], q["n_local"]
        np.testing.assert_array_equal(to_host(rp), w * np.arange(n + 1))
        np.testing.assert_array_equal(to_host(col), ref.col[w * b:w * (b + n)])
        np.testing.assert_array_equal(to_host(val), ref.val[w * b:w * (b + n)])
        ctx.close()


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_gauss2_every_p(torch_cuda, oracle_lib, space, p):
    m = mg.box_mesh(3, (3, 2, 2) if p <= 4 else (2, 2, 2), p, jitter=True, scramble=True)
    full_case(oracle_lib, m, dict(space=space, alpha=1.3, beta=0.7, quad="gauss2"), f"{space} gauss2 p={p}")


@pytest.mark.parametrize("which", ["grad", "curl"])
def test_discrete_map_path_equals_block_path(torch_cuda, monkeypatch, which):
    """G / C from the setup element restrictions (k_discrete_map, default) and from the per-element
    affine blocks (k_discrete, LOR_EMAP=0): bit-identical arrays"""
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(3, (3, 3, 2), 3, jitter=True, scramble=True)
    outs = []
    for emap in ("1", "0"):
        monkeypatch.setenv("LOR_EMAP", emap)
        ctx = LOR(m)
        outs.append([to_host(t).copy() for t in ctx.discrete(which)])
        ctx.sync()
        ctx.close()
    for a, b in zip(*outs):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg", ["C2", "C4", "C5"])
def test_variable_coefficients_full_size(torch_cuda, oracle_lib, cfg):
    """BASELINE configs with the bench's coefficient fields (C2-V / C4-V / C5-V, the launch
    configuration bench.py times): 3000 sampled rows + all rows of the first and last element against
    the row oracle with the same coefficient E-vectors"""
    from paper_2210_12253_b200.lor import LOR
    from tests.parity import compare_rows
    m, form = mg.config_mesh(cfg)
    xs = [m.X[:, d, :] for d in range(3)]
    ca = np.ascontiguousarray(1.0 + 0.5 * np.sin(3.0 * xs[0]) * np.cos(2.0 * xs[1]) + xs[2] * xs[2])
    cb = np.ascontiguousarray(2.0 + np.cos(xs[0] + xs[1] + xs[2]))
    ctx = LOR(m)
    ctx.set_coefficients(ca, cb)
    sp = form["space"]
    rp, col, val = (to_host(t) for t in ctx.assemble(sp, 1.0, 1.0, "vertex"))
    ctx.sync()
    n = rp.shape[0] - 1
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([rng.choice(n, 3000, replace=False), np.arange(100), np.arange(n - 100, n)]))
    ref = oracle_lib.assemble_rows(m, rows, sp, "vertex", 1.0, 1.0, coef=(ca, cb))
    compare_rows(rp, col, val, ref, 0, None, f"{cfg}-V sampled rows")
    ctx.close()


def test_coordinates_full_size_c2(torch_cuda):
    """C2-X: the coordinate vectors at full size -- every owned vertex equals its E-vector copy in the
    minimal element (the copies of a shared vertex agree to rounding) and the Cartesian lattice"""
    from paper_2210_12253_b200.lor import LOR
    m, _ = mg.config_mesh("C2")
    ctx = LOR(m)
    xyz = to_host(ctx.coordinates())
    mp, _ = ctx.dof_map("h1")
    mp = to_host(mp)
    ctx.sync()
    # every element's E-vector agrees with the deduplicated coordinates of its dofs
    for d in range(3):
        assert np.max(np.abs(xyz[d][mp] - m.X[:, d, :])) < 1e-15
    # the lattice: 32 elements x GLL(4) per axis, each point once
    x1 = mg.gll_points_01(4)
    axis = np.unique(np.round(np.concatenate([(e + x1) / 32 for e in range(32)]), 14))
    assert axis.shape[0] == 129
    for d in range(3):
        assert np.max(np.min(np.abs(xyz[d][:, None] - axis[None, :]), axis=1)) < 1e-14
