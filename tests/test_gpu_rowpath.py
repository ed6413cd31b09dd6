"""GPU parity of the per-row path lor_assemble_{h1,nd,rt} take at p = 1 on one rank (lor_fill_path 2,
lor_legacy.cu, DESIGN.md section 4 "p = 1"): a macro-element of order 1 is a single LOR cell
(the LOR mesh is then the mesh itself), so the assembly is the unstructured one --
dense 8x8 cell matrices (the sub-cell math of every other path, P-10b values), one warp per row
gathering the <= 64 candidates of its <= 8 cells through the dof -> cell transpose, ascending
columns, duplicates summed.  Compared with the oracle row by row on Cartesian, jittered/scrambled,
Kershaw, shuffled-numbering and irregular (L-shaped, valence-3 edge) meshes, through numeric
re-assembly, a coordinate update, degenerate geometry and the fallbacks (coefficients, Gauss-2,
LOR_ROWPATH=0).  ND / RT: the element restriction and orientation signs of the space (element =
cell), 12x12 / 6x6 cell matrices, values s_i s_j A_ij; orientation-scrambled meshes included."""
import numpy as np
import pytest

from paper_2210_12253_b200 import meshgen as mg
from tests.parity import compare_full, compare_rows, to_host
from tests.test_gpu_xframe import l_shaped, shuffled

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _mesh(kind):
    if kind == "cartesian":
        return mg.box_mesh(3, (5, 4, 3), 1)
    if kind == "jitscr":
        return mg.box_mesh(3, (5, 4, 3), 1, jitter=True, scramble=True)
    if kind == "kershaw":
        return mg.box_mesh(3, (6, 6, 6), 1, kershaw=0.3)
    if kind == "shuffled":
        return shuffled(mg.box_mesh(3, (4, 4, 3), 1, jitter=True, scramble=True), seed=5)
    return l_shaped(mg.box_mesh(3, (4, 4, 3), 1, jitter=True, scramble=True))


@pytest.mark.parametrize("kind", ["cartesian", "jitscr", "kershaw", "shuffled", "lshaped"])
def test_rowpath_parity(torch_cuda, oracle_lib, kind):
    from paper_2210_12253_b200.lor import LOR
    m = _mesh(kind)
    ctx = LOR(m)
    assert ctx.fill_path("h1") == 2
    q = ctx.query("h1")
    rp, col, val = ctx.assemble("h1", 1.3, 0.7, "vertex")
    ctx.sync()
    ref = oracle_lib.assemble(m, "h1", "vertex", 1.3, 0.7)
    assert q["nnz"] == ref.nnz
    compare_full(to_host(rp), to_host(col), to_host(val), ref, 0, q["n_local"], f"rowpath {kind}")
    # numeric-only re-assembly with other constants: same pattern, the oracle's values
    ctx.reassemble("h1", 0.4, 2.5, "vertex", out=(rp, col, val))
    ctx.sync()
    compare_full(to_host(rp), to_host(col), to_host(val), oracle_lib.assemble(m, "h1", "vertex", 0.4, 2.5), 0,
                 q["n_local"], f"rowpath {kind} reassembly")
    ctx.close()


def test_rowpath_coordinate_update(torch_cuda, oracle_lib):
    """the broken LOR coordinates of the per-row path follow lor_update_coordinates"""
    import torch
    from paper_2210_12253_b200.lor import LOR
    ma = mg.box_mesh(3, (4, 3, 3), 1)
    mb = mg.box_mesh(3, (4, 3, 3), 1, jitter=True)
    ctx = LOR(ma)
    assert ctx.fill_path("h1") == 2
    out = ctx.assemble("h1", 1.3, 0.7, "vertex")
    ctx.sync()
    ctx.update_coordinates(torch.from_numpy(np.ascontiguousarray(mb.X)).cuda())
    ctx.reassemble("h1", 1.3, 0.7, "vertex", out=out)
    ctx.sync()
    q = ctx.query("h1")
    compare_full(*(to_host(t) for t in out), oracle_lib.assemble(mb, "h1", "vertex", 1.3, 0.7), 0, q["n_local"],
                 "rowpath after coordinate update")
    ctx.close()


@pytest.mark.parametrize("what", ["coef", "gauss2", "off"])
def test_rowpath_fallbacks(torch_cuda, oracle_lib, monkeypatch, what):
    """variable coefficients and Gauss-2 take the other paths; LOR_ROWPATH=0 keeps the frame"""
    from paper_2210_12253_b200.lor import LOR
    from tests.test_gpu_coef import _coefs
    if what == "off":
        monkeypatch.setenv("LOR_ROWPATH", "0")
    m = mg.box_mesh(3, (4, 3, 3), 1, jitter=True, scramble=True)
    ctx = LOR(m)
    quad, coef = ("gauss2" if what == "gauss2" else "vertex"), None
    if what == "coef":
        coef = _coefs(m)
        ctx.set_coefficients(*coef)
    assert ctx.fill_path("h1") == (1 if what in ("coef", "off") else 2)
    q = ctx.query("h1")
    out = ctx.assemble("h1", 1.3, 0.7, quad)
    ctx.sync()
    compare_full(*(to_host(t) for t in out), oracle_lib.assemble(m, "h1", quad, 1.3, 0.7, coef=coef), 0,
                 q["n_local"], f"p=1 {what}")
    ctx.close()


def test_rowpath_degenerate_reported(torch_cuda):
    from paper_2210_12253_b200.lor import LOR, LorError
    m = mg.box_mesh(3, (3, 3, 3), 1)
    X = m.X.copy()
    X[13, :, 0] = X[13, :, 7] + (X[13, :, 7] - X[13, :, 0])  # corner 0 beyond corner 7: det J < 0
    m.X = X
    ctx = LOR(m)
    assert ctx.fill_path("h1") == 2
    ctx.assemble("h1")
    with pytest.raises(LorError) as ei:
        ctx.sync()
    assert "degenerate-geometry(element=" in str(ei.value)


def test_rowpath_sampled_large(torch_cuda, oracle_lib):
    """96^3 Kershaw elements (the vector_sweep / legacy_sweep size) in the launch configuration the
    sweeps time: the Q1 pattern closed form (nnz = (3n+1)^3, row lengths 8..27), 2000 sampled rows
    against the oracle's row routine"""
    from paper_2210_12253_b200.lor import LOR
    n = 96
    m = mg.box_mesh(3, (n, n, n), 1, kershaw=0.3)
    ctx = LOR(m)
    assert ctx.fill_path("h1") == 2
    q = ctx.query("h1")
    assert q["n_local"] == (n + 1) ** 3 and q["nnz"] == (3 * n + 1) ** 3
    rp, col, val = ctx.assemble("h1", 1.0, 1.0, "vertex")
    ctx.sync()
    rp, col, val = to_host(rp), to_host(col), to_host(val)
    d = np.diff(rp)
    assert d.min() == 8 and d.max() == 27
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([rng.integers(0, q["n_local"], 2000), [0, q["n_local"] - 1]]))
    ref = oracle_lib.assemble_rows(m, rows, "h1", "vertex", 1.0, 1.0)
    compare_rows(rp, col, val, ref, 0, what="p=1 96^3 sampled")
    ctx.close()


@pytest.mark.parametrize("space", ["nd", "rt"])
@pytest.mark.parametrize("kind", ["cartesian", "jitscr", "kershaw", "shuffled", "lshaped"])
def test_rowpath_vector_parity(torch_cuda, oracle_lib, space, kind):
    from paper_2210_12253_b200.lor import LOR
    m = _mesh(kind)
    ctx = LOR(m)
    assert ctx.fill_path(space) == 2
    q = ctx.query(space)
    rp, col, val = ctx.assemble(space, 1.3, 0.7, "vertex")
    ctx.sync()
    ref = oracle_lib.assemble(m, space, "vertex", 1.3, 0.7)
    assert q["nnz"] == ref.nnz
    compare_full(to_host(rp), to_host(col), to_host(val), ref, 0, q["n_local"], f"rowpath {space} {kind}")
    ctx.reassemble(space, 0.4, 2.5, "vertex", out=(rp, col, val))
    ctx.sync()
    compare_full(to_host(rp), to_host(col), to_host(val), oracle_lib.assemble(m, space, "vertex", 0.4, 2.5), 0,
                 q["n_local"], f"rowpath {space} {kind} reassembly")
    ctx.close()


@pytest.mark.parametrize("space", ["nd", "rt"])
@pytest.mark.parametrize("what", ["coef", "gauss2", "off", "coords"])
def test_rowpath_vector_fallbacks(torch_cuda, oracle_lib, monkeypatch, space, what):
    """coefficients / Gauss-2 / LOR_ROWPATH=0 take the other paths; a coordinate update is seen"""
    import torch
    from paper_2210_12253_b200.lor import LOR
    from tests.test_gpu_coef import _coefs
    if what == "off":
        monkeypatch.setenv("LOR_ROWPATH", "0")
    m = mg.box_mesh(3, (4, 3, 3), 1, jitter=True, scramble=True)
    ctx = LOR(m if what != "coords" else mg.box_mesh(3, (4, 3, 3), 1, scramble=True))
    quad, coef = ("gauss2" if what == "gauss2" else "vertex"), None
    if what == "coef":
        coef = _coefs(m)
        ctx.set_coefficients(*coef)
    if what == "coords":
        ctx.update_coordinates(torch.from_numpy(np.ascontiguousarray(m.X)).cuda())
    assert ctx.fill_path(space) == (2 if what in ("gauss2", "coords") else (0 if space == "nd" else 1))
    q = ctx.query(space)
    out = ctx.assemble(space, 1.3, 0.7, quad)
    ctx.sync()
    compare_full(*(to_host(t) for t in out), oracle_lib.assemble(m, space, quad, 1.3, 0.7, coef=coef), 0,
                 q["n_local"], f"p=1 {space} {what}")
    ctx.close()


@pytest.mark.parametrize("space", ["nd", "rt"])
def test_rowpath_vector_sampled_large(torch_cuda, oracle_lib, space):
    """96^3 Kershaw elements: closed-form row lengths (ND 12..33, RT 6..11 on a hex lattice), 2000
    sampled rows against the oracle's row routine"""
    from paper_2210_12253_b200.lor import LOR
    n = 96
    m = mg.box_mesh(3, (n, n, n), 1, kershaw=0.3)
    ctx = LOR(m, spaces=(space,))
    assert ctx.fill_path(space) == 2
    q = ctx.query(space)
    assert q["n_local"] == (3 * n * (n + 1) ** 2 if space == "nd" else 3 * n * n * (n + 1))
    rp, col, val = ctx.assemble(space, 1.0, 1.0, "vertex")
    ctx.sync()
    rp, col, val = to_host(rp), to_host(col), to_host(val)
    d = np.diff(rp)
    assert (d.min(), d.max()) == ((12, 33) if space == "nd" else (6, 11))
    rng = np.random.default_rng(5)
    rows = np.unique(np.concatenate([rng.integers(0, q["n_local"], 2000), [0, q["n_local"] - 1]]))
    ref = oracle_lib.assemble_rows(m, rows, space, "vertex", 1.0, 1.0)
    compare_rows(rp, col, val, ref, 0, what=f"p=1 {space} 96^3 sampled")
    ctx.close()


def test_rowpath_vector_degenerate_reported(torch_cuda):
    from paper_2210_12253_b200.lor import LOR, LorError
    m = mg.box_mesh(3, (3, 3, 3), 1)
    X = m.X.copy()
    X[13, :, 0] = X[13, :, 7] + (X[13, :, 7] - X[13, :, 0])
    m.X = X
    ctx = LOR(m)
    assert ctx.fill_path("rt") == 2
    ctx.assemble("rt")
    with pytest.raises(LorError) as ei:
        ctx.sync()
    assert "degenerate-geometry(element=13" in str(ei.value)
