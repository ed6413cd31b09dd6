"""GPU checks of the boundary entry points added in round 2 and of input-domain edge cases:

* lor_dof_transpose (the element restriction's dof -> element "inverse offsets",
  PAPER.md l.412-415) against its definition applied to the oracle's pinned dof map: bit-exact,
  one rank and per rank of a slab split;
* meshes scaled far from unit size (coordinates x 1e-14 and x 1e12) on every fill path: the cell
  volumes leave the float range, which the extended-frame kernel's reciprocal must not depend on;
* det J <= 0 reported with the element that holds the degenerate cell.
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


def transpose_definition(om, row_begin, n_local, e0, e1):
    """entries of row g: sorted { (e - e0) * ndpe + l : e0 <= e < e1, om[e, l] == g }"""
    ndpe = om.shape[1]
    loc = om[e0:e1].reshape(-1).astype(np.int64)
    own = (loc >= row_begin) & (loc < row_begin + n_local)
    idx = np.flatnonzero(own)
    rows = loc[idx] - row_begin
    order = np.lexsort((idx, rows))
    off = np.zeros(n_local + 1, dtype=np.int64)
    np.add.at(off, rows + 1, 1)
    return np.cumsum(off), idx[order].astype(np.int32)


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
@pytest.mark.parametrize("p", [1, 3, 8])
def test_dof_transpose_one_rank(torch_cuda, oracle_lib, space, p):
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(3, (3, 2, 2) if p < 8 else (2, 2, 2), p, jitter=True, scramble=True)
    ctx = LOR(m)
    q = ctx.query(space)
    off, ent = ctx.dof_transpose(space)
    ctx.sync()
    om, _ = oracle_lib.dof_map(m, space)
    eo, ee = transpose_definition(om, 0, q["n_local"], 0, m.nel)
    assert ee.size == m.nel * om.shape[1]
    np.testing.assert_array_equal(to_host(off), eo)
    np.testing.assert_array_equal(to_host(ent), ee)
    ctx.close()


def test_dof_transpose_2d(torch_cuda, oracle_lib):
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(2, (4, 3), 5, jitter=True, scramble=True)
    ctx = LOR(m)
    q = ctx.query("h1")
    off, ent = ctx.dof_transpose("h1")
    ctx.sync()
    om, _ = oracle_lib.dof_map(m, "h1")
    eo, ee = transpose_definition(om, 0, q["n_local"], 0, m.nel)
    np.testing.assert_array_equal(to_host(off), eo)
    np.testing.assert_array_equal(to_host(ent), ee)


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
def test_dof_transpose_per_rank(torch_cuda, oracle_lib, space):
    from paper_2210_12253_b200.lor import LOR
    nranks = 3
    m = mg.box_mesh(3, (2, 2, 2 * nranks), 3, jitter=True, scramble=True, nranks=nranks)
    om, _ = oracle_lib.dof_map(m, space, nranks=nranks)
    for r in range(nranks):
        ctx = LOR(m, rank=r, nranks=nranks)
        q = ctx.query(space)
        off, ent = ctx.dof_transpose(space)
        ctx.sync()
        e0, e1 = int(m.elem_rank_begin[r]), int(m.elem_rank_begin[r + 1])
        eo, ee = transpose_definition(om, q["row_begin"], q["n_local"], e0, e1)
        np.testing.assert_array_equal(to_host(off), eo)
        np.testing.assert_array_equal(to_host(ent), ee)
        ctx.close()


def scaled(m, s):
    m.X = np.ascontiguousarray(m.X * s)
    m.vert = np.ascontiguousarray(m.vert * s)
    return m


@pytest.mark.parametrize("scale", [1e-14, 1e12])
@pytest.mark.parametrize("space,quad,p", [("h1", "vertex", 4), ("h1", "vertex", 6), ("h1", "gauss2", 3),
                                          ("nd", "vertex", 3), ("rt", "vertex", 3)])
def test_scaled_mesh(torch_cuda, oracle_lib, scale, space, quad, p):
    """cell volumes ~1e-48 / ~1e31: outside the float range the extended-frame reciprocal seed is
    built on (rcp.approx.f32); every path must still match the oracle entry by entry"""
    from paper_2210_12253_b200.lor import LOR
    m = scaled(mg.box_mesh(3, (3, 2, 2), p, jitter=True), scale)
    ctx = LOR(m)
    if space == "h1" and quad == "vertex":
        assert ctx.fill_path("h1") == 1
    q = ctx.query(space)
    rp, col, val = ctx.assemble(space, 1.3, 0.7, quad)
    ctx.sync()
    ref = oracle_lib.assemble(m, space, quad, 1.3, 0.7)
    compare_csr_arrays(to_host(rp), to_host(col), to_host(val), ref, 0, q["n_local"], f"{space} x{scale:g}")
    ctx.close()


@pytest.mark.parametrize("p", [2, 3])
@pytest.mark.parametrize("shuffle", [False, True])
def test_degenerate_cell_reported_from_any_box(torch_cuda, p, shuffle):
    """a conforming mesh whose element `bad` has an inverted interior: its first interior GLL point
    is moved beyond its corner 0 (no other element holds that point).  The neighbour CTAs of the
    extended-frame fill recompute the cells next to their shared faces, which include this point;
    whichever CTA finds det J <= 0 first, the error names the element the cell belongs to.  With
    shuffled numbering ownership falls on every side of an element."""
    from paper_2210_12253_b200.lor import LOR, LorError
    from tests.test_gpu_xframe import shuffled
    m = mg.box_mesh(3, (3, 3, 3), p)
    if shuffle:
        m = shuffled(m, seed=11)
    bad = 13
    P = p + 1
    X = m.X.copy()
    c0, c7, inner = 0, P ** 3 - 1, 1 + P + P * P
    X[bad, :, inner] = X[bad, :, c0] - (X[bad, :, c7] - X[bad, :, c0])
    m.X = X
    ctx = LOR(m)
    assert ctx.fill_path("h1") == 1
    ctx.assemble("h1")
    with pytest.raises(LorError) as ei:
        ctx.sync()
    assert f"degenerate-geometry(element={bad}," in str(ei.value)


@pytest.mark.parametrize("space,quad,p", [("h1", "vertex", 4), ("h1", "vertex", 7), ("h1", "gauss2", 3),
                                          ("nd", "vertex", 3), ("rt", "vertex", 3)])
def test_reassemble_after_mesh_motion(torch_cuda, oracle_lib, space, quad, p):
    """lor_reassemble_* (numeric-only re-assembly with pattern reuse): full
    assembly on mesh A, then the coordinates move to mesh B (same topology, lor_update_coordinates)
    and only the values are recomputed into the same buffers: equal to the oracle on B, and the
    pattern arrays are those of the full call."""
    from paper_2210_12253_b200.lor import LOR
    ma = mg.box_mesh(3, (3, 2, 2), p)
    mb = mg.box_mesh(3, (3, 2, 2), p, jitter=True)
    ctx = LOR(ma)
    q = ctx.query(space)
    out = ctx.assemble(space, 1.0, 1.0, quad)
    ctx.sync()
    rp0, col0 = to_host(out[0]).copy(), to_host(out[1]).copy()
    import torch
    ctx.update_coordinates(torch.from_numpy(np.ascontiguousarray(mb.X)).cuda())
    ctx.reassemble(space, 1.3, 0.7, quad, out=out)
    ctx.sync()
    rp, col, val = (to_host(t) for t in out)
    assert np.array_equal(rp, rp0) and np.array_equal(col, col0)
    ref = oracle_lib.assemble(mb, space, quad, 1.3, 0.7)
    compare_csr_arrays(rp, col, val, ref, 0, q["n_local"], f"reassemble {space} {quad} p={p}")
    ctx.close()
