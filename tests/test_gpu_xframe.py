"""GPU parity of the extended-frame H1 fill path (lor_xframe.h, DESIGN.md §4 k_xh1) and of the
fallback decision: regular-neighbourhood meshes take the single-pass path, irregular ones (a
re-entrant edge of valence 3) and LOR_XFRAME=0 take the element + merge passes; both match the
oracle element by element (bit-exact pattern, P-10 values)."""
import os

import numpy as np
import pytest

from paper_2210_12253_b200 import meshgen as mg
from tests.parity import compare_full, compare_rows, to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def shuffled(m, seed=5):
    """same geometry, element and vertex ids permuted: ownership (minimal element) lands on every
    side of an element, so cell boxes reach -1 and p on the same axis"""
    rng = np.random.default_rng(seed)
    pe = rng.permutation(m.nel)
    pv = rng.permutation(m.nv)
    inv = np.empty_like(pv)
    inv[pv] = np.arange(m.nv)
    vert = m.vert[pv]
    elem = inv[m.elem[pe]]
    return mg.Mesh(dim=m.dim, p=m.p, vert=np.ascontiguousarray(vert), elem=np.ascontiguousarray(elem),
                   X=np.ascontiguousarray(m.X[pe]), shape=m.shape,
                   elem_rank_begin=np.array([0, m.nel], dtype=np.int64), name=m.name + "-shuffled")


def l_shaped(m):
    """drop the column of elements at (ix, iy) = (nx-1, ny-1): the edge along z at the re-entrant
    corner has valence 3, so the neighbourhood is not a 3x3x3 block"""
    nx, ny, nz = m.shape
    keep = [e for e in range(m.nel) if not (e % nx == nx - 1 and (e // nx) % ny == ny - 1)]
    keep = np.array(keep)
    elem = m.elem[keep]
    used = np.unique(elem)
    remap = -np.ones(m.nv, dtype=np.int64)
    remap[used] = np.arange(used.size)
    return mg.Mesh(dim=3, p=m.p, vert=np.ascontiguousarray(m.vert[used]), elem=np.ascontiguousarray(remap[elem]),
                   X=np.ascontiguousarray(m.X[keep]), shape=m.shape,
                   elem_rank_begin=np.array([0, keep.size], dtype=np.int64), name="L")


def run(O, m, expect_path, alpha=1.3, beta=0.7, what=""):
    from paper_2210_12253_b200.lor import LOR
    ctx = LOR(m)
    assert ctx.fill_path("h1") == expect_path, what
    q = ctx.query("h1")
    rp, col, val = ctx.assemble("h1", alpha, beta, "vertex")
    ctx.sync()
    ref = O.assemble(m, "h1", "vertex", alpha, beta)
    assert q["nnz"] == ref.nnz
    compare_full(to_host(rp), to_host(col), to_host(val), ref, 0, q["n_local"], what)
    ctx.close()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 8])
@pytest.mark.parametrize("kind", ["cartesian", "jitscr", "kershaw", "shuffled"])
def test_xframe_parity(torch_cuda, oracle_lib, monkeypatch, kind, p):
    monkeypatch.setenv("LOR_ROWPATH", "0")  # p = 1 takes the per-row path by default (test_gpu_rowpath.py)
    shape = (3, 3, 2) if p <= 4 else (2, 2, 2)
    if kind == "cartesian":
        m = mg.box_mesh(3, shape, p)
    elif kind == "jitscr":
        m = mg.box_mesh(3, shape, p, jitter=True, scramble=True)
    elif kind == "kershaw":
        m = mg.box_mesh(3, (6, 2, 2) if p <= 4 else (6, 2, 1), p, kershaw=0.3)
    else:
        m = shuffled(mg.box_mesh(3, shape, p, jitter=True, scramble=True))
    run(oracle_lib, m, 1, what=f"xframe {kind} p={p}")


@pytest.mark.parametrize("p", [1, 2, 4])
def test_irregular_mesh_uses_general_path(torch_cuda, oracle_lib, p):
    m = l_shaped(mg.box_mesh(3, (3, 3, 2), p, jitter=True, scramble=True))
    run(oracle_lib, m, 2 if p == 1 else 0, what=f"L-shaped p={p}")  # p = 1: the per-row path needs no frame


def test_forced_general_path(torch_cuda, oracle_lib, monkeypatch):
    monkeypatch.setenv("LOR_XFRAME", "0")
    m = mg.box_mesh(3, (3, 2, 2), 3, jitter=True, scramble=True)
    run(oracle_lib, m, 0, what="LOR_XFRAME=0")


def test_xframe_degenerate_geometry_reported(torch_cuda):
    from paper_2210_12253_b200.lor import LOR, LorError
    m = mg.box_mesh(3, (2, 2, 2), 2)
    X = m.X.copy()
    X[5, 1, :] = X[5, 1, ::-1].copy()
    m.X = X
    ctx = LOR(m)
    assert ctx.fill_path("h1") == 1
    ctx.assemble("h1")
    with pytest.raises(LorError) as ei:
        ctx.sync()
    assert "degenerate-geometry(element=5" in str(ei.value)


def test_full_size_c3_row_sampled(torch_cuda, oracle_lib):
    """BASELINE configs[2] at one GPU (C3: 24^3 Kershaw hexes, p=8) in the launch configuration
    bench.py times: pattern closed form for every row, sampled rows vs the oracle row routine."""
    from paper_2210_12253_b200.lor import LOR
    m, form = mg.config_mesh("C3")
    ctx = LOR(m)
    assert ctx.fill_path("h1") == 1
    q = ctx.query("h1")
    N = 24 * 8
    assert q["n_local"] == (N + 1) ** 3 and q["nnz"] == (3 * N + 1) ** 3
    rp, col, val = ctx.assemble("h1", form["alpha"], form["beta"], form["quad"])
    ctx.sync()
    rp, col, val = to_host(rp), to_host(col), to_host(val)
    rng = np.random.default_rng(3)
    rows = np.unique(np.concatenate([rng.integers(0, q["n_local"], 2000), [0, q["n_local"] - 1]]))
    ref = oracle_lib.assemble_rows(m, rows, "h1", "vertex", form["alpha"], form["beta"])
    compare_rows(rp, col, val, ref, 0, what="C3 sampled")
    d = np.diff(rp)
    assert d.min() >= 8 and d.max() == 27
