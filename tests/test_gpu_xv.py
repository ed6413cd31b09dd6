"""GPU parity of the extended-frame ("owner computes") path of the vector spaces (lor_xv.cuh,
DESIGN.md section 4 "k_xv"): H(curl) Nedelec and H(div) Raviart-Thomas rows written complete by
their owning element, the neighbour cells recomputed in its frame, orientation signs of the box
dofs from the neighbours' restrictions.  On one rank RT and ND take this path by default at the
orders where it measured faster (ND p = 4-5, RT p != 5; LOR_XV=1 forces it at every order it fits,
LOR_XV=0 / LOR_XV_ND=0 keep the element + merge passes); ND at p >= 6 falls back to them when the
frame does not fit.  Both
are compared with the oracle element by element (bit-exact pattern, P-10b values), on meshes whose
numbering is shuffled (ownership on every side of an element) and orientation-scrambled, for every
p the instantiations cover."""
import numpy as np
import pytest

from paper_2210_12253_b200 import meshgen as mg
from tests.parity import compare_csr_arrays, to_host
from tests.test_gpu_xframe import shuffled

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def run(O, m, space, expect_path, what):
    from paper_2210_12253_b200.lor import LOR
    ctx = LOR(m)  # LOR_XV=1 (the tests below): the frame at every order it supports
    if expect_path is not None:
        assert ctx.fill_path(space) == expect_path, what
    q = ctx.query(space)
    rp, col, val = ctx.assemble(space, 1.3, 0.7, "vertex")
    ctx.sync()
    ref = O.assemble(m, space, "vertex", 1.3, 0.7)
    compare_csr_arrays(to_host(rp), to_host(col), to_host(val), ref, 0, q["n_local"], what)
    # numeric-only re-assembly on the same path gives the same arrays
    rp2, col2, val2 = (to_host(t).copy() for t in (rp, col, val))
    ctx.reassemble(space, 1.3, 0.7, "vertex", out=(rp, col, val))
    ctx.sync()
    assert np.array_equal(to_host(val), val2) and np.array_equal(to_host(col), col2)
    ctx.close()


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("kind", ["scrambled", "shuffled"])
def test_rt_xframe(torch_cuda, oracle_lib, monkeypatch, p, kind):
    monkeypatch.setenv("LOR_XV", "1")
    monkeypatch.setenv("LOR_ROWPATH", "0")  # p = 1: the per-row path otherwise (test_gpu_rowpath.py)
    shape = (3, 3, 2) if p <= 4 else (3, 2, 2)
    m = mg.box_mesh(3, shape, p, jitter=True, scramble=(kind == "scrambled"))
    if kind == "shuffled":
        m = shuffled(m, seed=p)
    run(oracle_lib, m, "rt", 1, f"rt {kind} p={p}")


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("kind", ["scrambled", "shuffled", "kershaw"])
def test_nd_xframe(torch_cuda, oracle_lib, monkeypatch, p, kind):
    monkeypatch.setenv("LOR_XV", "1")
    monkeypatch.setenv("LOR_ROWPATH", "0")
    if kind == "kershaw":
        m = mg.box_mesh(3, (6, 2, 2), p, kershaw=0.3)
    else:
        m = mg.box_mesh(3, (3, 3, 2), p, jitter=True, scramble=(kind == "scrambled"))
        if kind == "shuffled":
            m = shuffled(m, seed=10 + p)
    run(oracle_lib, m, "nd", 1 if p <= 5 else None, f"nd {kind} p={p}")


@pytest.mark.parametrize("space", ["rt", "nd"])
def test_xframe_off_is_general_path(torch_cuda, oracle_lib, monkeypatch, space):
    """LOR_XV=0 keeps the element + merge passes (fill path 0); same oracle parity."""
    monkeypatch.setenv("LOR_XV", "0")
    m = mg.box_mesh(3, (3, 2, 2), 3, jitter=True, scramble=True)
    run(oracle_lib, m, space, 0, f"{space} general path")


@pytest.mark.parametrize("space,p,expect", [("nd", 3, 0), ("nd", 4, 1), ("nd", 5, 1), ("nd", 6, 0),
                                            ("rt", 3, 1), ("rt", 5, 0), ("rt", 6, 1)])
def test_default_routing(torch_cuda, oracle_lib, monkeypatch, space, p, expect):
    """default one-rank routing follows the measured table (xv_preferred in lor_capi.cu); same
    oracle parity on either path"""
    monkeypatch.delenv("LOR_XV", raising=False)
    monkeypatch.delenv("LOR_XV_ND", raising=False)
    m = mg.box_mesh(3, (3, 2, 2), p, jitter=True, scramble=True)
    run(oracle_lib, m, space, expect, f"{space} p={p} default routing")
