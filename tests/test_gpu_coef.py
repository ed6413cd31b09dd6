"""GPU parity of variable coefficients (reading P-28) through the C
ABI (lor_set_coefficients): alpha a(x), beta b(x) with a, b given as E-vectors at the LOR vertices,
against the oracle with the same E-vectors -- pattern bit-exact, values within the P-10b rule; H1 /
ND / RT, both rules, p = 1..8, 2D, several emulated ranks, numeric-only re-assembly."""
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


def _coefs(m):
    x = [m.X[:, d, :] for d in range(m.dim)]
    z = x[2] if m.dim == 3 else 0.0
    a = 1.0 + 0.5 * np.sin(3.0 * x[0]) * np.cos(2.0 * x[1]) + z * z
    b = 2.0 + np.cos(x[0] + x[1] + z)
    return np.ascontiguousarray(a), np.ascontiguousarray(b)


def _run(O, m, space, quad, p_what, nranks=1):
    from paper_2210_12253_b200.lor import LOR
    a, b = _coefs(m)
    ref = O.assemble(m, space, quad, 1.3, 0.7, nranks=nranks, coef=(a, b))
    ctxs = [LOR(m, rank=r, nranks=nranks) for r in range(nranks)]
    outs = []
    for r, c in enumerate(ctxs):
        e0, e1 = int(m.elem_rank_begin[r]), int(m.elem_rank_begin[r + 1])
        fp0 = c.fill_path(space)
        c.set_coefficients(a[e0:e1], b[e0:e1])
        # the extended frames are kept on one rank (coefficient boxes beside the coordinates); the
        # p = 1 per-row path (fill path 2) has no coefficients and hands over to the frame
        assert c.fill_path(space) == ((1 if fp0 == 2 else fp0) if (nranks == 1 and space != "nd") else 0)
        outs.append(c.assemble(space, 1.3, 0.7, quad))
        c.sync()
    if nranks > 1:
        for r, c in enumerate(ctxs):
            for q, src in enumerate(ctxs):
                if q != r:
                    c.exchange_copy_from(src, space)
            c.assemble_finish(space, outs[r])
            c.sync()
    for r, c in enumerate(ctxs):
        q = c.query(space)
        compare_full(*(to_host(t) for t in outs[r]), ref, q["row_begin"], q["n_local"], f"{p_what} rank {r}")
    return ctxs, outs, ref


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
def test_coef_3d(torch_cuda, oracle_lib, space, p, quad):
    shape = (3, 2, 2) if p <= 4 else (2, 2, 2)
    m = mg.box_mesh(3, shape, p, jitter=True, scramble=True)
    ctxs, _, _ = _run(oracle_lib, m, space, quad, f"coef {space} p={p} {quad}")
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("quad", ["vertex", "gauss2"])
def test_coef_2d(torch_cuda, oracle_lib, quad):
    m = mg.box_mesh(2, (3, 4), 3, jitter=True, scramble=True)
    _run(oracle_lib, m, "h1", quad, f"coef 2d {quad}")


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
def test_coef_multirank(torch_cuda, oracle_lib, space):
    m = mg.box_mesh(3, (2, 2, 6), 3, kershaw=0.3, nranks=3)
    _run(oracle_lib, m, space, "vertex", f"coef {space} 3 ranks", nranks=3)


@pytest.mark.parametrize("space", ["h1", "rt"])
def test_coef_reassemble_and_reset(torch_cuda, oracle_lib, space):
    """pattern of a constant-coefficient (extended-frame) call reused for a variable-coefficient
    re-assembly; clearing the coefficients restores the extended-frame path and its values"""
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(3, (3, 2, 2), 4, jitter=True, scramble=True)
    ctx = LOR(m)
    assert ctx.fill_path(space) == 1
    out = ctx.assemble(space, 1.3, 0.7, "vertex")
    ctx.sync()
    a, b = _coefs(m)
    ctx.set_coefficients(a, b)
    ctx.reassemble(space, 1.3, 0.7, "vertex", out=out)
    ctx.sync()
    q = ctx.query(space)
    compare_full(*(to_host(t) for t in out), oracle_lib.assemble(m, space, "vertex", 1.3, 0.7, coef=(a, b)), 0,
                 q["n_local"], f"{space} coef reassembly")
    ctx.set_coefficients(None, None)
    assert ctx.fill_path(space) == 1
    out = ctx.assemble(space, 1.3, 0.7, "vertex")
    ctx.sync()
    compare_full(*(to_host(t) for t in out), oracle_lib.assemble(m, space, "vertex", 1.3, 0.7), 0, q["n_local"],
                 f"{space} constant again")


@pytest.mark.parametrize("space", ["h1", "rt"])
@pytest.mark.parametrize("nranks", [2, 3])
def test_coef_multirank_extended_frame(torch_cuda, oracle_lib, space, nranks):
    """global coefficient E-vectors: every rank keeps its ghost layer's coefficients and the
    extended-frame single pass (no partial-row exchange), rows equal to the oracle's"""
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(3, (2, 3, 2 * nranks), 3, kershaw=0.3, scramble=True, nranks=nranks)
    a, b = _coefs(m)
    ref = oracle_lib.assemble(m, space, "vertex", 1.3, 0.7, nranks=nranks, coef=(a, b))
    for r in range(nranks):
        c = LOR(m, rank=r, nranks=nranks)
        c.set_coefficients_global(a, b)
        assert c.fill_path(space) == 1
        q = c.query(space)
        out = c.assemble(space, 1.3, 0.7, "vertex")
        c.sync()
        compare_full(*(to_host(t) for t in out), ref, q["row_begin"], q["n_local"], f"{space} coef rank {r}/{nranks}")
        c.close()
