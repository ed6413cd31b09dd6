"""The unstructured ("legacy") comparator through the C ABI:
the same H1 matrix as the oracle (pattern bit-exact, values within the P-10b rule) on small meshes at
every p, and the same pattern as the macro-element path at full C2 size with values equal to
rounding."""
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


@pytest.mark.parametrize("p", [1, 2, 3, 4, 5, 6, 7, 8])
def test_legacy_parity(torch_cuda, oracle_lib, p):
    from paper_2210_12253_b200.lor import LOR
    shape = (3, 2, 2) if p <= 4 else (2, 2, 2)
    m = mg.box_mesh(3, shape, p, jitter=True, scramble=True)
    ctx = LOR(m)
    ctx.legacy_setup()
    out = ctx.legacy_assemble(1.3, 0.7)
    ctx.sync()
    q = ctx.query("h1")
    compare_full(*(to_host(t) for t in out), oracle_lib.assemble(m, "h1", "vertex", 1.3, 0.7), 0, q["n_local"],
                 f"legacy p={p}")


def test_legacy_vs_macro_c2(torch_cuda):
    from paper_2210_12253_b200.lor import LOR
    m, _ = mg.config_mesh("C2-J")
    ctx = LOR(m)
    A = [to_host(t) for t in ctx.assemble("h1", 1.0, 1.0, "vertex")]
    ctx.sync()
    ctx.legacy_setup()
    L = [to_host(t) for t in ctx.legacy_assemble(1.0, 1.0)]
    ctx.sync()
    assert np.array_equal(A[0], L[0]) and np.array_equal(A[1], L[1])
    rows = np.repeat(np.arange(A[0].shape[0] - 1), np.diff(A[0]))
    rmax = np.maximum.reduceat(np.abs(A[2]), A[0][:-1])
    assert np.all(np.abs(A[2] - L[2]) <= np.maximum(1e-12 * np.abs(A[2]), 64 * 2.0 ** -53 * rmax[rows]))
