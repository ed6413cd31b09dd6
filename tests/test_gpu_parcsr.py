"""GPU parity of the steps after the local assembly (SURVEY 8(f) NEXT-1 and the coordinate vectors
of NEXT-2) through the C ABI, against oracle/bc.py: the ParCSR split (bit-exact: row pointers,
local / offd column ids, col_map_offd, values copied), the boundary dofs (bit-exact), the A4
elimination (bit-exact values: copies, 0.0 and 1.0) on one rank and on emulated ranks with the
manual marker exchange, and the LOR vertex coordinate vectors (bit-exact copies)."""
import numpy as np
import pytest

from paper_2210_12253_b200 import meshgen as mg
from tests.parity import to_host

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    return torch


def _assemble(ctx, op):
    if op in ("grad", "curl"):
        A = ctx.discrete(op)
    else:
        A = ctx.assemble(op, 1.3, 0.7, "vertex")
    ctx.sync()
    return A


def _assemble_ranks(ctxs, space):
    """every rank's rows; the general (ND) path completes its interface rows after the manual
    exchange of partial rows (lor_exchange_copy + lor_assemble_finish, as the NCCL path)."""
    outs = [c.assemble(space, 1.3, 0.7, "vertex") for c in ctxs]
    for c in ctxs:
        c.sync()
    if len(ctxs) > 1:
        for r, c in enumerate(ctxs):
            for q, src in enumerate(ctxs):
                if q != r:
                    c.exchange_copy_from(src, space)
            c.assemble_finish(space, outs[r])
            c.sync()
    return outs


def _ref(O, m, op, nranks):
    if op in ("grad", "curl"):
        return O.discrete(m, op, nranks=nranks)
    return O.assemble(m, op, "vertex", 1.3, 0.7, nranks=nranks)


def _col_space(op):
    return {"grad": "h1", "curl": "nd"}.get(op, op)


def _check_split(P, R, what):
    for k in ("diag_row_ptr", "offd_row_ptr"):
        assert np.array_equal(to_host(P[k]), R[k]), f"{what}: {k}"
    nd, no, nc = P["sizes"]
    assert (nd, no, nc) == (len(R["diag_col"]), len(R["offd_col"]), len(R["col_map_offd"])), what
    assert np.array_equal(to_host(P["diag_col"])[:nd], R["diag_col"]), f"{what}: diag_col"
    assert np.array_equal(to_host(P["offd_col"])[:no], R["offd_col"]), f"{what}: offd_col"
    assert np.array_equal(to_host(P["col_map_offd"])[:nc], R["col_map_offd"]), f"{what}: col_map_offd"
    return nd, no


def _check_vals(P, R, nd, no, what):
    # bit-exact: the split copies values, elimination writes 0.0 / 1.0 (+0.0 == -0.0)
    assert np.array_equal(to_host(P["diag_val"])[:nd], R["diag_val"]), f"{what}: diag_val"
    assert np.array_equal(to_host(P["offd_val"])[:no], R["offd_val"]), f"{what}: offd_val"


@pytest.mark.parametrize("op", ["h1", "nd", "rt", "grad", "curl"])
@pytest.mark.parametrize("nranks", [1, 2, 3])
def test_parcsr_split(torch_cuda, oracle_lib, op, nranks):
    from oracle import bc
    from paper_2210_12253_b200.lor import LOR
    p = 2
    m = mg.box_mesh(3, (2, 2, 2 * nranks), p, jitter=True, scramble=True, nranks=nranks)
    ref = _ref(oracle_lib, m, op, nranks)
    _, _, coff = oracle_lib.space_size(m, _col_space(op), nranks)
    ctxs = [LOR(m, rank=r, nranks=nranks) for r in range(nranks)]
    As = [_assemble(c, op) for c in ctxs] if op in ("grad", "curl") else _assemble_ranks(ctxs, op)
    for r in range(nranks):
        ctx, A = ctxs[r], As[r]
        q = ctx.query(op) if op not in ("grad", "curl") else ctx.query({"grad": "nd", "curl": "rt"}[op])
        P = ctx.parcsr(op, A)
        ctx.sync()
        R = bc.parcsr_split(ref, q["row_begin"], q["n_local"], coff[r], coff[r + 1], square=op in ("h1", "nd", "rt"))
        nd, no = _check_split(P, R, f"{op} rank {r}/{nranks}")
        if op in ("grad", "curl"):
            _check_vals(P, R, nd, no, f"{op} rank {r}/{nranks}")
        else:  # values: the split copies the (parity-tested) assembled values; compare to the copy
            A_h = [to_host(t) for t in A]
            dv, ov = to_host(P["diag_val"])[:nd], to_host(P["offd_val"])[:no]
            assert np.sort(np.concatenate([dv, ov])).tolist() == np.sort(A_h[2][:nd + no]).tolist()
        ctx.close()


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
@pytest.mark.parametrize("nranks", [1, 3])
def test_boundary_dofs(torch_cuda, oracle_lib, space, nranks):
    from oracle import bc
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(3, (2, 3, 2 * nranks), 3, jitter=True, scramble=True, nranks=nranks)
    ess = bc.boundary_dofs(m, space, nranks)
    for r in range(nranks):
        ctx = LOR(m, rank=r, nranks=nranks)
        q = ctx.query(space)
        mine = ess[(ess >= q["row_begin"]) & (ess < q["row_begin"] + q["n_local"])] - q["row_begin"]
        assert np.array_equal(to_host(ctx.boundary_dofs(space)).astype(np.int64), mine), f"{space} rank {r}"
        ctx.close()


def test_boundary_dofs_2d(torch_cuda, oracle_lib):
    from oracle import bc
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(2, (3, 4), 3, jitter=True, scramble=True)
    ctx = LOR(m)
    assert np.array_equal(to_host(ctx.boundary_dofs("h1")).astype(np.int64), bc.boundary_dofs(m, "h1"))


@pytest.mark.parametrize("space", ["h1", "nd", "rt"])
@pytest.mark.parametrize("nranks,p", [(1, 1), (1, 3), (2, 2), (3, 2)])
def test_eliminate_bc(torch_cuda, oracle_lib, space, nranks, p):
    """A4 on the ParCSR of every rank (several ranks: manual marker exchange, the same kernels and
    buffers as the NCCL path) == oracle eliminate of the global matrix, split per rank."""
    from oracle import bc
    from paper_2210_12253_b200.lor import LOR
    m = mg.box_mesh(3, (2, 2, 2 * nranks), p, jitter=True, scramble=True, nranks=nranks)
    ref = oracle_lib.assemble(m, space, "vertex", 1.3, 0.7, nranks=nranks)
    ess = bc.boundary_dofs(m, space, nranks)
    # plus a few interior dofs (any essential set is allowed)
    rng = np.random.default_rng(7)
    ess = np.union1d(ess, rng.choice(ref.n_cols, size=max(1, ref.n_cols // 50), replace=False))
    refE = bc.eliminate(ref, ess)
    _, _, off = oracle_lib.space_size(m, space, nranks)
    ctxs = [LOR(m, rank=r, nranks=nranks) for r in range(nranks)]
    As = _assemble_ranks(ctxs, space)
    Ps = [c.parcsr(space, A) for c, A in zip(ctxs, As)]
    if nranks > 1:  # the marker-exchange plan is symmetric
        counts = [c.parcsr_exchange_counts(space) for c in ctxs]
        for r in range(nranks):
            for q in range(nranks):
                assert counts[r][0][q] == counts[q][1][r]
    import torch
    for r, c in enumerate(ctxs):
        mine = ess[(ess >= off[r]) & (ess < off[r + 1])] - off[r]
        et = torch.tensor(np.concatenate([mine, mine[:3]]).astype(np.int32), device="cuda")  # duplicates allowed
        c.eliminate_bc(space, et, Ps[r])
        c.sync()
    for r, c in enumerate(ctxs):
        for q, src in enumerate(ctxs):
            if q != r:
                c.bc_exchange_copy_from(src, space)
        c.eliminate_bc_finish(space, Ps[r])
        c.sync()
    for r, c in enumerate(ctxs):
        R = bc.parcsr_split(refE, off[r], off[r + 1] - off[r], off[r], off[r + 1], square=True)
        nd, no = _check_split(Ps[r], R, f"{space} elim rank {r}/{nranks}")
        # values: the GPU and oracle assemblies differ by rounding (P-10b); the eliminated entries
        # (essential row or column) must be exactly R's 0.0 / 1.0, the others R's values to 1e-12
        dv, ov = to_host(Ps[r]["diag_val"])[:nd], to_host(Ps[r]["offd_val"])[:no]
        mark = np.zeros(ref.n_cols, dtype=bool)
        mark[ess] = True
        n_r = off[r + 1] - off[r]
        rows_d = off[r] + np.repeat(np.arange(n_r), np.diff(R["diag_row_ptr"]))
        rows_o = off[r] + np.repeat(np.arange(n_r), np.diff(R["offd_row_ptr"]))
        kd = mark[rows_d] | mark[off[r] + R["diag_col"]]
        ko = mark[rows_o] | mark[R["col_map_offd"][R["offd_col"]]] if no else np.zeros(0, dtype=bool)
        assert np.array_equal(dv[kd], R["diag_val"][kd]), f"{space} rank {r}: eliminated diag entries"
        assert np.array_equal(ov[ko], R["offd_val"][ko]), f"{space} rank {r}: eliminated offd entries"
        scale = 64 * 2.0 ** -53 * np.abs(ref.val).max()
        assert np.all(np.abs(dv[~kd] - R["diag_val"][~kd]) <= np.maximum(1e-12 * np.abs(R["diag_val"][~kd]), scale))
        assert np.all(np.abs(ov[~ko] - R["offd_val"][~ko]) <= np.maximum(1e-12 * np.abs(R["offd_val"][~ko]), scale))
        # the eliminated rows are unit rows, bit-exact
        for j in (ess[(ess >= off[r]) & (ess < off[r + 1])] - off[r])[:50]:
            s, e = R["diag_row_ptr"][j], R["diag_row_ptr"][j + 1]
            assert dv[s] == 1.0 and not dv[s + 1:e].any()
            s, e = R["offd_row_ptr"][j], R["offd_row_ptr"][j + 1]
            assert not ov[s:e].any()
    for c in ctxs:
        c.close()


@pytest.mark.parametrize("dim,p,nranks", [(2, 3, 1), (3, 1, 1), (3, 4, 1), (3, 2, 3), (3, 8, 1)])
def test_coordinates(torch_cuda, oracle_lib, dim, p, nranks):
    from oracle import bc
    from paper_2210_12253_b200.lor import LOR
    shape = (3, 2) if dim == 2 else ((2, 2, 2 * nranks) if p < 8 else (2, 2, 2))
    kw = dict(jitter=True) if dim == 2 else dict(kershaw=0.3) if nranks == 1 else dict(jitter=True)
    m = mg.box_mesh(dim, shape, p, scramble=True, nranks=nranks, **kw)
    ref = bc.coordinates(m, nranks)
    for r in range(nranks):
        ctx = LOR(m, rank=r, nranks=nranks)
        q = ctx.query("h1")
        xyz = to_host(ctx.coordinates())
        ctx.sync()
        assert np.array_equal(xyz, ref[:, q["row_begin"]:q["row_begin"] + q["n_local"]]), f"coords rank {r}"
        ctx.close()


@pytest.mark.parametrize("cfg", ["C2", "C4", "C5"])
def test_parcsr_eliminate_fullsize(torch_cuda, cfg):
    """C2 / C4 / C5 at full size: split + A4 on the full matrix -- properties that hold at any size:
    the number of boundary dofs (closed form of the LOR surface lattice), row pointers, diagonal
    first, unit rows of the boundary dofs, no entry of a boundary column left, every other value
    equal to the assembled one"""
    import torch
    from paper_2210_12253_b200.lor import LOR
    m, form = mg.config_mesh(cfg)
    sp = form["space"]
    ctx = LOR(m)
    A = ctx.assemble(sp, 1.0, 1.0, "vertex")
    ctx.sync()
    P = ctx.parcsr(sp, A)
    ess = ctx.boundary_dofs(sp)
    N = 32 * 4
    closed = {"h1": (N + 1) ** 3 - (N - 1) ** 3, "nd": 3 * N * ((N + 1) ** 2 - (N - 1) ** 2), "rt": 6 * N * N}[sp]
    assert ess.numel() == closed
    ctx.sync()
    assert P["sizes"][1] == 0 and P["sizes"][2] == 0
    assert torch.equal(P["diag_row_ptr"], A[0])
    ctx.eliminate_bc(sp, ess, P)
    ctx.sync()
    rp = P["diag_row_ptr"]
    n = rp.numel() - 1
    col, val = P["diag_col"], P["diag_val"]
    first = rp[:-1]
    assert torch.equal(col[first].long(), torch.arange(n, device="cuda"))
    mark = torch.zeros(n, dtype=torch.bool, device="cuda")
    mark[ess.long()] = True
    rows = torch.repeat_interleave(torch.arange(n, device="cuda"), rp[1:] - rp[:-1])
    killed = mark[rows] | mark[col.long()]
    diag = col.long() == rows
    assert torch.all(val[killed & diag] == 1.0) and torch.all(val[killed & ~diag] == 0.0)
    # untouched entries: the assembled value of the same (row, col)
    a_rows = torch.repeat_interleave(torch.arange(n, device="cuda"), A[0][1:] - A[0][:-1])
    key_a = a_rows * n + A[1].long()
    key_p = rows * n + col.long()
    order = torch.argsort(key_p)
    assert torch.equal(key_p[order], key_a)
    assert torch.equal(val[order][~killed[order]], A[2][~killed[order]])
