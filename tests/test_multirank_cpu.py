"""Multi-rank host logic on CPU (world_size 2 and 3, gloo): every rank builds its own setup plan
(lor_plan_dry_run -- the same C++ code lor_setup runs, no GPU), the ranks exchange their plans
over torch.distributed/gloo and check that they agree with each other and with the oracle:
contiguous owned row ranges that tile [0, n_global), send/recv record counts that match pairwise,
row ranges equal to the oracle's rank-major numbering."""
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _worker(rank, world, port, shape, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_12253_b200 import meshgen as mg
        from paper_2210_12253_b200.lor import plan_dry_run
        m = mg.box_mesh(3, shape, p, jitter=True, scramble=True, nranks=world)
        info, send, recv = plan_dry_run(m, rank, world)
        t = torch.from_numpy(np.concatenate([info.ravel(), send.ravel(), recv.ravel()]))
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        if rank == 0:
            q.put([g.numpy() for g in gathered])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_plans_agree(world, oracle_lib):
    from paper_2210_12253_b200 import meshgen as mg
    shape, p = (2, 3, 2 * world), 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29500 + world * 7 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, shape, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    m = mg.box_mesh(3, shape, p, jitter=True, scramble=True, nranks=world)
    for s, space in enumerate(("h1", "nd", "rt")):
        infos = [r[:24].reshape(3, 8)[s] for r in res]
        send = np.stack([r[24:24 + 3 * world].reshape(3, world)[s] for r in res])
        recv = np.stack([r[24 + 3 * world:].reshape(3, world)[s] for r in res])
        n_global = infos[0][1]
        begins = [int(i[2]) for i in infos]
        sizes = [int(i[3]) for i in infos]
        assert all(i[1] == n_global for i in infos)
        assert begins[0] == 0 and all(begins[r] + sizes[r] == begins[r + 1] for r in range(world - 1))
        assert begins[-1] + sizes[-1] == n_global
        # pairwise: what r sends to q is what q expects from r
        np.testing.assert_array_equal(send, recv.T)
        assert (np.diag(send) == 0).all()
        # interior ranks both send (down) and receive (from above); last rank receives nothing
        assert send[1:, :].sum() > 0 and recv[-1].sum() == 0
        # oracle rank-major numbering gives the same row ranges
        n, _, off = oracle_lib.space_size(m, space)
        assert n == n_global
        np.testing.assert_array_equal(np.array(begins + [n_global]), off)


def _xworker(rank, world, port, shape, p, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2210_12253_b200 import meshgen as mg
        from paper_2210_12253_b200.lor import xframe_dry_run
        m = mg.box_mesh(3, shape, p, kershaw=0.3, nranks=world)
        info, send, recv = xframe_dry_run(m, rank, world)
        t = torch.from_numpy(np.concatenate([info, send, recv]))
        gathered = [torch.zeros_like(t) for _ in range(world)]
        dist.all_gather(gathered, t)
        if rank == 0:
            q.put([g.numpy() for g in gathered])
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_xframe_ghost_layers_agree(world):
    """Extended frame on several ranks: every rank keeps the single-pass path
    (regular neighbourhoods across slab interfaces), and the coordinate ghost exchange is pairwise
    consistent: what r sends q is what q receives from r; only slab neighbours exchange; a slab
    interface moves one element layer (nx * ny elements) each way."""
    nx, ny, nzr = 3, 4, 2
    shape, p = (nx, ny, nzr * world), 4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29700 + world * 11 + os.getpid() % 1000
    procs = [ctx.Process(target=_xworker, args=(r, world, port, shape, p, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = q.get(timeout=300)
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    info = np.stack([r[:4] for r in res])
    send = np.stack([r[4:4 + world] for r in res])
    recv = np.stack([r[4 + world:] for r in res])
    assert (info[:, 0] == 1).all()                          # single pass on every rank
    np.testing.assert_array_equal(send, recv.T)             # pairwise consistent
    assert (np.diag(send) == 0).all()
    for r in range(world):
        for s in range(world):
            expect = nx * ny if abs(r - s) == 1 else 0
            assert send[r, s] == expect and recv[r, s] == expect
        assert info[r, 1] == recv[r].sum()                  # ghost layer = what the peers send
