"""NCCL path on >= 2 GPUs (skipped with fewer): one process per GPU, ncclUniqueId broadcast over
torch.distributed.  Each rank's owned rows against the oracle's rank-major matrix:
  * H1, ND and RT: single-pass extended frame with the ghost layer (no partial-row exchange);
  * after lor_update_coordinates with new (jittered) coordinates, whose ghost layer is refreshed from
    the peers over NCCL, the re-assembly matches the oracle on the moved mesh;
  * ParCSR split + A4 elimination with the boundary markers exchanged over NCCL on the side stream:
    structure bit-exact against oracle/bc.py, eliminated entries exactly 0 / 1."""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    errs = []
    try:
        from oracle import oracle as O
        from paper_2210_12253_b200 import meshgen as mg
        from paper_2210_12253_b200.lor import LOR, nccl_unique_id
        from tests.parity import compare_csr_arrays
        obj = [nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        ma = mg.box_mesh(3, (3, 3, 2 * world), 4, kershaw=0.3, nranks=world)
        mb = mg.box_mesh(3, (3, 3, 2 * world), 4, jitter=True, nranks=world)
        for space in ("h1", "nd", "rt"):
            ctx = LOR(ma, rank=rank, nranks=world, nccl_id=obj[0], device=rank)
            qq = ctx.query(space)
            out = ctx.assemble(space, 1.3, 0.7, "vertex")
            ctx.sync()
            ref = O.assemble(ma, space, "vertex", 1.3, 0.7)
            try:
                compare_csr_arrays(*(t.cpu().numpy() for t in out), ref, qq["row_begin"], qq["n_local"],
                                   f"{space} rank {rank}")
            except AssertionError as e:
                errs.append(str(e))
            e0, e1 = int(mb.elem_rank_begin[rank]), int(mb.elem_rank_begin[rank + 1])
            ctx.update_coordinates(torch.from_numpy(np.ascontiguousarray(mb.X[e0:e1])).cuda())
            ctx.reassemble(space, 1.3, 0.7, "vertex", out=out)
            ctx.sync()
            refb = O.assemble(mb, space, "vertex", 1.3, 0.7)
            try:
                compare_csr_arrays(*(t.cpu().numpy() for t in out), refb, qq["row_begin"], qq["n_local"],
                                   f"{space} moved rank {rank}")
            except AssertionError as e:
                errs.append(str(e))
            # A4 over NCCL: the boundary markers of the peers zero this rank's offd columns
            from oracle import bc
            P = ctx.parcsr(space, out)
            ess = ctx.boundary_dofs(space)
            ctx.eliminate_bc(space, ess, P)
            ctx.sync()
            essg = bc.boundary_dofs(mb, space, world)
            R = bc.parcsr_split(bc.eliminate(refb, essg), qq["row_begin"], qq["n_local"], qq["row_begin"],
                                qq["row_begin"] + qq["n_local"])
            for k in ("diag_row_ptr", "diag_col", "offd_row_ptr", "offd_col", "col_map_offd"):
                n = len(R[k])
                if not np.array_equal(P[k].cpu().numpy()[:n], R[k]):
                    errs.append(f"{space} rank {rank}: parcsr {k}")
            ov = P["offd_val"].cpu().numpy()[:len(R["offd_val"])]
            zero = R["offd_val"] == 0.0
            if not np.array_equal(ov[zero], R["offd_val"][zero]):
                errs.append(f"{space} rank {rank}: eliminated offd columns")
            ctx.close()
    except Exception as e:  # noqa: BLE001
        errs.append(repr(e))
    finally:
        dist.destroy_process_group()
    q.put((rank, errs))


def test_nccl_two_gpus():
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
        pytest.skip("needs >= 2 GPUs")
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = 29900 + os.getpid() % 1000
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for rank, errs in res:
        assert not errs, f"rank {rank}: {errs}"
