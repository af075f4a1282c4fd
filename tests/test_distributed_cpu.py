"""World-size-2 gloo tests (CPU) of the multi-GPU host logic: NCCL id
broadcast, consistent per-rank plans, slab ownership, identical seeded
inputs on every rank, max-over-ranks timing."""
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1410_6609_b200 import dist as D
        from paper_1410_6609_b200 import mg
        from paper_1410_6609_b200 import workloads as W

        def make_id():
            try:
                return mg.nccl_unique_id()
            except mg.MGError:
                return bytes(np.random.default_rng(5).integers(0, 256, 128, np.uint8))

        uid = D.share_nccl_id(rank, make_id)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        shape = (1024, 512, 512)
        dims, lnx, agg = mg.plan(shape, min_coarse=8, nranks=world, rank=rank,
                                 halo="nccl")
        plans = [None] * world
        dist.all_gather_object(plans, (dims, lnx, agg))
        lo, hi = D.slab_range(shape[0], world, rank)
        ranges = [None] * world
        dist.all_gather_object(ranges, (lo, hi))
        w = W.cfg4(P=world, n=64, seed=3)
        h = float(np.sum(w.centers) + np.sum(w.charges))
        hs = [None] * world
        dist.all_gather_object(hs, h)
        tmax = D.max_over_ranks(float(rank + 1))
        q.put((rank, ids, plans, ranges, hs, tmax, lnx[0]))
    finally:
        dist.destroy_process_group()


def test_two_rank_host_logic():
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    out.sort()
    for rank, ids, plans, ranges, hs, tmax, lnx0 in out:
        assert ids[0] == ids[1] and len(ids[0]) == 128
        assert plans[0] == plans[1]
        assert ranges == [(0, 512), (512, 1024)]
        assert hs[0] == hs[1]
        assert tmax == 2.0
        assert lnx0 == 512
    dims, lnx, agg = out[0][2][0]
    assert dims[-1] == (16, 8, 8) and agg == 4


def _halo_worker(rank, world, port, periodic, q):
    """Run the library's ghost-plane schedule (mg_halo_schedule, the exact
    sequence halo() posts in one NCCL group) with gloo point-to-point
    messages over slabs whose planes carry their global x index."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1410_6609_b200 import mg
        nxl, plane = 3, 5
        A = torch.full((nxl + 2, plane), -1.0, dtype=torch.float64)
        for il in range(nxl):
            A[il + 1] = rank * nxl + il          # global plane index
        idx = {mg.MG_PLANE_FIRST: 1, mg.MG_PLANE_LAST: nxl,
               mg.MG_GHOST_LO: 0, mg.MG_GHOST_HI: nxl + 1}
        reqs = []
        for op, peer, pl in mg.halo_schedule(world, rank, periodic):
            buf = A[idx[pl]]
            if op == mg.MG_OP_SEND:
                reqs.append(dist.isend(buf.clone(), peer))
            else:
                reqs.append(dist.irecv(buf, peer))
        for r in reqs:
            r.wait()
        q.put((rank, A[0, 0].item(), A[nxl + 1, 0].item()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,periodic", [(2, False), (2, True), (3, True),
                                           (3, False)])
def test_halo_schedule_exchanges_ghost_planes(world, periodic):
    """Ghost planes receive the neighbours' boundary planes; with a periodic
    x axis rank 0 and rank P-1 are neighbours, including P = 2
    where both neighbours are the same rank (messages match in order)."""
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_worker, args=(r, world, port, periodic, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nx, nxl = 3 * world, 3
    for rank, lo, hi in out:
        exp_lo = rank * nxl - 1
        exp_hi = (rank + 1) * nxl
        if periodic:
            exp_lo %= nx
            exp_hi %= nx
        else:
            exp_lo = -1.0 if rank == 0 else exp_lo          # untouched
            exp_hi = -1.0 if rank == world - 1 else exp_hi
        assert (lo, hi) == (exp_lo, exp_hi), (rank, lo, hi)
