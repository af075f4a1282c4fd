"""The NCCL data plane on real GPUs (needs >= 2 visible devices; skipped on
the single-B200 boxes of this pool, where tests/test_gpu_multislab.py runs
the same layout through the EMULATE backend).

Two or four processes, one GPU each: the NCCL id is created
on rank 0 and broadcast through torch.distributed (gloo), each rank builds
its x-slab context with halo="nccl", sets the config-2/4 recipe's charged
spheres, solves to 1e-8 and writes its Phi slab.  The gathered solution is
compared with the single-domain CPU oracle (Phi rel-L2 <= 1e-10, equal cycle
counts, residual histories 1e-8 relative), and a killed peer makes the
survivor return MG_ERR_NCCL within the timeout instead of hanging
(mg_opts.nccl_timeout_ms).
"""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_1410_6609_b200 import workloads as W

pytestmark = pytest.mark.gpu


def _ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _case(kind):
    if kind == "channel":
        return W.cfg2(seed=5, shape=(256, 64, 128), n_spheres=50)
    w = W.cfg2(seed=6, shape=(256, 32, 128), n_spheres=30)
    w.bc_type, w.bc_value = W.periodic_channel_bc(1.0)
    return w


def _rank_main(rank, world, port, kind, outdir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank)
        from paper_1410_6609_b200 import dist as D
        from paper_1410_6609_b200 import mg
        uid = D.share_nccl_id(rank, mg.nccl_unique_id)
        w = _case(kind)
        s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, device=rank,
                         min_coarse=w.min_coarse, nranks=world, rank=rank,
                         halo="nccl", nccl_id=uid, nccl_timeout_ms=120000)
        s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
        rc, cyc, hist = s.solve(w.tol, 40)
        np.save(os.path.join(outdir, "phi%d.npy" % rank), s.get_solution())
        np.save(os.path.join(outdir, "hist%d.npy" % rank), hist)
        s.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["channel", "periodic"])
@pytest.mark.parametrize("world", [2, 4])
def test_nccl_slabs_equal_oracle(tmp_path, world, kind):
    if _ngpus() < world:
        pytest.skip("needs %d GPUs" % world)
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, kind, str(tmp_path)))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(600)
        assert p.exitcode == 0
    w = _case(kind)
    phi = np.concatenate([np.load(tmp_path / ("phi%d.npy" % r)) for r in range(world)])
    hists = [np.load(tmp_path / ("hist%d.npy" % r)) for r in range(world)]
    for h in hists[1:]:
        assert np.array_equal(h, hists[0])  # one collective norm
    o = oracle.Oracle(w.shape, w.h, w.bc_type, w.bc_value, min_coarse=w.min_coarse)
    o.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    st, cyc, ho = o.solve(w.tol, 40)
    assert st == 0 and len(ho) == len(hists[0])
    for a, b in zip(hists[0], ho):
        assert abs(a - b) <= 1e-8 * b + 1e-15 * ho[0]
    err = np.linalg.norm(phi - o.phi()) / np.linalg.norm(o.phi())
    assert err <= 1e-10


def _dead_peer_main(rank, port, outdir):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(rank)
    from paper_1410_6609_b200 import dist as D
    from paper_1410_6609_b200 import mg
    uid = D.share_nccl_id(rank, mg.nccl_unique_id)
    w = _case("channel")
    s = mg.Multigrid(w.shape, w.h, w.bc_type, w.bc_value, device=rank,
                     min_coarse=w.min_coarse, nranks=2, rank=rank, halo="nccl",
                     nccl_id=uid, nccl_timeout_ms=5000)
    s.set_rhs_from_spheres(w.centers, w.radii, w.charges)
    s.vcycle()
    dist.barrier()
    if rank == 1:
        os._exit(0)  # the peer dies without a word
    code = 0
    try:
        for _ in range(4):
            s.vcycle()
    except mg.MGError as e:
        code = e.code
    open(os.path.join(outdir, "code"), "w").write(str(code))
    os._exit(0)


def test_dead_peer_returns_nccl_error(tmp_path):
    if _ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    import torch.multiprocessing as tmp
    ctx = tmp.get_context("spawn")
    port = _free_port()
    procs = [ctx.Process(target=_dead_peer_main, args=(r, port, str(tmp_path)))
             for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(300)
    code = int(open(tmp_path / "code").read())
    from paper_1410_6609_b200 import mg
    assert code == mg.MG_ERR_NCCL
