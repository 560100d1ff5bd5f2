"""Sharded (multi-rank) PAGANI on the GPU.

Only one GPU is available to the test harness, so R ranks run as R processes
sharing cuda:0 and exchanging through the host-callback transport over
torch.distributed/gloo.  The sharded driver code path (2048-aligned slices,
allgathered block records, speculative probes, re-partition + exchange after
every bisection) is the one NCCL runs on 8 GPUs; its results must be
bit-identical to the 1-GPU run (and hence to the reference).
"""
import os
import socket

import pytest

pytestmark = pytest.mark.gpu

CASES = [("f4", 5, 1e-3, {}), ("f3", 8, 1e-3, {}), ("f6", 6, 1e-3, {}), ("f2", 6, 1e-3, {}),
         ("f1", 3, 1e-3, {"rel_filtering_enabled": False}),
         ("f4", 3, 5e-7, {"max_regions": 1 << 12, "init_target": 1 << 10}),
         ("f5", 8, 1e-3, {"it_max": 9})]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _summary(r):
    return (r.estimate, r.errorest, str(r.status), r.iterations, r.regions_generated,
            r.eval_count, [(e.iteration, e.success, e.batch_size, e.finished_count,
                            e.discarded_error, e.budget_limit) for e in r.threshold_events])


def _worker(rank, size, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import paper_2104_06494_b200 as pg
        from paper_2104_06494_b200 import dist as pdist
        comm = pdist.torch_host_transport(device=0)
        out = []
        for name, n, tau, extra in CASES:
            cfg = pg.Config(tau_rel=tau, comm=comm, **extra)
            r = pg.integrate(pg.integrand_by_id(name), pg.Bounds.unit_cube(n), cfg, trace=True)
            out.append((_summary(r), r.trace, r.region_evals))
        comm.destroy()
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("size", [2, 3])
def test_sharded_run_is_bit_identical_to_one_gpu(pg, gpu, size):
    import torch.multiprocessing as mp
    single = []
    for name, n, tau, extra in CASES:
        r = pg.integrate(pg.integrand_by_id(name), pg.Bounds.unit_cube(n),
                         pg.Config(tau_rel=tau, **extra), trace=True)
        single.append((_summary(r), r.trace, r.region_evals))
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q)) for r in range(size)]
    for p in procs:
        p.start()
    got = {}
    for _ in range(size):
        rank, out = q.get(timeout=900)
        got[rank] = out
    for p in procs:
        p.join(timeout=120)
    for rank in range(size):
        assert not isinstance(got[rank], str), got[rank]
        evals = 0
        for (s1, t1, e1), (s2, t2, e2) in zip(single, got[rank]):
            assert s2 == s1
            assert t2 == t1  # every per-iteration trace field
    for i in range(len(CASES)):  # the ranks split the work: local evals sum to the total
        assert sum(got[r][i][2] for r in range(size)) == single[i][2]


def test_nccl_transport_single_rank(pg, gpu):
    """The NCCL transport (dlopen'ed libnccl) drives the sharded path with one
    rank: allgathers and the post-bisection exchange go through NCCL; results
    stay bit-identical."""
    from paper_2104_06494_b200 import dist as pdist
    comm = pdist.Communicator.nccl(pdist.Communicator.unique_id(), 1, 0, 0)
    try:
        for name, n, tau, extra in CASES[:4]:
            a = pg.integrate(pg.integrand_by_id(name), pg.Bounds.unit_cube(n),
                             pg.Config(tau_rel=tau, **extra), trace=True)
            b = pg.integrate(pg.integrand_by_id(name), pg.Bounds.unit_cube(n),
                             pg.Config(tau_rel=tau, comm=comm, **extra), trace=True)
            assert _summary(a) == _summary(b) and a.trace == b.trace
    finally:
        comm.destroy()


def test_generic_integrand_rejected_when_sharded(pg, gpu):
    from paper_2104_06494_b200 import dist as pdist
    comm = pdist.Communicator.nccl(pdist.Communicator.unique_id(), 1, 0, 0)
    try:
        with pytest.raises(NotImplementedError):
            pg.integrate(pg.Integrand.constant(1.0), pg.Bounds.unit_cube(2), pg.Config(comm=comm))
    finally:
        comm.destroy()
