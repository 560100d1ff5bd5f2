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


def _worker(rank, size, port, q, cases=None):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import paper_2104_06494_b200 as pg
        from paper_2104_06494_b200 import dist as pdist
        comm = pdist.torch_host_transport(device=0)
        out = []
        for name, n, tau, extra in (cases or CASES):
            cfg = pg.Config(tau_rel=tau, comm=comm, profile=cases is not None, **extra)
            r = pg.integrate(pg.integrand_by_id(name), pg.Bounds.unit_cube(n), cfg, trace=True)
            out.append((_summary(r), r.trace, r.region_evals,
                        {"exchange_bytes": r.kernel_bytes["exchange"],
                         "exchanges": r.kernel_launches["exchange"],
                         "exchange_ms": r.kernel_ms["exchange"], "device_ms": r.device_ms,
                         "evaluate_ms": r.kernel_ms["evaluate"], "peak_local": r.peak_regions}))
        comm.destroy()
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run_ranks(size, cases=None, timeout=900):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, size, port, q, cases)) for r in range(size)]
    for p in procs:
        p.start()
    got = {}
    try:
        for _ in range(size):
            rank, out = q.get(timeout=timeout)
            got[rank] = out
    finally:
        for p in procs:
            p.join(timeout=120)
            if p.is_alive():
                p.kill()
    return got


@pytest.mark.parametrize("size", [2, 3])
def test_sharded_run_is_bit_identical_to_one_gpu(pg, gpu, size):
    single = []
    for name, n, tau, extra in CASES:
        r = pg.integrate(pg.integrand_by_id(name), pg.Bounds.unit_cube(n),
                         pg.Config(tau_rel=tau, **extra), trace=True)
        single.append((_summary(r), r.trace, r.region_evals))
    got = _run_ranks(size)
    for rank in range(size):
        assert not isinstance(got[rank], str), got[rank]
        evals = 0
        for (s1, t1, e1), (s2, t2, e2, _) in zip(single, got[rank]):
            assert s2 == s1
            assert t2 == t1  # every per-iteration trace field
    for i in range(len(CASES)):  # the ranks split the work: local evals sum to the total
        assert sum(got[r][i][2] for r in range(size)) == single[i][2]


# BASELINE configs[3] (f5 / f6 8D tau=1e-8, the sharded-with-rebalance
# config) and the largest 8D suite member, at full size (cap 2^22)
FULL_CASES = [("f5", 8, 1e-8, {}), ("f6", 8, 1e-8, {}), ("f4", 8, 1e-6, {})]


@pytest.mark.parametrize("size", [2, 4, 8])
def test_sharded_full_size_matches_reference(pg, gpu, size):
    """Full-size BASELINE runs through the sharded driver (R ranks sharing
    cuda:0 over the host transport): every per-iteration trace field equals
    the 1-GPU run's, and the finals equal the unmodified reference's
    (tests/golden/finals_deep.json).  Per-rank exchange volume is logged to
    $PAGANI_XCHG_LOG."""
    import json

    from conftest import load_golden, unhex
    want = load_golden("finals_deep.json")
    single = []
    for name, n, tau, extra in FULL_CASES:
        r = pg.integrate(pg.integrand_by_id(name), pg.Bounds.unit_cube(n),
                         pg.Config(tau_rel=tau, **extra), trace=True)
        single.append((_summary(r), r.trace, r.region_evals))
        w = want[f"{name}_{n}d_{tau:g}"]
        assert (r.estimate, r.errorest, str(r.status), r.iterations, r.regions_generated,
                r.eval_count) == (unhex(w["estimate"]), unhex(w["errorest"]), w["status"],
                                  w["iterations"], w["regions_generated"], w["eval_count"])
    got = _run_ranks(size, FULL_CASES, timeout=1800)
    log = []
    for rank in range(size):
        assert not isinstance(got[rank], str), got[rank]
        for (s1, t1, e1), (s2, t2, e2, x), case in zip(single, got[rank], FULL_CASES):
            assert s2 == s1, (case, rank)
            assert t2 == t1, (case, rank)
            log.append({"ranks": size, "rank": rank, "case": f"{case[0]} {case[1]}D {case[2]:g}",
                        "iterations": s2[3], "local_region_evals": e2, **x})
    for i in range(len(FULL_CASES)):
        assert sum(got[r][i][2] for r in range(size)) == single[i][2]
    path = os.environ.get("PAGANI_XCHG_LOG")
    if path:
        old = json.load(open(path)) if os.path.exists(path) else []
        json.dump(old + log, open(path, "w"), indent=1)


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


GENERIC = [  # (integrand factory, n, tau, extra): the reference's unit-test lambdas
    (lambda pg: pg.Integrand.exp_sq(), 4, 1e-6, {}),
    (lambda pg: pg.Integrand.cos_sum(1.5, [0.7, 1.9, 2.6]), 3, 1e-5, {}),
    (lambda pg: pg.Integrand.constant(1.0), 3, 1e-3, {"init_subdiv": 2}),
]


def test_validate_invariants_sharded(pg, gpu, ref):
    """validate_invariants through the sharded driver (NCCL transport, one
    rank): the same outcome as the reference, incl. its volume-check abort."""
    from ref_ctypes import make_config

    from paper_2104_06494_b200 import dist as pdist
    comm = pdist.Communicator.nccl(pdist.Communicator.unique_id(), 1, 0, 0)
    try:
        for fid, n, tau in ((4, 3, 1e-6), (5, 5, 1e-4), (4, 5, 1e-3)):
            try:
                r = pg.integrate(pg.Integrand(fid), pg.Bounds.unit_cube(n),
                                 pg.Config(tau_rel=tau, validate_invariants=True, comm=comm))
                got = (r.estimate, r.errorest, str(r.status), r.iterations)
            except AssertionError as e:
                got = str(e)
            try:
                w = ref.integrate(fid, n, make_config(tau_rel=tau, validate_invariants=True))
                want = (w.estimate, w.errorest, w.status, w.iterations)
            except AssertionError as e:
                want = str(e)
            assert got == want
    finally:
        comm.destroy()


def test_generic_integrand_sharded_matches_single(pg, gpu):
    """Non-separable integrands (generic evaluator with its own fused block
    folds) run through the sharded path; bit-identical to one GPU."""
    from paper_2104_06494_b200 import dist as pdist
    comm = pdist.Communicator.nccl(pdist.Communicator.unique_id(), 1, 0, 0)
    try:
        for mk, n, tau, extra in GENERIC:
            a = pg.integrate(mk(pg), pg.Bounds.unit_cube(n), pg.Config(tau_rel=tau, **extra),
                             trace=True)
            b = pg.integrate(mk(pg), pg.Bounds.unit_cube(n),
                             pg.Config(tau_rel=tau, comm=comm, **extra), trace=True)
            assert _summary(a) == _summary(b) and a.trace == b.trace
    finally:
        comm.destroy()


def _generic_worker(rank, size, port, q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        import ctypes as C

        import numpy as np

        import paper_2104_06494_b200 as pg
        from paper_2104_06494_b200 import dist as pdist
        comm = pdist.torch_host_transport(device=0)
        out = []
        for mk, n, tau, extra in GENERIC:
            r = pg.integrate(mk(pg), pg.Bounds.unit_cube(n),
                             pg.Config(tau_rel=tau, comm=comm, **extra), trace=True)
            out.append((_summary(r), r.trace))
        # a caller-compiled functor (include/pagani_device.cuh), sharded
        lib = C.CDLL(os.path.join(os.path.dirname(os.path.abspath(__file__)), "ext",
                                  "libuser_integrands.so"))
        od, oi = np.zeros(2), np.zeros(4, dtype=np.int64)
        p = np.array([0.5, 625.0])
        rc = lib.user_integrate_comm(0, p.ctypes.data_as(C.c_void_p), 5, C.c_double(1e-3), 1,
                                     comm.handle, od.ctypes.data_as(C.c_void_p),
                                     oi.ctypes.data_as(C.c_void_p))
        out.append(("user", rc, float(od[0]), float(od[1]), [int(v) for v in oi]))
        comm.destroy()
        q.put((rank, out))
    except Exception as e:  # noqa: BLE001
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_generic_and_user_integrands_sharded_two_ranks(pg, gpu, ref):
    import torch.multiprocessing as mp

    from ref_ctypes import make_config
    single = [pg.integrate(mk(pg), pg.Bounds.unit_cube(n), pg.Config(tau_rel=tau, **extra),
                           trace=True) for mk, n, tau, extra in GENERIC]
    want = ref.integrate(4, 5, make_config(tau_rel=1e-3))  # the Gauss functor == f4
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_generic_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = dict(q.get(timeout=900) for _ in range(2))
    for p in procs:
        p.join(timeout=120)
    for rank in range(2):
        assert not isinstance(got[rank], str), got[rank]
        for a, (summ, tr) in zip(single, got[rank][:-1]):
            assert summ == _summary(a) and tr == a.trace
        _, rc, est, err, oi = got[rank][-1]
        assert rc == 0
        status = ["converged", "max_iterations", "memory_exhausted"][oi[0]]
        assert (est, err, status, oi[1], oi[2], oi[3]) == (
            want.estimate, want.errorest, want.status, want.iterations, want.regions_generated,
            want.eval_count)
