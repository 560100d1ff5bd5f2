"""Multi-rank host logic (CPU): the shard partition, the exchange plan, and a
world_size-2 gloo run of the exchange the sharded driver performs after each
bisection."""
import os
import socket

import numpy as np
import pytest

from paper_2104_06494_b200 import dist as pdist


def test_shard_bounds_properties():
    rng = np.random.default_rng(0)
    for _ in range(500):
        m = int(rng.integers(0, 50_000_000))
        R = int(rng.integers(1, 9))
        b = pdist.shard_bounds(m, R)
        assert b[0] == 0 and b[-1] == m
        assert np.all(np.diff(b) >= 0)
        assert all(x % 2048 == 0 for x in b[:-1] if x < m)
        nb = [(b[r + 1] - b[r] + 2047) // 2048 for r in range(R)]
        assert max(nb) - min(nb) <= 1  # balanced to one block


def test_exchange_plan_covers_every_child_once():
    rng = np.random.default_rng(1)
    for _ in range(300):
        R = int(rng.integers(1, 9))
        kept_per = rng.integers(0, 5000, size=R)
        kept = np.concatenate([[0], np.cumsum(kept_per)])
        total = 2 * int(kept[-1])
        nxt = pdist.shard_bounds(total, R)
        owner = np.full(total, -1)
        sends = {}
        for r in range(R):
            s, rc = pdist.shard_plan(R, r, kept)
            for peer, src, dst, cnt in rc:
                assert 0 <= dst and dst + cnt <= nxt[r + 1] - nxt[r]
                g0 = nxt[r] + dst
                assert (owner[g0:g0 + cnt] == -1).all()
                owner[g0:g0 + cnt] = r
                # the child range it receives is the sender's [2 kept[peer] + src, ...)
                assert g0 == 2 * kept[peer] + src
            for peer, src, dst, cnt in s:
                sends[(r, peer, src, dst, cnt)] = True
        assert (owner >= 0).all()
        for r in range(R):
            _, rc = pdist.shard_plan(R, r, kept)
            for peer, src, dst, cnt in rc:
                assert (peer, r, src, dst, cnt) in sends


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gloo_worker(rank, size, port, kept, result_q):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=size)
    try:
        kept = np.asarray(kept, dtype=np.int64)
        # this rank's children, identified by their global index (geometry.cpp:124-125)
        children = np.arange(2 * kept[rank], 2 * kept[rank + 1], dtype=np.int64)
        nxt = pdist.shard_bounds(2 * int(kept[-1]), size)
        sends, recvs = pdist.shard_plan(size, rank, kept)
        # the same closures the library's host transport calls back into
        import torch
        reqs, bufs = [], []
        out = np.full(nxt[rank + 1] - nxt[rank], -1, dtype=np.int64)
        for peer, src, dst, cnt in sends:
            if peer == rank:
                continue
            reqs.append(dist.isend(torch.from_numpy(children[src:src + cnt].copy()), int(peer)))
        for peer, src, dst, cnt in recvs:
            if peer == rank:
                out[dst:dst + cnt] = children[src:src + cnt]
                continue
            b = torch.empty(int(cnt), dtype=torch.int64)
            bufs.append((dst, b))
            reqs.append(dist.irecv(b, int(peer)))
        for r in reqs:
            r.wait()
        for dst, b in bufs:
            out[dst:dst + len(b)] = b.numpy()
        # the tiny collective the driver runs per fold: allgather of per-rank records
        rec = torch.tensor([rank, len(out)], dtype=torch.int64)
        gathered = [torch.empty_like(rec) for _ in range(size)]
        dist.all_gather(gathered, rec)
        result_q.put((rank, out.tolist(), [g.tolist() for g in gathered]))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kept", [[0, 3000, 4100], [0, 0, 5000], [0, 2500, 2500], [0, 70_000, 71_000]])
def test_gloo_world_size_2_exchange(kept):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, kept, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict()
    for _ in range(2):
        r, out, gathered = q.get(timeout=120)
        res[r] = (out, gathered)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    nxt = pdist.shard_bounds(2 * kept[-1], 2)
    for r in range(2):
        assert res[r][0] == list(range(nxt[r], nxt[r + 1]))
        assert res[r][1] == [[0, nxt[1] - nxt[0]], [1, nxt[2] - nxt[1]]]
