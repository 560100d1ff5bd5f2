"""Multi-GPU plumbing: one process per GPU.

`Communicator.nccl(...)` binds the library's NCCL transport (NVLink/NVSwitch);
`Communicator.host(...)` binds a host-callback transport.  `from_torch()`
builds either from an initialised torch.distributed process group: with the
NCCL backend the unique id is broadcast through torch and the library makes
its own NCCL communicator; with gloo (CPU tests, or several ranks sharing one
GPU) the exchanges run through torch.distributed on host memory.

    comm = dist.from_torch(device=local_rank)
    res = pg.integrate(f, bounds, pg.Config(..., comm=comm))
"""
from __future__ import annotations

import ctypes as C
import traceback

import numpy as np

from . import _native as N


class Communicator:
    def __init__(self, handle, rank, size, keepalive=None):
        self.handle = handle
        self.rank = rank
        self.size = size
        self._keep = keepalive

    @staticmethod
    def unique_id() -> bytes:
        buf = (C.c_uint8 * N.PAGANI_COMM_ID_BYTES)()
        N.check(N.load().pagani_comm_unique_id(buf))
        return bytes(buf)

    @staticmethod
    def nccl(unique_id: bytes, nranks: int, rank: int, device: int) -> "Communicator":
        buf = (C.c_uint8 * N.PAGANI_COMM_ID_BYTES).from_buffer_copy(unique_id)
        h = C.c_void_p()
        N.check(N.load().pagani_comm_init_rank(buf, nranks, rank, device, C.byref(h)))
        return Communicator(h, rank, nranks)

    @staticmethod
    def host(rank: int, size: int, allgather, exchange, device: int) -> "Communicator":
        """allgather(send: bytes) -> list[bytes] per rank;
        exchange(sends: list[(peer, bytes)], recvs: list[(peer, nbytes)]) -> list[bytes]."""

        def _ag(send, recv, nbytes, _user):
            try:
                data = C.string_at(send, nbytes) if nbytes else b""
                parts = allgather(data)
                blob = b"".join(parts)
                if blob:
                    C.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # noqa: BLE001 - reported to the library as a transport error
                traceback.print_exc()
                return 1

        def _ex(ns, speer, sbuf, sbytes, nr, rpeer, rbuf, rbytes, _user):
            try:
                sends = [(speer[i], C.string_at(sbuf[i], sbytes[i]) if sbytes[i] else b"")
                         for i in range(ns)]
                recvs = [(rpeer[i], rbytes[i]) for i in range(nr)]
                got = exchange(sends, recvs)
                for i in range(nr):
                    if rbytes[i]:
                        C.memmove(rbuf[i], got[i], rbytes[i])
                return 0
            except Exception:  # noqa: BLE001
                traceback.print_exc()
                return 1

        ag = N.ALLGATHER_FN(_ag)
        ex = N.EXCHANGE_FN(_ex)
        t = N.HostTransport(rank, size, None, ag, ex)
        h = C.c_void_p()
        N.check(N.load().pagani_comm_init_host(C.byref(t), device, C.byref(h)))
        return Communicator(h, rank, size, keepalive=(ag, ex, t))

    def destroy(self):
        if self.handle:
            N.check(N.load().pagani_comm_destroy(self.handle))
            self.handle = None


def torch_host_transport(device: int) -> Communicator:
    """Host-callback transport over the current torch.distributed group (gloo)."""
    import torch
    import torch.distributed as dist
    rank, size = dist.get_rank(), dist.get_world_size()

    def allgather(data: bytes):
        t = torch.frombuffer(bytearray(data), dtype=torch.uint8) if data else torch.zeros(0, dtype=torch.uint8)
        out = [torch.empty_like(t) for _ in range(size)]
        dist.all_gather(out, t)
        return [o.numpy().tobytes() for o in out]

    def exchange(sends, recvs):
        reqs = []
        for peer, data in sends:
            reqs.append(dist.isend(torch.frombuffer(bytearray(data), dtype=torch.uint8), peer))
        bufs = []
        for peer, nbytes in recvs:
            b = torch.empty(nbytes, dtype=torch.uint8)
            bufs.append(b)
            reqs.append(dist.irecv(b, peer))
        for r in reqs:
            r.wait()
        return [b.numpy().tobytes() for b in bufs]

    return Communicator.host(rank, size, allgather, exchange, device)


def from_torch(device: int) -> Communicator:
    """Library communicator for the current torch.distributed group: NCCL
    when the group's backend is nccl, else a host transport."""
    import torch
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        rank, size = dist.get_rank(), dist.get_world_size()
        obj = [Communicator.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return Communicator.nccl(obj[0], size, rank, device)
    return torch_host_transport(device)


def shard_bounds(m: int, nranks: int):
    b = np.empty(nranks + 1, dtype=np.int64)
    N.check(N.load().pagani_shard_bounds(m, nranks, b.ctypes.data_as(C.POINTER(C.c_int64))))
    return b


def shard_plan(nranks: int, rank: int, kept):
    kept = np.ascontiguousarray(kept, dtype=np.int64)
    maxp = 4 * nranks + 4
    s = np.empty((maxp, 4), dtype=np.int64)
    r = np.empty((maxp, 4), dtype=np.int64)
    ns, nr = C.c_int32(), C.c_int32()
    p = lambda a: a.ctypes.data_as(C.POINTER(C.c_int64))  # noqa: E731
    N.check(N.load().pagani_shard_plan(nranks, rank, p(kept), maxp, C.byref(ns), p(s),
                                       C.byref(nr), p(r)))
    return s[:ns.value], r[:nr.value]
