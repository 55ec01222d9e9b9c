"""The host-staged slab transport (engine.TorchDistTransport, the callbacks
of dfm_slab_transport) on CPU: two gloo ranks call the four callbacks exactly
as the library does (raw pointers, byte counts) — halo sendrecv with both
neighbours' buffers, fp64 sums, u64 maxima, and the unequal-count allgather
of owned slab blocks at a scale change."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    import torch.distributed as dist
    from paper_2404_01249_b200.engine import TorchDistTransport
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    tp = TorchDistTransport()
    res = {}
    # sendrecv: each rank sends its block to the other, receives theirs
    send = np.arange(6, dtype=np.float32) + 100 * rank
    recv = np.zeros(6, dtype=np.float32)
    rc = tp._cb[0](None, 1 - rank, send.ctypes.data, send.nbytes, recv.ctypes.data, recv.nbytes)
    res["sendrecv"] = (rc, recv.tolist())
    # fp64 sum over ranks, in place
    a = np.array([1.5, -2.0, 3.25], dtype=np.float64) * (rank + 1)
    rc = tp._cb[1](None, a.ctypes.data_as(C.POINTER(C.c_double)), a.size)
    res["sum"] = (rc, a.tolist())
    # u64 max (the max-step log: bit patterns of non-negative doubles)
    b = np.array([np.float64(0.25 * (rank + 1)).view(np.uint64), 7 + rank], dtype=np.uint64)
    rc = tp._cb[2](None, b.ctypes.data_as(C.POINTER(C.c_uint64)), b.size)
    res["max"] = (rc, [float(b[:1].view(np.float64)[0]), int(b[1])])
    # allgather of unequal blocks (slab owned planes differ by rank)
    counts = np.array([12, 20], dtype=np.int64)
    mine = np.full(counts[rank], rank + 1, dtype=np.uint8)
    allb = np.zeros(int(counts.sum()), dtype=np.uint8)
    rc = tp._cb[3](None, mine.ctypes.data, mine.nbytes, allb.ctypes.data,
                   counts.ctypes.data_as(C.POINTER(C.c_int64)))
    res["allgather"] = (rc, allb.tolist())
    out[rank] = res
    dist.destroy_process_group()


def test_torch_dist_transport_callbacks_two_ranks():
    ctx = mp.get_context("spawn")
    with ctx.Manager() as m:
        out = m.dict()
        port = _port()
        ps = [ctx.Process(target=_worker, args=(r, 2, port, out)) for r in range(2)]
        for p in ps:
            p.start()
        for p in ps:
            p.join(120)
            assert p.exitcode == 0
        r0, r1 = out[0], out[1]
    assert r0["sendrecv"] == (0, [100.0 + k for k in range(6)])
    assert r1["sendrecv"] == (0, [float(k) for k in range(6)])
    assert r0["sum"] == r1["sum"] == (0, [4.5, -6.0, 9.75])
    assert r0["max"] == r1["max"] == (0, [0.5, 8])
    assert r0["allgather"] == r1["allgather"] == (0, [1] * 12 + [2] * 20)
