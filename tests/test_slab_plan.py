"""Host logic of the z-slab decomposition on CPU with torch.distributed/gloo
(world size 2, 127.0.0.1): every rank computes its slab plan through the C-ABI
(dfm_slab_bounds), fills owned planes of a global test volume, exchanges H
halo planes with its neighbours exactly as the library's NCCL path does
(send owned boundary planes, receive into the halo), and checks the halos equal
the global volume.  Also checks the plan partitions z exactly once."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2404_01249_b200.engine import slab_bounds, slab_halo
from paper_2404_01249_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, nz, H, results):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    ny, nx = 3, 4
    glob = torch.arange(nz * ny * nx, dtype=torch.float64).reshape(nz, ny, nx)
    zlo, zhi, hlo, hhi = slab_bounds(nz, rank, world, H)
    local = torch.full((hlo + (zhi - zlo) + hhi, ny, nx), -1.0, dtype=torch.float64)
    local[hlo:hlo + zhi - zlo] = glob[zlo:zhi]
    ops = []
    if rank > 0:
        ops.append(dist.P2POp(dist.isend, local[hlo:2 * hlo].contiguous(), rank - 1))
        lo_buf = torch.empty((hlo, ny, nx), dtype=torch.float64)
        ops.append(dist.P2POp(dist.irecv, lo_buf, rank - 1))
    if rank + 1 < world:
        top = hlo + zhi - zlo
        ops.append(dist.P2POp(dist.isend, local[top - hhi:top].contiguous(), rank + 1))
        hi_buf = torch.empty((hhi, ny, nx), dtype=torch.float64)
        ops.append(dist.P2POp(dist.irecv, hi_buf, rank + 1))
    for r in dist.batch_isend_irecv(ops):
        r.wait()
    if rank > 0:
        local[:hlo] = lo_buf
    if rank + 1 < world:
        local[hlo + zhi - zlo:] = hi_buf
    ok = bool(torch.equal(local, glob[zlo - hlo:zhi + hhi]))
    results[rank] = (ok, zlo, zhi)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
@pytest.mark.parametrize("nz", [16, 37])
def test_halo_exchange_plan_gloo(world, nz):
    cfg = synth.baseline_config()
    H = slab_halo(cfg)
    assert H == 3  # max(lncc r=2, ceil(3*1.0)=3, ceil(3*0.5)+1=3)
    mgr = mp.Manager()
    res = mgr.dict()
    port = _free_port()
    mp.spawn(_worker, args=(world, port, nz, H, res), nprocs=world, join=True)
    spans = sorted((res[r][1], res[r][2]) for r in range(world))
    assert all(res[r][0] for r in range(world))
    assert spans[0][0] == 0 and spans[-1][1] == nz
    assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))


def test_plan_partitions_and_halos():
    for nz in (7, 16, 128, 1024):
        for parts in (1, 2, 3, 8):
            if nz // parts < 3:
                continue
            covered = []
            for k in range(parts):
                zlo, zhi, hlo, hhi = slab_bounds(nz, k, parts, 3)
                covered += list(range(zlo, zhi))
                assert hlo == (0 if k == 0 else 3) and hhi == (0 if k == parts - 1 else 3)
            assert covered == list(range(nz))
