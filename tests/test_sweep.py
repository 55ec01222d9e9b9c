"""Sweep host logic on CPU: the restatement's sweep vs the reference's
(pipeline.cpp:226-313), and the multi-process config sharding (gloo,
world_size 2) the GPU sweep uses."""
import os

import numpy as np
import pytest

from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200 import sweep as S
from sweep_checker import run_checker


def _pairs(n=2, shape=(16, 16, 16)):
    out = []
    for k in range(n):
        p = synth.make_pair(0, seed=30 + k, shape=shape)
        out.append(S.SweepPair(p.grid, p.fixed, p.moving, p.fixed_labels.astype(np.int32),
                               p.moving_labels.astype(np.int32), f"pair{k}"))
    return out


GRID = dict(etas=[0.3, 0.6], sigma_warps=[0.0, 0.5], sigma_grads=[1.0, 1.5])
SCHED = A.PyramidSchedule((2.0, 1.0), (4, 3))


@pytest.mark.parametrize("metric", ["loss", "overlap"])
def test_restatement_sweep_matches_reference(oracle_port, metric):
    from oracle import pyoracle
    if not pyoracle.reference_available():
        pytest.skip("reference library not built")
    pairs = _pairs()
    base = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=4)
    a = run_checker(oracle_port, pairs, base, SCHED, metric=metric, **GRID)
    b = run_checker(pyoracle.reference(), pairs, base, SCHED, metric=metric, workers=3,
                      **GRID)
    assert len(a) == len(b) == 8
    for ra, rb in zip(a, b):
        assert (ra.eta, ra.sigma_warp, ra.sigma_grad) == (rb.eta, rb.sigma_warp, rb.sigma_grad)
        assert ra.failed == rb.failed and ra.error == rb.error
        assert np.array_equal([ra.metric_mean, ra.metric_sd], [rb.metric_mean, rb.metric_sd],
                              equal_nan=True)


def test_sweep_validation(oracle_port):
    base = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=4)
    with pytest.raises(A.InvalidArgument):
        run_checker(oracle_port, _pairs(1), base, SCHED, etas=[], sigma_warps=[0.5],
                      sigma_grads=[1.0])
    p = _pairs(1)
    p[0].fixed_labels = None
    with pytest.raises(A.InvalidArgument):
        run_checker(oracle_port, p, base, SCHED, metric="overlap", **GRID)


def test_config_axes_and_heatmaps():
    n_eta, n_sw, n_sg = 3, 2, 4
    rows = [S.SweepRow(0, 0, 0, metric_mean=float(k)) for k in range(n_eta * n_sw * n_sg)]
    h = S.heatmaps(rows, n_eta, n_sw, n_sg)
    for k in range(len(rows)):
        ei, wi, gi = S.config_axes(k, n_sw, n_sg)
        assert k == (ei * n_sw + wi) * n_sg + gi
        assert h[ei][wi][gi] == float(k)


def test_merge_shards_rejects_gaps_and_duplicates():
    r = S.SweepRow(0, 0, 0)
    with pytest.raises(RuntimeError):
        S.merge_shards([[r, None], [None, None]])
    with pytest.raises(RuntimeError):
        S.merge_shards([[r, None], [r, r]])
    assert S.merge_shards([[r, None], [None, r]]) == [r, r]


def _worker(rank, world, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_cfg = 2 * 2 * 2

    def runner(shard):  # stands in for dfm_sweep on this rank's GPU
        b, step = shard
        out = [None] * n_cfg
        for k in range(b, n_cfg, step):
            out[k] = S.SweepRow(0, 0, 0, metric_mean=100.0 * k + rank)
        return out

    res = S.sweep_distributed([], None, None, [0.1, 0.2], [0.0, 0.5], [1.0, 2.0],
                              runner=runner)
    if rank == 0:
        q.put([r.metric_mean for r in res.rows])
    dist.destroy_process_group()


def test_distributed_sharding_gloo():
    import multiprocessing as mp
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
    assert got == [100.0 * k + (k % 2) for k in range(8)]
