"""The native multi-context GPU sweep (dfm_sweep) against the reference's
sweep (pipeline.cpp:226-313) on the same pairs and grid.

fp64: every row's metric mean within 1e-6 relative of the reference (loss
metric; end-to-end criterion 1e-4), identical failure pattern (folded warps
when sigma_warp = 0) with the reference's error message; overlap metric: TO
means within 0.002 (the Dice-style label criterion).  Sharded runs (0,2) and
(1,2) together reproduce the unsharded rows bit for bit.
"""
import numpy as np
import pytest

from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200 import sweep as S
from sweep_checker import run_checker

pytestmark = pytest.mark.gpu

GRID = dict(etas=[0.3, 0.6], sigma_warps=[0.0, 0.5], sigma_grads=[1.0, 1.5])
SCHED = A.PyramidSchedule((2.0, 1.0), (4, 3))


def _pairs(n=2, shape=(16, 16, 16)):
    out = []
    for k in range(n):
        p = synth.make_pair(0, seed=30 + k, shape=shape)
        out.append(S.SweepPair(p.grid, p.fixed, p.moving, p.fixed_labels.astype(np.int32),
                               p.moving_labels.astype(np.int32), f"pair{k}"))
    return out


@pytest.mark.parametrize("workers", [1, 3])
def test_fp64_sweep_matches_reference(oracle_port, workers):
    from oracle import pyoracle
    ref = pyoracle.best()
    pairs = _pairs()
    base = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=4)
    got = S.sweep(pairs, base, SCHED, precision="f64", workers_per_device=workers, **GRID)
    want = run_checker(ref, pairs, base, SCHED, **GRID)
    assert len(got.rows) == len(want) == 8
    for a, b in zip(got.rows, want):
        assert (a.eta, a.sigma_warp, a.sigma_grad) == (b.eta, b.sigma_warp, b.sigma_grad)
        assert a.failed == b.failed, (a, b)
        if a.failed:
            assert a.error == b.error
        else:
            assert abs(a.metric_mean - b.metric_mean) <= 1e-6 * abs(b.metric_mean)
    assert got.heatmaps[1][1][0] == got.rows[(1 * 2 + 1) * 2 + 0].metric_mean or np.isnan(
        got.rows[6].metric_mean)


def test_overlap_metric_and_sharding(oracle_port):
    from oracle import pyoracle
    ref = pyoracle.best()
    pairs = _pairs()
    base = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=4)
    full = S.run_native(pairs, base, SCHED, metric="overlap", precision="f64",
                        workers_per_device=2, **GRID)
    want = run_checker(ref, pairs, base, SCHED, metric="overlap", **GRID)
    for a, b in zip(full, want):
        assert a.failed == b.failed
        if not a.failed:
            assert abs(a.metric_mean - b.metric_mean) <= 0.002
    parts = [S.run_native(pairs, base, SCHED, metric="overlap", precision="f64",
                          shard=(r, 2), **GRID) for r in range(2)]
    merged = S.merge_shards(parts)
    assert [r.metric_mean for r in merged if not r.failed] == \
        [r.metric_mean for r in full if not r.failed]


def test_sweep_errors(ctx32):
    base = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=4)
    with pytest.raises(A.InvalidArgument):
        S.run_native([], base, SCHED, **GRID)
    p = _pairs(1)
    p[0].moving_labels = None
    with pytest.raises(A.InvalidArgument):
        S.run_native(p, base, SCHED, metric="overlap", **GRID)
