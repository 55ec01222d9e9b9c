"""Results do not depend on concurrency (the reference's thread-count
bit-identity, test_pipeline.cpp:201-219, and its re-entrant sweep workers,
pipeline.cpp:287-301): registrations running at the same time on separate
contexts of one GPU — the batch/sweep pattern — give the bits each gives alone,
and the native sweep gives the same rows with 1 and 3 workers per device."""
import threading

import numpy as np
import pytest

from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200 import sweep as S
from paper_2404_01249_b200.engine import Context

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_concurrent_contexts_bit_identical(prec):
    # a brick level and a plane-streaming level per pair
    pairs = [synth.make_pair(1, seed=40 + k, shape=(64, 48, 96)) for k in range(3)]
    sched = A.PyramidSchedule((2.0, 1.0), (6, 4))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=6)
    cfg.eta = 0.3

    def run(p):
        ctx = Context(0, prec)
        f, log = ctx.register_images(p.grid, p.fixed, p.moving, cfg, sched)
        ctx.close()
        return f, [r.loss for r in log.iterations]

    alone = [run(p) for p in pairs]
    together = [None] * len(pairs)

    def worker(k):
        together[k] = run(pairs[k])

    th = [threading.Thread(target=worker, args=(k,)) for k in range(len(pairs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for (fa, la), (fb, lb) in zip(alone, together):
        assert np.array_equal(fa, fb)
        assert la == lb


def test_sweep_rows_independent_of_workers():
    pairs = []
    for k in range(2):
        p = synth.make_pair(0, seed=30 + k, shape=(16, 16, 16))
        pairs.append(S.SweepPair(p.grid, p.fixed, p.moving, p.fixed_labels.astype(np.int32),
                                 p.moving_labels.astype(np.int32), f"pair{k}"))
    base = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=4)
    grid = dict(etas=[0.3, 0.6], sigma_warps=[0.5], sigma_grads=[1.0, 1.5])
    sched = A.PyramidSchedule((2.0, 1.0), (4, 3))
    rows = [S.sweep(pairs, base, sched, precision="f32", workers_per_device=w, **grid).rows
            for w in (1, 3)]
    assert [(r.failed, r.metric_mean) for r in rows[0]] == \
        [(r.failed, r.metric_mean) for r in rows[1]]


@pytest.mark.parametrize("persist", [2, 3])
def test_concurrent_persistent_levels(persist):
    """The neighbour-synchronised persistent solver is one cooperative launch
    per brick level whose CTAs spin on their neighbours: several contexts
    launching it at once must neither deadlock (a stall would raise) nor
    change any bit.  40x48x56 is the config-1 coarse level (420 bricks, the
    default solver's size); persist 3 also forces it on the small level."""
    from paper_2404_01249_b200.engine import OPT_PERSIST
    pairs = [synth.make_pair(1, seed=50 + k, shape=(112, 96, 80)) for k in range(3)]
    sched = A.PyramidSchedule((2.0, 1.0), (12, 2))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=12)
    cfg.eta = 0.3

    def run(p):
        ctx = Context(0, "f32")
        ctx.set_option(OPT_PERSIST, persist)
        f, log = ctx.register_images(p.grid, p.fixed, p.moving, cfg, sched)
        ctx.close()
        return f, [r.loss for r in log.iterations]

    alone = [run(p) for p in pairs]
    together = [None] * len(pairs)
    errors = []

    def worker(k):
        try:
            together[k] = run(pairs[k])
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(e)

    th = [threading.Thread(target=worker, args=(k,)) for k in range(len(pairs))]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors, errors
    for (fa, la), (fb, lb) in zip(alone, together):
        assert np.array_equal(fa, fb)
        assert la == lb
