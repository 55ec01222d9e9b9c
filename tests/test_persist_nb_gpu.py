"""The neighbour-synchronised persistent level solver (kernels_brick.cu
k_persist_nb): every brick level of an LNCC registration in one cooperative
launch, bricks synchronised with their 26 neighbours only.  DFM_OPT_PERSIST = 3
forces it on every brick level (by default, 2, it runs where it is faster:
at least two bricks per SM and at most one per CTA slot).

It runs the brick kernels' per-voxel arithmetic in the same order, so it must
reproduce the per-iteration CUDA-graph brick path (DFM_OPT_PERSIST = 0) bit for
bit — fields, losses and max steps — including early stops (the levels where
the monitor can fire wait for its record), numerical failures (same error) and
step caps above 0.5 (the 2-voxel compose gather).  The graph path itself is
held to the reference in test_kernel_families_gpu.py; here the fp64 run is
also compared with the committed reference golden directly.
"""
import numpy as np
import pytest

import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context, OPT_BRICK_MAX, OPT_PERSIST

pytestmark = pytest.mark.gpu


def _run(prec, persist, g, fixed, moving, cfg, sched, brick_max=1 << 40):
    ctx = Context(0, prec)
    ctx.set_option(OPT_BRICK_MAX, brick_max)
    ctx.set_option(OPT_PERSIST, persist)
    try:
        return ctx.register_images(g, fixed, moving, cfg, sched)
    finally:
        ctx.close()


def _same(a, b):
    fa, la = a
    fb, lb = b
    assert [(r.scale_index, r.iter) for r in la.iterations] == \
        [(r.scale_index, r.iter) for r in lb.iterations]
    assert [r.loss for r in la.iterations] == [r.loss for r in lb.iterations]
    assert [r.max_step for r in la.iterations] == [r.max_step for r in lb.iterations]
    assert np.array_equal(fa, fb), np.abs(fa - fb).max()
    assert la.final_loss == lb.final_loss


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_matches_graph_path_bitwise(prec):
    z, g, sched = G.register_inputs("lncc")
    cfg = G.register_config("lncc", z, sched)
    dt = np.float64 if prec == "f64" else np.float32
    F, M = z["fixed"].astype(dt), z["moving"].astype(dt)
    nb = _run(prec, 3, g, F, M, cfg, sched)
    _same(nb, _run(prec, 0, g, F, M, cfg, sched))
    if prec == "f64":  # and the reference golden (north_star criteria)
        losses = np.array([r.loss for r in nb[1].iterations])
        assert np.all(np.abs(losses - z["losses"]) <= 1e-4 * np.abs(z["losses"]))
        assert np.abs(nb[0] - z["field"]).max() <= 1e-3


@pytest.mark.parametrize("shape,r,cap", [((21, 18, 13), 1, 0.5), ((24, 20, 17), 3, 0.5),
                                         ((37, 9, 11), 2, 1.0), ((40, 48, 56), 2, 0.5)])
def test_ragged_shapes_radii_caps(shape, r, cap):
    """partial bricks on every face, LNCC radii 1..3, the 2-voxel compose gather
    (cap 1.0), and the config-1 coarse level's 40x48x56 (420 bricks)"""
    rng = np.random.default_rng(sum(shape) + r)
    g = A.GridMeta(3, shape)
    n = int(np.prod(shape))
    x = np.linspace(0, 1, n).reshape(shape[::-1])
    fixed = (0.5 + 0.3 * np.sin(7 * x) + 0.05 * rng.standard_normal(shape[::-1])).ravel()
    moving = (0.5 + 0.3 * np.sin(7 * x + 0.2) + 0.05 * rng.standard_normal(shape[::-1])).ravel()
    sched = A.PyramidSchedule((1.0,), (9,))
    cfg = synth.baseline_config(A.LOSS_LNCC, r, 1.0, max_iters=9)
    cfg.step_cap = cap
    for prec in ("f64", "f32"):
        dt = np.float64 if prec == "f64" else np.float32
        _same(_run(prec, 3, g, fixed.astype(dt), moving.astype(dt), cfg, sched),
              _run(prec, 0, g, fixed.astype(dt), moving.astype(dt), cfg, sched))


@pytest.mark.parametrize("window,tol", [(5, 1e-3), (2, 1e-2), (1, 10.0)])
def test_early_stop_identical(window, tol):
    """levels that converge: every brick stops before the same update"""
    z, g, sched = G.register_inputs("lncc")
    cfg = G.register_config("lncc", z, sched)
    cfg.conv_window, cfg.conv_tol = window, tol
    a = _run("f64", 3, g, z["fixed"], z["moving"], cfg, sched)
    b = _run("f64", 0, g, z["fixed"], z["moving"], cfg, sched)
    _same(a, b)
    assert len(a[1].iterations) < sum(sched.iterations)


def test_self_registration_stops():
    z = G.load("register_self.npz")
    g = A.GridMeta.make_3d(16, 16, 16)
    cfg = A.RegistrationConfig()
    sched = A.PyramidSchedule()
    _same(_run("f64", 3, g, z["fixed"], z["fixed"], cfg, sched),
          _run("f64", 0, g, z["fixed"], z["fixed"], cfg, sched))


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_nonfinite_input_raises(prec):
    g = A.GridMeta.make_3d(24, 16, 16)
    rng = np.random.default_rng(41)
    F, M = rng.random(g.shape), rng.random(g.shape)
    F[3, 2, 1] = np.nan
    sched = A.PyramidSchedule((1.0,), (5,))
    msgs = []
    for persist in (3, 0):
        with pytest.raises(A.NumericalError) as e:
            _run(prec, persist, g, F, M, A.RegistrationConfig(), sched)
        msgs.append(str(e.value))
    assert msgs[0] == msgs[1]


def test_config1_coarse_levels():
    """the config-1 phantom's pyramid levels at 1/4 and 1/2 resolution, several
    iterations each, fp32; persist 3: the 1/2 level's 3360 bricks share the
    CTAs (several bricks per CTA and phase)"""
    p = synth.make_pair(1, seed=3, shape=(160, 192, 224), iters=(12, 4, 0))
    sched = A.PyramidSchedule((4.0, 2.0), (12, 4))
    a = _run("f32", 3, p.grid, p.fixed, p.moving, p.config, sched)
    b = _run("f32", 0, p.grid, p.fixed, p.moving, p.config, sched)
    _same(a, b)
    # the default (2) runs the 1/4 level (420 bricks) persistent, 1/2 on graphs
    _same(_run("f32", 2, p.grid, p.fixed, p.moving, p.config, sched), b)
