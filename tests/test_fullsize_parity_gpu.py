"""Parity at the sizes BASELINE quotes, in the precision that is timed.

* Per kernel (tests/loop_probe.py): the loop's own intermediates after
  iterations 0 and 1 — Adam moments, capped step, composed field, smoothed
  field, W/G gather, loss values — against the oracle fed the same GPU inputs:
  fp32 within 1e-5 relative + 1e-6 of the output's peak (north_star's per-kernel
  criterion, the absolute term scaled to the peak for the 2/N-scaled LNCC
  gradients); fp64 within 1e-10 / 1e-12.  With default context
  options these are the benchmarked kernels: at 160x192x224 the two-row fp32
  smooth+Adam, the radius-0 compose kernel and the cp.async compose-smooth
  (DFM_OPT_LARGE_MIN, DFM_OPT_SPLIT_FOLD_MAX: 2M voxels).
* The same large-level variants forced at small sizes (DFM_OPT_LARGE_MIN = 0)
  end to end against the reference goldens.
* End to end: config 1 at full size, scale 1 x 3 iterations, every loss within
  1e-4 relative of the reference in both precisions; config 3 (SSD, sigma_grad
  1.5 -> radius-5 smoothing) at full size with a short schedule and with the
  full 250/150/75 schedule against the committed reference run (fp64: losses
  within 1e-4, field within 1e-3 voxel); configs 0 and 1 (LNCC) with the full
  200/100/50 schedule against the reference, where the loop is chaotic: the
  reference built with FMA contraction (an IEEE-valid rounding change of the
  reference itself) drifts from the plain build by 1.3e-3 / 2.0e-3 in the loss
  and 0.56 / 4.6 voxels in the field, so the GPU fp64 context is held to that
  envelope (_envelope_check) and to 1e-6 while the reference's own drift is
  below 1e-8; fp32 warped-label Dice within 0.002 of the reference run.
"""
import functools
import hashlib
import os

import numpy as np
import pytest

import loop_probe
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import (Context, OPT_BRICK_MAX, OPT_LARGE_MIN,
                                          OPT_SPLIT_FOLD_MAX)

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))
TOL = {"f32": (1e-5, 1e-6, 1e-5), "f64": (1e-10, 1e-12, 1e-10)}


@functools.lru_cache(maxsize=None)
def pair(config, shape=None):
    return synth.make_pair(config, seed=0, shape=shape)


@functools.lru_cache(maxsize=None)
def oracle():
    from oracle import pyoracle
    return pyoracle.best()


@functools.lru_cache(maxsize=None)
def ref_full_schedule(config):
    p = pair(config)
    return oracle().register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)


FORCE_LARGE = {OPT_LARGE_MIN: 0, OPT_SPLIT_FOLD_MAX: 0, OPT_BRICK_MAX: 0}


def _ctx(prec, opts=None):
    c = Context(0, prec)
    for k, v in (opts or {}).items():
        c.set_option(k, v)
    return c


def _assert_probe(ctx, p, cfg, prec):
    P = loop_probe.probe(ctx, p.grid, p.fixed, p.moving, cfg)
    r = loop_probe.check(oracle(), p.grid, p.fixed, p.moving, cfg, P, *TOL[prec])
    print({k: f"{v:.3g}" for k, v in r.items()})
    bad = {k: v for k, v in r.items() if not v <= 1.0}
    assert not bad, bad


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_config1_fullsize_per_kernel(prec):
    """The benchmarked kernels at 160x192x224 (default options)."""
    p = pair(1)
    ctx = _ctx(prec)
    try:
        _assert_probe(ctx, p, p.config, prec)
    finally:
        ctx.close()


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_config3_fullsize_per_kernel(prec):
    """SSD with sigma_grad 1.5 (radius-5 smooth+Adam) at 192x192x208."""
    p = pair(3)
    ctx = _ctx(prec)
    try:
        _assert_probe(ctx, p, p.config, prec)
    finally:
        ctx.close()


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_large_variants_forced_small_per_kernel(prec):
    """Two-row smooth+Adam, radius-0 compose and cp.async compose-smooth at
    40x48x56 (LARGE_MIN = 0, SPLIT_FOLD_MAX = 0, no bricks)."""
    p = pair(1, (56, 48, 40))
    ctx = _ctx(prec, FORCE_LARGE)
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=2)
    cfg.eta = 0.2  # eta 0.5 folds this small phantom after one step (in the reference too)
    try:
        _assert_probe(ctx, p, cfg, prec)
    finally:
        ctx.close()


@pytest.mark.parametrize("name", ["lncc", "ssd"])
def test_large_variants_forced_small_end_to_end_fp64(name):
    import golden_cases as G
    z, g, sched = G.register_inputs(name)
    cfg = synth.baseline_config(A.LOSS_LNCC if name == "lncc" else A.LOSS_SSD, 2, 1.0,
                                max_iters=max(sched.iterations))
    ctx = _ctx("f64", FORCE_LARGE)
    fld, log = ctx.register_images(g, z["fixed"], z["moving"], cfg, sched)
    ctx.close()
    losses = np.array([r.loss for r in log.iterations])
    assert np.all(np.abs(losses - z["losses"]) <= 1e-4 * np.abs(z["losses"]))
    assert np.abs(fld - z["field"]).max() <= 1e-3


def test_large_variants_forced_small_dice_fp32(oracle_port):
    import golden_cases as G
    z, g, sched = G.register_inputs("lncc")
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=max(sched.iterations))
    ctx = _ctx("f32", FORCE_LARGE)
    fld, log = ctx.register_images(g, z["fixed"].astype(np.float32),
                                   z["moving"].astype(np.float32), cfg, sched)
    ctx.close()
    d_gpu = oracle_port.overlap_dice(g, oracle_port.warp_labels(g, z["moving_labels"], fld),
                                     z["fixed_labels"])[0]
    d_ref = oracle_port.overlap_dice(g, oracle_port.warp_labels(g, z["moving_labels"],
                                                                z["field"]),
                                     z["fixed_labels"])[0]
    assert abs(d_gpu - d_ref) <= 0.002, (d_gpu, d_ref)


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_config1_fullsize_three_iterations(prec):
    """Scale 1 only, 3 iterations at 160x192x224: every iteration's loss within
    1e-4 relative (north_star) and the final field against the reference."""
    p = pair(1)
    sched = A.PyramidSchedule((1.0,), (3,))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=3)
    ctx = _ctx(prec)
    fa, la = ctx.register_images(p.grid, p.fixed, p.moving, cfg, sched)
    ctx.close()
    fb, lb = oracle().register_images(p.grid, p.fixed, p.moving, cfg, sched)
    a = np.array([r.loss for r in la.iterations])
    b = np.array([r.loss for r in lb.iterations])
    print(prec, "loss rel", np.abs(a - b) / np.abs(b), "field max", np.abs(fa - fb).max())
    assert a.shape == b.shape
    assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b))
    assert abs(la.final_loss - lb.final_loss) <= 1e-4 * abs(lb.final_loss)
    d = np.abs(fa - fb)
    print(prec, "field |diff| max", d.max(), "p99.99", np.quantile(d, 0.9999), "mean", d.mean())
    if prec == "f64":
        assert d.max() <= 1e-8
    else:
        # fp32: Adam's first steps are sign-like, dir = g / (|g| + eps) with eps
        # 1e-8 ~ |g| at 2/N-scaled LNCC gradients, so voxels where |g| ~ eps
        # amplify fp32 rounding (bounded by cap 0.5 before sigma_warp smoothing);
        # everywhere else the field agrees to fp32 rounding
        assert np.quantile(d, 0.9999) <= 1e-3 and d.max() <= 0.05


def _envelope_check(a, b, fa, fb, lf, ff, what):
    """GPU fp64 (a, fa) against the reference (b, fb) on a chaotic LNCC run.
    north_star's end-to-end criteria (losses within 1e-4 relative, field
    within 1e-3 voxel) hold wherever the problem allows them: the bound is
    max(criterion, envelope), the envelope being how far the SAME reference
    drifts from itself under an IEEE-valid rounding change (its FMA build:
    losses lf, field ff).  Loss: the whole curve within the envelope's
    maximum.  Field: max and mean |diff| within 2x the envelope's (one
    rounding realisation of a chaotic map is a sample, not a bound).  Before
    the reference's own drift exceeds 1e-8 the GPU must agree to 1e-6."""
    rel = np.abs(a - b) / np.abs(b)
    env = np.abs(lf - b) / np.abs(b)
    env_max = np.maximum.accumulate(env)
    d, e = np.abs(fa - fb), np.abs(ff - fb)
    print(f"{what}: GPU-vs-ref loss rel max {rel.max():.2e} (reference FMA build: "
          f"{env.max():.2e}); field max {d.max():.3e} mean {d.mean():.2e} "
          f"(FMA build {e.max():.3e} / {e.mean():.2e})")
    calm = env_max < 1e-8
    assert np.all(rel[calm] <= 1e-6), rel[calm].max()
    assert rel.max() <= max(1e-4, env.max())
    assert d.max() <= max(1e-3, 2 * e.max())
    assert d.mean() <= max(1e-4, 2 * e.mean())


def test_config0_full_schedule_fp64(ctx64):
    """Config 0 as BASELINE states it: 64^3, scales 4/2/1 x 200/100/50, LNCC."""
    from oracle import pyoracle
    p = pair(0)
    fa, la = ctx64.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    fb, lb = ref_full_schedule(0)
    ff, lfma = pyoracle.reference_fma().register_images(p.grid, p.fixed, p.moving, p.config,
                                                         p.schedule)
    a = np.array([r.loss for r in la.iterations])
    b = np.array([r.loss for r in lb.iterations])
    lf = np.array([r.loss for r in lfma.iterations])
    assert a.shape == b.shape == lf.shape == (350,)
    _envelope_check(a, b, fa, fb, lf, ff, "config 0")
    assert la.final_singularity_fraction == 0.0


def test_config0_full_schedule_fp32_dice(ctx32):
    p = pair(0)
    o = oracle()
    fa, la = ctx32.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    fb, lb = ref_full_schedule(0)
    da = o.overlap_dice(p.grid, o.warp_labels(p.grid, p.moving_labels, fa), p.fixed_labels)[0]
    db = o.overlap_dice(p.grid, o.warp_labels(p.grid, p.moving_labels, fb), p.fixed_labels)[0]
    assert abs(da - db) <= 0.002, (da, db)
    assert la.final_singularity_fraction == 0.0


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_config3_fullsize_short_schedule(prec):
    """Config 3 (SSD, sigma_grad 1.5, 192x192x208) through all three scales with
    a short schedule: losses within 1e-4 relative; fp64 field within 1e-3."""
    p = pair(3)
    sched = A.PyramidSchedule((4.0, 2.0, 1.0), (6, 4, 2))
    cfg = p.config
    ctx = _ctx(prec)
    fa, la = ctx.register_images(p.grid, p.fixed, p.moving, cfg, sched)
    ctx.close()
    fb, lb = oracle().register_images(p.grid, p.fixed, p.moving, cfg, sched)
    a = np.array([r.loss for r in la.iterations])
    b = np.array([r.loss for r in lb.iterations])
    print(prec, "loss rel max", (np.abs(a - b) / np.abs(b)).max(), "field",
          np.abs(fa - fb).max())
    assert a.shape == b.shape
    assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b))
    if prec == "f64":
        assert np.abs(fa - fb).max() <= 1e-3


def _golden_full(config):
    path = os.path.join(HERE, "golden", f"fullsize_cfg{config}.npz")
    if not os.path.exists(path):
        pytest.fail(f"{path} missing: run tests/golden/make_golden_fullsize.py")
    z = np.load(path)
    p = pair(config)
    sha = lambda a: hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()  # noqa: E731
    assert sha(p.fixed) == str(z["fixed_sha"]) and sha(p.moving) == str(z["moving_sha"]), \
        "regenerated inputs differ from the ones the golden run used"
    return z, p


@pytest.mark.parametrize("config", [1, 3])
def test_full_schedule_fp64_matches_reference_run(ctx64, config):
    """The benchmarked schedule in the parity context against the committed
    reference run (every 4th voxel per axis of the field).  Config 3 (SSD)
    is well conditioned: every loss within 1e-4 relative, the field within
    1e-3 voxel.  Config 1 (LNCC) is chaotic: _envelope_check."""
    z, p = _golden_full(config)
    fa, la = ctx64.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    a = np.array([r.loss for r in la.iterations])
    b = z["losses"]
    assert a.shape == b.shape
    s = int(z["stride"])
    fsub = fa[::s, ::s, ::s]
    if config == 3:
        print("fp64 loss rel max", (np.abs(a - b) / np.abs(b)).max())
        assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b))
        assert np.abs(fsub - z["field_sub"]).max() <= 1e-3
        assert abs(la.final_loss - float(z["final_loss"])) <= 1e-4 * abs(float(z["final_loss"]))
    else:
        _envelope_check(a, b, fsub, z["field_sub"], z["fma_losses"], z["fma_field_sub"],
                        "config 1 (every 4th voxel)")
    assert la.final_singularity_fraction == float(z["sing"])


@pytest.mark.parametrize("config", [1, 3])
def test_full_schedule_fp32_dice_matches_reference_run(ctx32, oracle_port, config):
    """The benchmarked run itself (fp32, full schedule): warped-label Dice
    within 0.002 of the reference run's (north_star)."""
    z, p = _golden_full(config)
    fa, la = ctx32.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    w = oracle_port.warp_labels(p.grid, p.moving_labels, fa)
    d = oracle_port.overlap_dice(p.grid, w, p.fixed_labels)[0]
    a = np.array([r.loss for r in la.iterations])
    print("fp32 dice", d, "ref", float(z["dice_mo"]), "loss rel max",
          (np.abs(a - z["losses"]) / np.abs(z["losses"])).max())
    assert abs(d - float(z["dice_mo"])) <= 0.002
    assert la.final_singularity_fraction == 0.0
    assert np.abs(a - z["losses"]).max() <= 1e-2 * np.abs(z["losses"]).max()
