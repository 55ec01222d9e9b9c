"""SVF mode on the device: exp_map, svf_pullback
(diffeo.cpp:66-167) and register_images in svf mode (pipeline.cpp:166-167,
189-206, 213-215), against the reference's golden vectors.

Tolerances: fp64 kernels within 1e-10 of the reference (different but exact
arithmetic order in the Jacobian term); fp32 kernels 1e-5 relative to the
output's peak (BASELINE per-kernel criterion, scaled like the LNCC gradients);
fp64 end to end: losses 1e-4 relative, final field 1e-3 voxel; fp32 end to end:
warped-label Dice within 0.002.
"""
import numpy as np
import pytest

import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth

pytestmark = pytest.mark.gpu


def _tol(prec, want):
    peak = float(np.abs(want).max()) or 1.0
    return (1e-10 if prec == "f64" else 1e-5) * peak


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("tag", ["3d", "2d"])
def test_exp_map_and_pullback_match_reference(request, prec, tag):
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    for key, (got, want) in G.compute_svf(ctx, tag).items():
        err = np.abs(got - want).max()
        assert err <= _tol(prec, want), (key, err)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_pullback_is_bit_stable(request, prec):
    """The sorted-gather scatter: identical bits run to run (the reference's
    serial scatter is deterministic; a float-atomic one would not be)."""
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    rng = np.random.default_rng(5)
    g = A.GridMeta.make_3d(40, 36, 30)
    v = rng.normal(0, 2.0, g.field_shape)
    w = rng.normal(0, 1.0, g.field_shape)
    a = ctx.svf_pullback(g, v, w, 6)
    b = ctx.svf_pullback(g, v, w, 6)
    assert np.array_equal(a, b)


def test_pullback_is_the_adjoint_of_exp_map(ctx64):
    """<pullback(v, w), dv> equals the directional derivative <w, d exp(v)[dv]>
    (central differences) at a size the golden vectors do not cover."""
    rng = np.random.default_rng(9)
    g = A.GridMeta.make_3d(48, 40, 32)
    from scipy import ndimage
    v = np.stack([ndimage.gaussian_filter(rng.normal(0, 1, g.shape), 3) * 20 for _ in range(3)],
                 axis=-1)
    dv = np.stack([ndimage.gaussian_filter(rng.normal(0, 1, g.shape), 3) for _ in range(3)],
                  axis=-1)
    w = rng.normal(0, 1, g.field_shape)
    M = 4
    lhs = float(np.sum(ctx64.svf_pullback(g, v, w, M) * dv))
    eps = 1e-6
    dphi = (ctx64.exp_map(g, v + eps * dv, M) - ctx64.exp_map(g, v - eps * dv, M)) / (2 * eps)
    rhs = float(np.sum(w * dphi))
    assert abs(lhs - rhs) <= 1e-5 * max(abs(rhs), 1.0), (lhs, rhs)


@pytest.mark.parametrize("name", ["svf_lncc", "svf_ssd"])
def test_fp64_svf_registration_matches_reference(ctx64, name):
    z, g, sched = G.register_inputs(name)
    cfg = G.register_config(name, z, sched)
    fld, log = ctx64.register_images(g, z["fixed"], z["moving"], cfg, sched)
    losses = np.array([r.loss for r in log.iterations])
    assert len(losses) == len(z["losses"])
    assert np.all(np.abs(losses - z["losses"]) <= 1e-4 * np.abs(z["losses"]))
    assert np.abs(fld - z["field"]).max() <= 1e-3
    assert abs(log.final_loss - float(z["final_loss"])) <= 1e-4 * abs(float(z["final_loss"]))
    ms = np.array([r.max_step for r in log.iterations])
    assert np.allclose(ms, z["max_steps"], rtol=1e-6, atol=1e-9)


def test_fp32_svf_registration_dice(ctx32, oracle_port):
    z, g, sched = G.register_inputs("svf_lncc")
    cfg = G.register_config("svf_lncc", z, sched)
    fld, log = ctx32.register_images(g, z["fixed"].astype(np.float32),
                                     z["moving"].astype(np.float32), cfg, sched)
    w_gpu = oracle_port.warp_labels(g, z["moving_labels"], fld)
    w_ref = oracle_port.warp_labels(g, z["moving_labels"], z["field"])
    d_gpu = oracle_port.overlap_dice(g, w_gpu, z["fixed_labels"])[0]
    d_ref = oracle_port.overlap_dice(g, w_ref, z["fixed_labels"])[0]
    assert abs(d_gpu - d_ref) <= 0.002, (d_gpu, d_ref)


def test_svf_runs_are_bit_reproducible(ctx32):
    z, g, sched = G.register_inputs("svf_ssd")
    cfg = G.register_config("svf_ssd", z, sched)
    a, la = ctx32.register_images(g, z["fixed"], z["moving"], cfg, sched)
    b, lb = ctx32.register_images(g, z["fixed"], z["moving"], cfg, sched)
    assert np.array_equal(a, b)
    assert [r.loss for r in la.iterations] == [r.loss for r in lb.iterations]


def test_svf_errors_map_to_reference_exceptions(ctx32):
    g = A.GridMeta.make_3d(8, 8, 8)
    v = np.zeros(g.field_shape)
    with pytest.raises(A.InvalidArgument):
        ctx32.exp_map(g, v, -1)
    with pytest.raises(A.InvalidArgument):
        ctx32.svf_pullback(g, v, v, -1)
    p = synth.make_pair(0, seed=1, shape=(16, 16, 16))
    cfg = synth.baseline_config(A.LOSS_DICE, 2, 1.0, max_iters=2)
    cfg.mode = A.MODE_SVF
    with pytest.raises(A.InvalidArgument):
        ctx32.register_images(p.grid, np.clip(p.fixed, 0, 1), np.clip(p.moving, 0, 1), cfg,
                              A.PyramidSchedule((1.0,), (2,)))


@pytest.mark.parametrize("mode", [A.MODE_DIRECT, A.MODE_SVF])
def test_nonfinite_step_raises_numerical(ctx32, mode):
    """A gradient that overflows fp32 (intensities ~3e19: the fp64 loss stays
    finite, (W - F) * grad M does not) makes the Adam step non-finite: both
    modes must fail with NumericalError (diffeo.cpp:52-53) instead of
    clamping NaN into the field and returning a corrupted result."""
    g = A.GridMeta.make_3d(12, 12, 12)
    rng = np.random.default_rng(3)
    F = (rng.random(g.shape) * 3e19).astype(np.float32)
    M = (rng.random(g.shape) * 3e19).astype(np.float32)
    cfg = A.RegistrationConfig(loss=A.LOSS_SSD, mode=mode)
    with pytest.raises(A.NumericalError):
        ctx32.register_images(g, F, M, cfg, A.PyramidSchedule((1.0,), (4,)))
