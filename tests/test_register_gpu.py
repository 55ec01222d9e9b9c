"""End-to-end parity of register_images on the device (through the C-ABI).

Criteria (BASELINE north_star), with SURVEY §8(c)'s finding that the loop is
chaotic (1 fp32 ulp on the inputs moves the fp64 oracle's final field by
0.235 voxel): the end-to-end field/loss criteria are held by the fp64
context; the fp32 context is held to the warped-label Dice criterion.
  fp64: final field max-abs <= 1e-3 voxel; every iteration loss within 1e-4
        relative; final loss within 1e-4 relative; same record count.
  fp32: |Dice(MO mean) - reference Dice| <= 0.002 on warped labels.
"""
import numpy as np
import pytest

import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth

pytestmark = pytest.mark.gpu


def cfg_for(name, sched):
    loss = A.LOSS_LNCC if name == "lncc" else A.LOSS_SSD
    return synth.baseline_config(loss, 2, 1.0, max_iters=max(sched.iterations))


@pytest.mark.parametrize("name", ["lncc", "ssd"])
def test_fp64_matches_reference_end_to_end(ctx64, name):
    z, g, sched = G.register_inputs(name)
    fld, log = ctx64.register_images(g, z["fixed"], z["moving"], cfg_for(name, sched), sched)
    losses = np.array([r.loss for r in log.iterations])
    assert len(losses) == len(z["losses"])
    assert np.all(np.abs(losses - z["losses"]) <= 1e-4 * np.abs(z["losses"]))
    assert np.abs(fld - z["field"]).max() <= 1e-3
    assert abs(log.final_loss - float(z["final_loss"])) <= 1e-4 * abs(float(z["final_loss"]))
    assert [r.scale_index for r in log.iterations] == list(z["scale_index"])
    assert log.final_singularity_fraction == 0.0
    ms = np.array([r.max_step for r in log.iterations])
    assert np.allclose(ms, z["max_steps"], rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("name", ["lncc", "ssd"])
def test_fp32_dice_within_0p002(ctx32, oracle_port, name):
    z, g, sched = G.register_inputs(name)
    fld, log = ctx32.register_images(g, z["fixed"].astype(np.float32),
                                     z["moving"].astype(np.float32), cfg_for(name, sched), sched)
    assert log.final_singularity_fraction == 0.0
    w_gpu = oracle_port.warp_labels(g, z["moving_labels"], fld)
    w_ref = oracle_port.warp_labels(g, z["moving_labels"], z["field"])
    d_gpu = oracle_port.overlap_dice(g, w_gpu, z["fixed_labels"])[0]
    d_ref = oracle_port.overlap_dice(g, w_ref, z["fixed_labels"])[0]
    assert abs(d_gpu - d_ref) <= 0.002, (d_gpu, d_ref)
    losses = np.array([r.loss for r in log.iterations])
    assert len(losses) == len(z["losses"])
    # fp32 trajectory stays close in the loss (chaotic dynamics bound it loosely)
    assert np.abs(losses - z["losses"]).max() <= 2e-2 * np.abs(z["losses"]).max()


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_self_registration_early_stop(request, prec):
    """test_pipeline.cpp:69-93: zero loss -> each scale exits after window+1."""
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    z = G.load("register_self.npz")
    g = A.GridMeta.make_3d(16, 16, 16)
    fld, log = ctx.register_images(g, z["fixed"], z["fixed"], A.RegistrationConfig(),
                                   A.PyramidSchedule())
    assert len(log.iterations) == 3 * 11
    assert [r.global_iter for r in log.iterations] == list(range(33))
    assert all(r.loss == 0.0 for r in log.iterations)
    assert log.iterations[-1].max_step == 0.0
    assert np.abs(fld).max() < 0.1
    assert log.final_loss < 1e-6


def test_default_early_stop_matches_reference(ctx64):
    """Default conv window/tol with LNCC: the stop iterations must agree."""
    z, g, sched = G.register_inputs("lncc")
    cfg = cfg_for("lncc", sched)
    cfg.conv_window, cfg.conv_tol = 5, 1e-3
    from oracle import pyoracle
    fa, la = ctx64.register_images(g, z["fixed"], z["moving"], cfg, sched)
    fb, lb = pyoracle.port().register_images(g, z["fixed"], z["moving"], cfg, sched)
    assert [(r.scale_index, r.iter) for r in la.iterations] == \
        [(r.scale_index, r.iter) for r in lb.iterations]
    assert np.abs(fa - fb).max() <= 1e-3


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_nonfinite_input_raises_numerical(request, prec):
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    g = A.GridMeta.make_3d(8, 8, 8)
    rng = np.random.default_rng(41)
    F, M = rng.random(g.shape), rng.random(g.shape)
    F[3, 2, 1] = np.nan
    with pytest.raises(A.NumericalError):
        ctx.register_images(g, F, M, A.RegistrationConfig(), A.PyramidSchedule((1.0,), (5,)))


def _textured_pair(seed):
    """noise phantom (like the reference's synth_phantom, synth.hpp:17-19) and a
    3-voxel smooth warp: strong gradients, so eta = 1000 folds the warp"""
    from scipy import ndimage
    g = A.GridMeta.make_3d(16, 16, 16)
    rng = np.random.default_rng(seed)
    M = ndimage.gaussian_filter(rng.random(g.shape), 1.0)
    M = (M - M.min()) / (M.max() - M.min())
    v = np.stack([ndimage.gaussian_filter(rng.standard_normal(g.shape), 3.0, mode="nearest")
                  for _ in range(3)], axis=-1)
    v *= 3.0 / np.abs(v).max()
    return g, synth.warp(M, synth.exp_velocity(v)), M


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_absurd_step_folds_and_raises(request, oracle_port, prec):
    """test_pipeline.cpp:191-199: eta = 1000 -> folded warp -> runtime_error."""
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    g, F, M = _textured_pair(51)
    cfg = A.RegistrationConfig(eta=1000.0)
    sched = A.PyramidSchedule((1.0,), (20,))
    with pytest.raises(A.NumericalError):
        oracle_port.register_images(g, F, M, cfg, sched)
    with pytest.raises(A.NumericalError, match="folded"):
        ctx.register_images(g, F, M, cfg, sched)


def test_zero_iterations_returns_init(ctx64):
    g = A.GridMeta.make_3d(12, 12, 12)
    rng = np.random.default_rng(5)
    F, M = rng.random(g.shape), rng.random(g.shape)
    init = np.zeros(g.field_shape)
    init[..., 0], init[..., 1], init[..., 2] = 0.3, -0.2, 0.1
    fld, log = ctx64.register_images(g, F, M, A.RegistrationConfig(),
                                     A.PyramidSchedule((1.0,), (0,)), init=(g, init))
    assert np.array_equal(fld, init)
    assert log.iterations == []
    T = A.AffineTransform(3, (1, 0, 0, 0, 1, 0, 0, 0, 1), (1.0, -0.5, 0.25))
    fld, _ = ctx64.register_images(g, F, M, A.RegistrationConfig(),
                                   A.PyramidSchedule((1.0,), (0,)), init=T)
    assert np.allclose(fld[..., 0], 1.0) and np.allclose(fld[..., 1], -0.5)


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_init_field_and_affine_match_oracle(request, oracle_port, prec):
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    p = synth.make_pair(0, seed=9, shape=(20, 20, 20), iters=(6, 4))
    sched = A.PyramidSchedule((2.0, 1.0), (6, 4))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=6)
    init_full = (p.grid, 0.3 * np.random.default_rng(1).normal(size=p.grid.field_shape))
    T = A.AffineTransform(3, (1.02, 0.01, 0, 0, 0.98, 0.02, 0, 0, 1.0), (0.5, -0.3, 0.2))
    for init in (init_full, T):
        a, la = ctx.register_images(p.grid, p.fixed, p.moving, cfg, sched, init=init)
        b, lb = oracle_port.register_images(p.grid, p.fixed, p.moving, cfg, sched, init=init)
        tol = 1e-6 if prec == "f64" else 5e-2
        assert np.abs(a - b).max() <= tol


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_2d_registration(request, oracle_port, prec):
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    g = A.GridMeta.make_2d(48, 40)
    rng = np.random.default_rng(71)
    from scipy import ndimage
    M = ndimage.gaussian_filter(rng.random((1, 40, 48)), (0, 2, 2))
    u = np.zeros(g.field_shape)
    u[..., 0] = 1.5 * np.sin(np.linspace(0, 3, 48))[None, None, :]
    F = oracle_port.warp_image(g, M, u)
    sched = A.PyramidSchedule((2.0, 1.0), (30, 20))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=30)
    fa, la = ctx.register_images(g, F, M, cfg, sched)
    fb, lb = oracle_port.register_images(g, F, M, cfg, sched)
    assert fa.shape == g.field_shape
    assert la.final_singularity_fraction == 0.0
    if prec == "f64":
        assert np.abs(fa - fb).max() <= 1e-3
    assert la.final_loss < la.iterations[0].loss


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_runs_are_bit_reproducible(request, prec):
    """test_pipeline.cpp:201-219 analogue: no float atomics -> replay identical."""
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    z, g, sched = G.register_inputs("lncc")
    cfg = cfg_for("lncc", sched)
    a, la = ctx.register_images(g, z["fixed"], z["moving"], cfg, sched)
    b, lb = ctx.register_images(g, z["fixed"], z["moving"], cfg, sched)
    assert np.array_equal(a, b)
    assert [r.loss for r in la.iterations] == [r.loss for r in lb.iterations]


def test_device_entry_point_matches_host_entry_point(ctx32):
    import torch
    z, g, sched = G.register_inputs("lncc")
    cfg = cfg_for("lncc", sched)
    a, la = ctx32.register_images(g, z["fixed"].astype(np.float32),
                                  z["moving"].astype(np.float32), cfg, sched,
                                  field_dtype=np.float32)
    F = torch.from_numpy(z["fixed"].astype(np.float32)).cuda()
    M = torch.from_numpy(z["moving"].astype(np.float32)).cuda()
    out = torch.empty((3,) + g.shape, dtype=torch.float32, device="cuda")
    torch.cuda.synchronize()
    lb = ctx32.register_device(g, F.data_ptr(), M.data_ptr(), cfg, sched, out.data_ptr())
    b = out.permute(1, 2, 3, 0).cpu().numpy()
    assert np.array_equal(a, b)
    assert [r.loss for r in la.iterations] == [r.loss for r in lb.iterations]


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_config1_full_size_properties(request, prec):
    """BASELINE config 1 at full size (the CPU oracle needs ~6 min for it): the
    size-independent properties — no folds, every iteration recorded, the
    full-resolution loss decreases, the label Dice improves over identity."""
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    p = synth.make_pair(1, seed=0)
    fld, log = ctx.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    assert log.final_singularity_fraction == 0.0
    assert len(log.iterations) == sum(p.schedule.iterations)
    ls = [r.loss for r in log.iterations if r.scale_index == 2]
    assert ls[-1] < ls[0]
    assert abs(log.final_loss - ls[-1]) < 1e-2
    from oracle import pyoracle
    o = pyoracle.port()
    w = o.warp_labels(p.grid, p.moving_labels, fld)
    d_after = o.overlap_dice(p.grid, w, p.fixed_labels)[0]
    d_before = o.overlap_dice(p.grid, p.moving_labels, p.fixed_labels)[0]
    assert d_after > d_before + 0.05, (d_before, d_after)


def test_config1_coarse_scales_match_reference(ctx64):
    """BASELINE config 1 shape through the reference's own pyramid (40x48x56 and
    80x96x112 scales, shortened schedule) plus the full-resolution epilogue."""
    from oracle import pyoracle
    o = pyoracle.best()
    p = synth.make_pair(1, seed=0)
    sched = A.PyramidSchedule((4.0, 2.0, 1.0), (12, 4, 0))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=12)
    fa, la = ctx64.register_images(p.grid, p.fixed, p.moving, cfg, sched)
    fb, lb = o.register_images(p.grid, p.fixed, p.moving, cfg, sched)
    a = np.array([r.loss for r in la.iterations])
    b = np.array([r.loss for r in lb.iterations])
    assert a.shape == b.shape
    assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b))
    assert np.abs(fa - fb).max() <= 1e-3
    assert abs(la.final_loss - lb.final_loss) <= 1e-4 * abs(lb.final_loss)


@pytest.mark.parametrize("name", ["lncc", "ssd"])
def test_use_jac_matches_reference_end_to_end(ctx64, ctx32, oracle_port, name):
    """eulerian_direction(use_jac = true) on the loop (diffeo.cpp:25-39,
    pipeline.cpp:184): v = -J(phi)^T grad applied inside the plane-streaming
    smooth+Adam.  fp64: every loss within 1e-4 relative, field within 1e-3
    voxel; fp32: warped-label Dice within 0.002."""
    z, g, sched = G.register_inputs(name)
    cfg = cfg_for(name, sched)
    cfg.use_jac = True
    fb, lb = oracle_port.register_images(g, z["fixed"], z["moving"], cfg, sched)
    fa, la = ctx64.register_images(g, z["fixed"], z["moving"], cfg, sched)
    a = np.array([r.loss for r in la.iterations])
    b = np.array([r.loss for r in lb.iterations])
    assert a.shape == b.shape
    assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b))
    assert np.abs(fa - fb).max() <= 1e-3
    f32, _ = ctx32.register_images(g, z["fixed"].astype(np.float32),
                                   z["moving"].astype(np.float32), cfg, sched)
    d32 = oracle_port.overlap_dice(g, oracle_port.warp_labels(g, z["moving_labels"], f32),
                                   z["fixed_labels"])[0]
    dref = oracle_port.overlap_dice(g, oracle_port.warp_labels(g, z["moving_labels"], fb),
                                    z["fixed_labels"])[0]
    assert abs(d32 - dref) <= 0.002, (d32, dref)
    # and it differs from the Jacobian-free run (the option is not ignored)
    cfg.use_jac = False
    fn, _ = ctx64.register_images(g, z["fixed"], z["moving"], cfg, sched)
    assert np.abs(fn - fa).max() > 1e-6
