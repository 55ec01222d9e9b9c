"""Affine pre-alignment on the device: affine_to_field,
affine_param_gradient and affine_register (affine.cpp:50-183) against the
reference's golden vectors, plus the hand-off into register_images through
RegInit = AffineTransform.

Tolerances: fp64 within 1e-9 relative to each output's peak (the 12 parameter
sums use a different, fixed, reduction order); fp32 1e-4 relative to peak for
the 12 sums over ~10^3 voxels.  affine_register in fp64: the optimiser path
(Adam on 12 parameters, 70 iterations) is held to 1e-6 on A and t and 1e-8
relative on the best loss.
"""
import numpy as np
import pytest

import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["f64", "f32"])
@pytest.mark.parametrize("tag", ["3d", "2d"])
def test_affine_kernels_match_reference(request, prec, tag):
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    rel = 1e-9 if prec == "f64" else 1e-4
    for key, (got, want) in G.compute_affine(ctx, tag).items():
        peak = float(np.abs(want).max()) or 1.0
        err = float(np.abs(np.asarray(got) - want).max())
        assert err <= rel * peak, (key, err, peak)


@pytest.mark.parametrize("loss", [A.LOSS_SSD, A.LOSS_LNCC])
def test_fp64_affine_register_matches_reference(ctx64, loss):
    z, g = G.affine_register_inputs()
    r = ctx64.affine_register(g, z["reg_fixed"], z["reg_moving"], loss, [4, 2, 1],
                              [40, 20, 10], 0.01)
    assert r["iterations"] == int(z[f"reg{loss}_iterations"])
    assert not r["diverged"]
    assert np.abs(r["A"] - z[f"reg{loss}_A"]).max() <= 1e-6
    assert np.abs(r["t"] - z[f"reg{loss}_t"]).max() <= 1e-6
    want = float(z[f"reg{loss}_loss"])
    assert abs(r["loss"] - want) <= 1e-8 * max(abs(want), 1e-12) + 1e-15


def test_fp32_affine_register_recovers_transform(ctx32):
    """fp32: the recovered transform agrees with the reference's within the
    accuracy the optimiser itself reaches (1e-2 on A entries, 0.1 voxel on t)."""
    z, g = G.affine_register_inputs()
    r = ctx32.affine_register(g, z["reg_fixed"], z["reg_moving"], A.LOSS_LNCC, [4, 2, 1],
                              [40, 20, 10], 0.01)
    assert np.abs(r["A"] - z[f"reg{A.LOSS_LNCC}_A"]).max() <= 1e-2
    assert np.abs(r["t"] - z[f"reg{A.LOSS_LNCC}_t"]).max() <= 0.1


def test_affine_then_diffeomorphic_matches_reference(ctx64, oracle_port):
    """The paper's pipeline: affine pre-alignment, then register_images seeded
    with the affine transform (RegInit) — both stages vs the restatement."""
    z, g = G.affine_register_inputs()
    F, M = z["reg_fixed"], z["reg_moving"]
    ra = ctx64.affine_register(g, F, M, A.LOSS_LNCC, [4, 2], [20, 10], 0.01)
    rb = oracle_port.affine_register(g, F, M, A.LOSS_LNCC, [4, 2], [20, 10], 0.01)
    assert np.abs(ra["A"] - rb["A"]).max() <= 1e-6
    init = A.AffineTransform(3, tuple(rb["A"].ravel()), tuple(rb["t"]))
    sched = A.PyramidSchedule((2.0, 1.0), (10, 5))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=10)
    fa, la = ctx64.register_images(g, F, M, cfg, sched, init=init)
    fb, lb = oracle_port.register_images(g, F, M, cfg, sched, init=init)
    a = np.array([r.loss for r in la.iterations])
    b = np.array([r.loss for r in lb.iterations])
    assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b))
    assert np.abs(fa - fb).max() <= 1e-3


def test_affine_errors_map_to_reference_exceptions(ctx32):
    g = A.GridMeta.make_3d(12, 12, 12)
    F = np.zeros(g.shape)
    with pytest.raises(A.InvalidArgument):
        ctx32.affine_register(g, F, F, A.LOSS_SSD, [], [], 0.1)
    with pytest.raises(A.InvalidArgument):  # window 2*6+1 > 12
        ctx32.affine_param_gradient(g, F, F, A.LOSS_LNCC, np.eye(3), np.zeros(3),
                                    lncc_radius=6)
    with pytest.raises(A.InvalidArgument):  # dice needs masks in [0, 1]
        ctx32.affine_param_gradient(g, F + 2.0, F, A.LOSS_DICE, np.eye(3), np.zeros(3))
