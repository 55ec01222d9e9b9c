"""Pins the plain-C restatement (oracle/difform_oracle.c) to the reference.

Golden vectors come from the unmodified reference compiled from its own
sources (tests/golden/make_golden.py); the restatement must reproduce them
BIT-FOR-BIT (same fp64 operation order, same 4096-block ordered sums).  When
oracle/_ref is present (built in the container that has /root/reference) the
restatement is also cross-checked live on fresh random inputs.
"""
import numpy as np
import pytest

import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth


@pytest.mark.parametrize("tag", ["3d", "2d"])
def test_restatement_matches_golden_bitwise(oracle_port, tag):
    bad = []
    for key, (got, want) in G.compute(oracle_port, tag).items():
        if not np.array_equal(np.asarray(got, dtype=want.dtype), want):
            bad.append(key)
    assert not bad, f"restatement differs from the reference golden vectors: {bad}"


def test_restatement_own_grid_bitwise(oracle_port):
    for key, (got, want) in G.compute_own_grid(oracle_port).items():
        assert np.array_equal(got, want), key


@pytest.mark.parametrize("name", ["lncc", "ssd"])
def test_restatement_register_bitwise(oracle_port, name):
    z, g, sched = G.register_inputs(name)
    loss = A.LOSS_LNCC if name == "lncc" else A.LOSS_SSD
    cfg = synth.baseline_config(loss, 2, 1.0, max_iters=max(sched.iterations))
    fld, log = oracle_port.register_images(g, z["fixed"], z["moving"], cfg, sched)
    assert np.array_equal(fld, z["field"])
    assert np.array_equal([r.loss for r in log.iterations], z["losses"])
    assert np.array_equal([r.max_step for r in log.iterations], z["max_steps"])
    assert log.final_loss == float(z["final_loss"])


@pytest.mark.parametrize("tag", ["3d", "2d"])
def test_restatement_svf_bitwise(oracle_port, tag):
    """exp_map / svf_pullback (diffeo.cpp:66-167): scaling and squaring and its
    discrete adjoint with the serial lerp-weight scatter, M in {0, 1, 4, 6}."""
    for key, (got, want) in G.compute_svf(oracle_port, tag).items():
        assert np.array_equal(got, want), key


@pytest.mark.parametrize("name", ["svf_lncc", "svf_ssd"])
def test_restatement_register_svf_bitwise(oracle_port, name):
    """SVF mode of register_images (pipeline.cpp:166-167, 189-206, 213-215)."""
    z, g, sched = G.register_inputs(name)
    cfg = G.register_config(name, z, sched)
    fld, log = oracle_port.register_images(g, z["fixed"], z["moving"], cfg, sched)
    assert np.array_equal(fld, z["field"])
    assert np.array_equal([r.loss for r in log.iterations], z["losses"])
    assert np.array_equal([r.max_step for r in log.iterations], z["max_steps"])
    assert log.final_loss == float(z["final_loss"])


@pytest.mark.parametrize("tag", ["3d", "2d"])
def test_restatement_affine_bitwise(oracle_port, tag):
    """affine_to_field / affine_param_gradient (affine.cpp:50-122), 3 losses."""
    for key, (got, want) in G.compute_affine(oracle_port, tag).items():
        assert np.array_equal(got, want), key


@pytest.mark.parametrize("loss", [A.LOSS_SSD, A.LOSS_LNCC])
def test_restatement_affine_register_bitwise(oracle_port, loss):
    """affine_register (affine.cpp:124-183): multi-scale parameter Adam."""
    z, g = G.affine_register_inputs()
    r = oracle_port.affine_register(g, z["reg_fixed"], z["reg_moving"], loss, [4, 2, 1],
                                    [40, 20, 10], 0.01)
    assert np.array_equal(r["A"], z[f"reg{loss}_A"])
    assert np.array_equal(r["t"], z[f"reg{loss}_t"])
    assert r["loss"] == float(z[f"reg{loss}_loss"])
    assert r["iterations"] == int(z[f"reg{loss}_iterations"])


def test_restatement_affine_errors(oracle_port):
    g = A.GridMeta.make_3d(12, 12, 12)
    F = np.zeros(g.shape)
    with pytest.raises(A.InvalidArgument):
        oracle_port.affine_register(g, F, F, A.LOSS_SSD, [], [], 0.1)
    # eta so large that A collapses / the loss stays finite: |det A| < 1e-3 -> runtime_error
    rng = np.random.default_rng(0)
    F = rng.random(g.shape)
    M = np.roll(F, 2, axis=0)
    try:
        r = oracle_port.affine_register(g, F, M, A.LOSS_SSD, [1], [40], 50.0)
        assert r["diverged"] or abs(np.linalg.det(r["A"])) >= 1e-3
    except A.NumericalError:
        pass


def test_restatement_overlap_and_landmarks_bitwise(oracle_port):
    """overlap_report (analysis.cpp:169-247) incl. negative / one-sided labels,
    and landmark_error (249-283) on grids with spacing and origin."""
    z, gf, gm = G.eval_inputs()
    r = oracle_port.overlap_report(gf, z["lab_w"], z["lab_f"])
    for k, v in r.items():
        if k != "regions":
            assert v == float(z[f"ov_{k}"]), k
    assert np.array_equal(G.region_rows(r), z["ov_regions"])
    dist, mean, mx = oracle_port.landmark_error(gf, gm, z["phi"], z["fixed_mm"], z["moving_mm"])
    assert np.array_equal(dist, z["lm_dist"])
    assert mean == float(z["lm_mean"]) and mx == float(z["lm_max"])


def test_restatement_early_stop_record_count(oracle_port):
    """test_pipeline.cpp:69-93 semantics: default window 10 on a self pair."""
    z = G.load("register_self.npz")
    g = A.GridMeta.make_3d(16, 16, 16)
    fld, log = oracle_port.register_images(g, z["fixed"], z["fixed"], A.RegistrationConfig(),
                                           A.PyramidSchedule())
    assert np.array_equal([r.loss for r in log.iterations], z["losses"])
    assert len(log.iterations) == 3 * 11
    assert all(r.loss == 0.0 for r in log.iterations)
    assert np.abs(fld).max() < 0.1


def test_restatement_errors(oracle_port):
    g = A.GridMeta.make_3d(8, 8, 8)
    rng = np.random.default_rng(0)
    F = rng.random(g.shape)
    M = rng.random(g.shape)
    phi = np.zeros(g.field_shape)
    with pytest.raises(A.InvalidArgument):
        oracle_port.lncc_eval(g, F, phi, M, 4)          # window 9 > 8
    with pytest.raises(A.InvalidArgument):
        oracle_port.lncc_eval(g, F, phi, M, 0)
    bad = F.copy()
    bad[1, 2, 3] = np.nan
    with pytest.raises(A.NumericalError):                # test_pipeline.cpp:183-189
        oracle_port.register_images(g, bad, M, A.RegistrationConfig(),
                                    A.PyramidSchedule((1.0,), (5,)))
    with pytest.raises(A.NumericalError):
        oracle_port.apply_update(g, phi, np.full(g.field_shape, np.inf), 0.5, 0.5)
    with pytest.raises(A.InvalidArgument):
        oracle_port.upsample_field(g, phi, A.GridMeta.make_3d(4, 8, 8))


def test_restatement_live_vs_reference(oracle_port):
    from oracle import pyoracle
    if not pyoracle.reference_available():
        pytest.skip("oracle/_ref not built here")
    ref = pyoracle.reference()
    rng = np.random.default_rng(99)
    for dims in ((7, 9, 6), (33, 5, 12)):
        g = A.GridMeta.make_3d(*dims)
        F, M = rng.random(g.shape), rng.random(g.shape)
        phi = rng.normal(0, 2.0, g.field_shape)
        for r in (1, 2):
            a = oracle_port.lncc_eval(g, F, phi, M, r)
            b = ref.lncc_eval(g, F, phi, M, r)
            assert a[0] == b[0] and np.array_equal(a[1], b[1])
        assert np.array_equal(oracle_port.apply_update(g, phi, phi, 0.7, 0.8),
                              ref.apply_update(g, phi, phi, 0.7, 0.8))
