"""The kernel families of the hot loop — brick kernels (small pyramid levels,
either one persistent cooperative launch per level or one CUDA graph per
iteration) and plane-streaming TMA kernels (large levels) — each held to the
reference on the same inputs (DFM_OPT_BRICK_MAX / DFM_OPT_PERSIST force one
family for every level).

fp64: every iteration loss within 1e-4 relative, final field within 1e-3
voxel (BASELINE north_star); fp32: warped-label Dice within 0.002.
"""
import numpy as np
import pytest

import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import (Context, OPT_BRICK_MAX, OPT_NARROW, OPT_PERSIST,
                                          OPT_SPLIT, OPT_SPLIT_FOLD_MAX)

pytestmark = pytest.mark.gpu

FAMILIES = {"persist": (1 << 40, 1), "persist_nb": (1 << 40, 3), "brick": (1 << 40, 0),
            "stream": (0, 0)}


def _ctx(prec, family):
    c = Context(0, prec)
    bm, pe = FAMILIES[family]
    c.set_option(OPT_BRICK_MAX, bm)
    c.set_option(OPT_PERSIST, pe)
    return c


def _cfg(name, sched):
    loss = A.LOSS_LNCC if name == "lncc" else A.LOSS_SSD
    return synth.baseline_config(loss, 2, 1.0, max_iters=max(sched.iterations))


@pytest.mark.parametrize("family", list(FAMILIES))
@pytest.mark.parametrize("name", ["lncc", "ssd"])
def test_fp64_family_matches_reference(family, name):
    z, g, sched = G.register_inputs(name)
    ctx = _ctx("f64", family)
    fld, log = ctx.register_images(g, z["fixed"], z["moving"], _cfg(name, sched), sched)
    ctx.close()
    losses = np.array([r.loss for r in log.iterations])
    assert len(losses) == len(z["losses"])
    assert np.all(np.abs(losses - z["losses"]) <= 1e-4 * np.abs(z["losses"]))
    assert np.abs(fld - z["field"]).max() <= 1e-3
    ms = np.array([r.max_step for r in log.iterations])
    assert np.allclose(ms, z["max_steps"], rtol=1e-6, atol=1e-9)


@pytest.mark.parametrize("family", list(FAMILIES))
def test_fp32_family_dice(family, oracle_port):
    z, g, sched = G.register_inputs("lncc")
    ctx = _ctx("f32", family)
    fld, log = ctx.register_images(g, z["fixed"].astype(np.float32),
                                   z["moving"].astype(np.float32), _cfg("lncc", sched), sched)
    ctx.close()
    assert log.final_singularity_fraction == 0.0
    w_gpu = oracle_port.warp_labels(g, z["moving_labels"], fld)
    w_ref = oracle_port.warp_labels(g, z["moving_labels"], z["field"])
    d_gpu = oracle_port.overlap_dice(g, w_gpu, z["fixed_labels"])[0]
    d_ref = oracle_port.overlap_dice(g, w_ref, z["fixed_labels"])[0]
    assert abs(d_gpu - d_ref) <= 0.002, (d_gpu, d_ref)


@pytest.mark.parametrize("shape,r", [((21, 18, 13), 1), ((24, 20, 17), 3), ((37, 9, 11), 2)])
def test_ragged_shapes_both_families_agree(shape, r, oracle_port):
    """Shapes that are not multiples of the 8^3 brick (partial bricks on every
    face) and LNCC radii 1..3: both families against the fp64 reference."""
    rng = np.random.default_rng(sum(shape) + r)
    g = A.GridMeta(3, shape)
    n = int(np.prod(shape))
    x = np.linspace(0, 1, n).reshape(shape[::-1])
    fixed = (0.5 + 0.3 * np.sin(7 * x) + 0.05 * rng.standard_normal(shape[::-1])).ravel()
    moving = (0.5 + 0.3 * np.sin(7 * x + 0.2) + 0.05 * rng.standard_normal(shape[::-1])).ravel()
    sched = A.PyramidSchedule((1.0,), (6,))
    cfg = synth.baseline_config(A.LOSS_LNCC, r, 1.0, max_iters=6)
    fr, lr = oracle_port.register_images(g, fixed, moving, cfg, sched)
    for family in FAMILIES:
        ctx = _ctx("f64", family)
        f, log = ctx.register_images(g, fixed, moving, cfg, sched)
        ctx.close()
        a = np.array([q.loss for q in log.iterations])
        b = np.array([q.loss for q in lr.iterations])
        assert a.shape == b.shape, family
        assert np.all(np.abs(a - b) <= 1e-4 * np.abs(b)), family
        assert np.abs(f - fr).max() <= 1e-3, family


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_persistent_solver_early_stop_and_replay(prec):
    """The persistent solver's device-side monitor: default early stopping gives
    the same record count and losses as the graph path, and reruns are
    bit-identical."""
    p = synth.make_pair(0, seed=3, shape=(40, 48, 56), iters=(30, 20, 10))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, conv_window=5)
    cfg.conv_tol = 1e-2
    runs = {}
    for family in ("persist", "brick"):
        ctx = _ctx(prec, family)
        a = ctx.register_images(p.grid, p.fixed, p.moving, cfg, p.schedule)
        b = ctx.register_images(p.grid, p.fixed, p.moving, cfg, p.schedule)
        ctx.close()
        assert np.array_equal(a[0], b[0]), family
        runs[family] = a
    la = [r.loss for r in runs["persist"][1].iterations]
    lb = [r.loss for r in runs["brick"][1].iterations]
    assert len(la) == len(lb) < sum(p.schedule.iterations)
    assert np.allclose(la, lb, rtol=1e-12 if prec == "f64" else 1e-5)


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_update_variants_bit_identical(prec):
    """The fused compose+smooth kernel, the split update with the compose folded
    into smooth+Adam, and the split update with a separate radius-0 compose
    kernel produce the same bits (stream family, every level)."""
    z, g, sched = G.register_inputs("lncc")
    fields = []
    for split, fold_max in ((0, 0), (1, 1 << 40), (1, 0)):
        ctx = Context(0, prec)
        ctx.set_option(OPT_BRICK_MAX, 0)
        ctx.set_option(OPT_SPLIT, split)
        ctx.set_option(OPT_SPLIT_FOLD_MAX, fold_max)
        f, log = ctx.register_images(g, z["fixed"], z["moving"], _cfg("lncc", sched), sched)
        ctx.close()
        fields.append((f, [r.loss for r in log.iterations]))
    for f, ls in fields[1:]:
        assert np.array_equal(f, fields[0][0])
        assert ls == fields[0][1]


@pytest.mark.parametrize("prec,split,fold_max", [("f32", 1, 1 << 40), ("f64", 1, 1 << 40),
                                                 ("f32", 1, 0), ("f32", 0, 0)])
def test_narrow_tiles_match_wide(prec, split, fold_max):
    """DFM_OPT_NARROW: an 80-column level on 16-wide z-march tiles gives the
    field of the 32-wide tiles bit for bit (the per-voxel arithmetic is the
    same; only the loss's block partial sums are grouped differently), with the
    folded, separate (radius-0 staged) and fused compose forms."""
    p = synth.make_pair(1, seed=7, shape=(56, 48, 80))
    sched = A.PyramidSchedule((1.0,), (6,))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=6)
    cfg.eta = 0.2
    out = []
    for narrow in (0, 1):
        ctx = Context(0, prec)
        ctx.set_option(OPT_BRICK_MAX, 0)
        ctx.set_option(OPT_SPLIT, split)
        ctx.set_option(OPT_SPLIT_FOLD_MAX, fold_max)
        ctx.set_option(OPT_NARROW, narrow)
        f, log = ctx.register_images(p.grid, p.fixed, p.moving, cfg, sched)
        ctx.close()
        out.append((f, np.array([r.loss for r in log.iterations])))
    assert np.array_equal(out[0][0], out[1][0])
    assert np.allclose(out[0][1], out[1][1], rtol=1e-12, atol=0)


def test_set_option_rejects_unknown_key():
    ctx = Context(0, "f32")
    with pytest.raises(ValueError):
        ctx.set_option(99, 1)
    with pytest.raises(ValueError):
        ctx.set_option(OPT_BRICK_MAX, -1)
    ctx.close()
