"""z-slab decomposition on one GPU: the volume is split into
2-4 emulated slabs exchanging halo planes by device copies — the same kernels
and exchange plan the NCCL path runs across GPUs.  Every voxel's arithmetic is
identical to the monolithic run, so the fields must be BIT-identical and the
loss log equal up to the summation order of the loss partials."""
import numpy as np
import pytest

from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import (Context, OPT_BRICK_MAX, OPT_SLAB_OVERLAP,
                                          OPT_SLAB_REPL_MAX, register_slab)

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["f32", "f64"])
@pytest.mark.parametrize("slabs,repl,overlap", [(2, 0, 0), (3, 0, 1), (4, 0, 0), (4, 20000, 1)])
def test_emulated_slabs_match_monolithic(prec, slabs, repl, overlap):
    """repl 0: every level decomposed; repl 20000: the coarsest level (16 x 10
    x 12) replicated, the finer ones decomposed (DFM_OPT_SLAB_REPL_MAX);
    overlap 1: boundary planes first, exchange on a second stream beside the
    interior planes (DFM_OPT_SLAB_OVERLAP)."""
    import torch
    # the slab path runs the plane-streaming kernels: so does the monolithic
    # reference run here (the brick family sums in another order)
    ctx = Context(0, prec)
    ctx.set_option(OPT_BRICK_MAX, 0)
    ctx.set_option(OPT_SLAB_REPL_MAX, repl)
    ctx.set_option(OPT_SLAB_OVERLAP, overlap)
    p = synth.make_pair(0, seed=5, shape=(64, 40, 48))   # z, y, x
    g = p.grid
    sched = A.PyramidSchedule((4.0, 2.0, 1.0), (12, 8, 4))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=12)
    dt = torch.float32 if prec == "f32" else torch.float64
    F = torch.from_numpy(p.fixed).cuda().to(dt)
    M = torch.from_numpy(p.moving).cuda().to(dt)
    a = torch.empty((3,) + g.shape, dtype=dt, device="cuda")
    b = torch.empty_like(a)
    torch.cuda.synchronize()
    la = ctx.register_device(g, F.data_ptr(), M.data_ptr(), cfg, sched, a.data_ptr())
    zlo, zhi, lb = register_slab(ctx, g, F.data_ptr(), M.data_ptr(), cfg, sched,
                                 emulate=slabs, d_out=b.data_ptr())
    assert (zlo, zhi) == (0, g.dims[2])
    assert torch.equal(a, b), float((a - b).abs().max())
    x = np.array([r.loss for r in la.iterations])
    y = np.array([r.loss for r in lb.iterations])
    assert x.shape == y.shape
    assert np.allclose(x, y, rtol=1e-12, atol=0)
    assert abs(la.final_loss - lb.final_loss) <= 1e-12 * abs(la.final_loss)
    assert lb.final_singularity_fraction == la.final_singularity_fraction
    ctx.close()


def test_slab_rejects_too_many_slabs(ctx32):
    import torch
    p = synth.make_pair(0, seed=5, shape=(16, 16, 16))
    F = torch.from_numpy(p.fixed).cuda()
    M = torch.from_numpy(p.moving).cuda()
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=2)
    with pytest.raises(A.InvalidArgument):
        register_slab(ctx32, p.grid, F.data_ptr(), M.data_ptr(), cfg,
                      A.PyramidSchedule((1.0,), (2,)), emulate=8)
