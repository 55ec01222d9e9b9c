"""Large volumes (> 2^28 voxels): the 1-D helper kernels (pyramid blur,
resample, warp, Jacobian) once capped their grids at 2^20 CTAs, silently
skipping voxels beyond 268M (found running BASELINE config 4 at 1024^3).
A 672^3 (303M voxels) config-4-recipe pair must register without non-finite
steps or folds, and 4 emulated z-slabs must reproduce it bit for bit."""
import pytest

from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context, register_slab

pytestmark = pytest.mark.gpu


def test_303M_voxels_register_and_slabs_match():
    import torch
    from paper_2404_01249_b200.synth_gpu import make_config4_pair
    n = 672  # 303M voxels; every level's x extent a multiple of 16 bytes (slab path)
    fixed, moving = make_config4_pair("cuda", seed=1, shape=(n, n, n), n_puncta=50_000)
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    g = A.GridMeta.make_3d(n, n, n)
    sched = A.PyramidSchedule((8.0, 4.0, 2.0, 1.0), (6, 4, 2, 2))
    cfg = synth.baseline_config(A.LOSS_LNCC, 3, 1.0, max_iters=6)
    out = torch.empty((3, n, n, n), dtype=torch.float32, device="cuda")
    ctx = Context(0, "f32")
    log = ctx.register_device(g, fixed.data_ptr(), moving.data_ptr(), cfg, sched, out.data_ptr())
    ctx.close()
    assert log.final_singularity_fraction == 0.0
    assert len(log.iterations) == 14
    assert bool(torch.isfinite(out).all())
    # the far end of the volume (beyond voxel 2^28) was actually updated
    assert float(out[:, -8:].abs().max()) > 0.0
    ctx = Context(0, "f32")
    out2 = torch.empty_like(out)
    register_slab(ctx, g, fixed.data_ptr(), moving.data_ptr(), cfg, sched, emulate=4,
                  d_out=out2.data_ptr())
    ctx.close()
    assert torch.equal(out, out2)
