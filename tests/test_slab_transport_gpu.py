"""The z-slab data plane between PROCESSES: two ranks on one
GPU run dfm_dev_register_slab_tp — the world > 1 call sequence with
rank-local slab views, every collective (halo exchange of coefficients,
gradient, composed field, u and W; the loss all-reduce feeding the global
convergence monitor; the non-finite-step flag; the gather at scale changes;
the fold count) host-staged over torch.distributed gloo.  The owned planes of
the two ranks must be BIT-identical to the monolithic registration, the
losses equal up to the summation order of their partials."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
pytestmark = pytest.mark.gpu


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("prec,repl", [("f32", 0), ("f64", 0), ("f32", 20000)])
def test_two_processes_match_monolithic(tmp_path, prec, repl):
    import torch
    sys.path.insert(0, HERE)
    import slab_worker
    from paper_2404_01249_b200.engine import Context, OPT_BRICK_MAX
    world, port = 2, _port()
    procs = [subprocess.Popen([sys.executable, os.path.join(HERE, "slab_worker.py"), str(r),
                               str(world), str(port), str(tmp_path), prec, str(repl)],
                              stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
             for r in range(world)]
    outs = [q.communicate(timeout=600)[0] for q in procs]
    for q, o in zip(procs, outs):
        assert q.returncode == 0, o
    p, sched, cfg = slab_worker.case()
    g = p.grid
    dt = torch.float32 if prec == "f32" else torch.float64
    ctx = Context(0, prec)
    ctx.set_option(OPT_BRICK_MAX, 0)  # the plane-streaming family, as the slabs run
    F = torch.from_numpy(p.fixed).cuda().to(dt)
    M = torch.from_numpy(p.moving).cuda().to(dt)
    ref = torch.empty((3,) + g.shape, dtype=dt, device="cuda")
    torch.cuda.synchronize()
    lref = ctx.register_device(g, F.data_ptr(), M.data_ptr(), cfg, sched, ref.data_ptr())
    ref = ref.reshape(3, -1).cpu().numpy()
    ctx.close()
    pl = g.dims[0] * g.dims[1]
    covered = 0
    for r in range(world):
        z = np.load(os.path.join(str(tmp_path), f"rank{r}.npz"))
        zlo, zhi = int(z["zlo"]), int(z["zhi"])
        assert np.array_equal(z["field"], ref[:, zlo * pl:zhi * pl]), r
        a = np.array([q.loss for q in lref.iterations])
        assert z["losses"].shape == a.shape
        assert np.allclose(z["losses"], a, rtol=1e-12, atol=0)
        assert abs(float(z["final_loss"]) - lref.final_loss) <= 1e-12 * abs(lref.final_loss)
        assert float(z["sing"]) == lref.final_singularity_fraction
        assert int(z["launches"]) > 0
        covered += zhi - zlo
    assert covered == g.dims[2]
