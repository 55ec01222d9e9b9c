"""A/B the TMA loop kernels against the legacy kernels on small registrations."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2404_01249_b200 import synth, _abi as A
from paper_2404_01249_b200.engine import Context
prec = sys.argv[1] if len(sys.argv) > 1 else "f64"
ctx_t = Context(0, prec)
os.environ["DFM_FORCE_LEGACY"] = "1"
ctx_l = Context(0, prec)
for shape, its, sig in [((24, 24, 24), 1, 1.0), ((24, 24, 24), 2, 1.0), ((32, 32, 32), 1, 1.0), ((32, 32, 32), 1, 0.0), ((32,32,32), 2, 0.0)]:
    p = synth.make_pair(0, seed=7, shape=shape)
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, sig, max_iters=its)
    sched = A.PyramidSchedule((1.0,), (its,))
    ft, lt = ctx_t.register_images(p.grid, p.fixed, p.moving, cfg, sched)
    fl, ll = ctx_l.register_images(p.grid, p.fixed, p.moving, cfg, sched)
    d = np.abs(ft - fl)
    print(shape, its, "sigma_g", sig, "max|du|", d.max(), "at", np.unravel_index(d.argmax(), d.shape),
          "losses", [r.loss for r in lt.iterations], [r.loss for r in ll.iterations],
          "maxstep", [r.max_step for r in lt.iterations], [r.max_step for r in ll.iterations])
