import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2404_01249_b200 import synth, _abi as A
from paper_2404_01249_b200.engine import Context
prec = sys.argv[1]
os.environ["DFM_FORCE_LEGACY"] = "1"
ctx_l = Context(0, prec)
del os.environ["DFM_FORCE_LEGACY"]
p = synth.make_pair(0, seed=7, shape=(24, 24, 24))
cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=2)
sched = A.PyramidSchedule((1.0,), (2,))
cfg.eta = 0.05
fl, ll = ctx_l.register_images(p.grid, p.fixed, p.moving, cfg, sched)
for mask in (0, 1, 2, 3, 4, 8, 15):
    os.environ["DFM_TMA_MASK"] = str(mask)
    c = Context(0, prec)
    try:
        ft, lt = c.register_images(p.grid, p.fixed, p.moving, cfg, sched)
        print(prec, "mask", mask, "max|du|", np.abs(ft - fl).max(), [r.loss for r in lt.iterations], [r.loss for r in ll.iterations], [r.max_step for r in lt.iterations])
    except Exception as e:
        print(prec, "mask", mask, "ERR", e)
    c.close()
