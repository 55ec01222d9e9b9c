"""use_jac diagnosis: GPU m after iterations 1, 2 vs the oracle (stream, legacy)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np
import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context, OPT_FORCE_LEGACY
from oracle import pyoracle
o = pyoracle.port()
z, g, sched = G.register_inputs("lncc")
cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=30)
cfg.use_jac = True
for legacy in (0, 1):
    ctx = Context(0, "f64"); ctx.set_option(OPT_FORCE_LEGACY, legacy)
    for it in (1, 2, 3):
        s = A.PyramidSchedule((1.0,), (it,))
        try:
            fa, la = ctx.register_images(g, z["fixed"], z["moving"], cfg, s)
        except Exception as e:
            print("legacy", legacy, it, "GPU ERR", e); continue
        fb, lb = o.register_images(g, z["fixed"], z["moving"], cfg, s)
        print("legacy", legacy, "iters", it, "field maxdiff", np.abs(fa - fb).max(),
              "loss diffs", [a.loss - b.loss for a, b in zip(la.iterations, lb.iterations)])
    for sc in ((4.0, 2.0, 1.0),):
        try:
            fa, la = ctx.register_images(g, z["fixed"], z["moving"], cfg, sched)
            fb, lb = o.register_images(g, z["fixed"], z["moving"], cfg, sched)
            print("legacy", legacy, "full sched maxdiff", np.abs(fa - fb).max())
        except Exception as e:
            print("legacy", legacy, "full sched ERR", e)
