"""How far is the fp64 context from bit-identical dynamics?  Field after k
iterations (GPU fp64 vs the reference), counting differing elements."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context, OPT_BRICK_MAX
from oracle import pyoracle
o = pyoracle.best()
p = synth.make_pair(1, seed=0)
q = synth.make_pair(1, seed=0, shape=(56, 48, 40))
cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=10)
for fam, bm in (("brick", 1 << 40), ("stream", 0)):
    ctx = Context(0, "f64"); ctx.set_option(OPT_BRICK_MAX, bm)
    for name, pp, sc in (("direct40", q, 1.0), ("pyr4", p, 4.0)):
        for k in (0, 1, 2, 5):
            s = A.PyramidSchedule((sc,), (k,))
            try:
                fa, la = ctx.register_images(pp.grid, pp.fixed, pp.moving, cfg, s)
                fb, lb = o.register_images(pp.grid, pp.fixed, pp.moving, cfg, s)
            except A.NumericalError as e:
                print(fam, name, k, "error", e); continue
            d = np.abs(fa - fb)
            ls = [(a.loss - b.loss) for a, b in zip(la.iterations, lb.iterations)]
            print(f"{fam:6s} {name:8s} k={k}: field maxdiff {d.max():.3e} ndiff {(d > 0).sum()}/{d.size} "
                  f"final loss diff {la.final_loss - lb.final_loss:.3e} loss diffs {ls}", flush=True)
    ctx.close()
