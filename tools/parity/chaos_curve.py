"""Loss-difference curves of the fp64 context vs the reference (configs 0, 1)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
from paper_2404_01249_b200 import synth
from paper_2404_01249_b200.engine import Context
from oracle import pyoracle
out = {}
ctx = Context(0, "f64")
p = synth.make_pair(0, seed=0)
fa, la = ctx.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
fb, lb = pyoracle.best().register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
out["c0_gpu"] = np.array([r.loss for r in la.iterations]); out["c0_ref"] = np.array([r.loss for r in lb.iterations])
out["c0_field_maxdiff"] = np.abs(fa - fb).max()
p = synth.make_pair(1, seed=0)
fa, la = ctx.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
out["c1_gpu"] = np.array([r.loss for r in la.iterations])
os.makedirs("gpurun_out", exist_ok=True)
np.savez("gpurun_out/chaos.npz", **out)
print("ok", out["c0_field_maxdiff"])
