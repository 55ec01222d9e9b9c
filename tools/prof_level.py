"""One registration at a single pyramid level (scale 1, `iters` iterations) of
the config-1 phantom resampled to NX x NY x NZ — the launches ncu should see
are all of that level.   python tools/prof_level.py NX NY NZ [iters] [f32|f64]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01249_b200 import _abi as A, synth  # noqa: E402
from paper_2404_01249_b200.engine import Context  # noqa: E402

nx, ny, nz = (int(v) for v in sys.argv[1:4])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 4
prec = sys.argv[5] if len(sys.argv) > 5 else "f32"
p = synth.make_pair(1, seed=0, shape=(nz, ny, nx))
cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=iters)
ctx = Context(0, prec)
try:
    ctx.register_images(p.grid, p.fixed, p.moving, cfg, A.PyramidSchedule((1.0,), (iters,)))
except A.NumericalError as e:  # a single level from identity may fold: launches still stand
    print("note:", e)
print("ok", ctx.launch_count)
