"""Per-iteration device time of one pyramid level in the production (graph)
path, for a list of volume sizes:  python tools/level_iter_time.py NXxNYxNZ ...
(one registration at scale 1 with 64 iterations per size, early stop off;
median IterationRecord.wall_ms, i.e. graph-chunk device time / iterations).
LIT_PERSIST=0/1/2 and LIT_BRICK_MAX select the brick solver (persistent
levels stamp each iteration's record on the device); LIT_OPTS="key=value,..."
sets any further dfm_ctx_set_option keys (numbers, include/difform_gpu.h)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_2404_01249_b200 import _abi as A, synth  # noqa: E402
from paper_2404_01249_b200.engine import Context, OPT_BRICK_MAX, OPT_PERSIST  # noqa: E402

iters = int(os.environ.get("LIT_ITERS", "64"))
for spec in sys.argv[1:]:
    nx, ny, nz = (int(v) for v in spec.split("x"))
    p = synth.make_pair(1, seed=0, shape=(nz, ny, nx))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=iters)
    cfg.eta = 0.2  # a single level from identity: keep it unfolded
    best = None
    for rep in range(2):
        ctx = Context(0, "f32")
        if "LIT_PERSIST" in os.environ:
            ctx.set_option(OPT_PERSIST, int(os.environ["LIT_PERSIST"]))
        if "LIT_BRICK_MAX" in os.environ:
            ctx.set_option(OPT_BRICK_MAX, int(os.environ["LIT_BRICK_MAX"]))
        for kv in filter(None, os.environ.get("LIT_OPTS", "").split(",")):
            k, v = kv.split("=")
            ctx.set_option(int(k), int(v))
        try:
            _, log = ctx.register_images(p.grid, p.fixed, p.moving, cfg,
                                         A.PyramidSchedule((1.0,), (iters,)))
            ws = np.array([r.wall_ms for r in log.iterations])
            med = float(np.median(ws[8:])) * 1e3
            best = med if best is None else min(best, med)
        except A.NumericalError as e:
            print(spec, "note:", e)
        ctx.close()
    print(f"{spec:>14}  {nx * ny * nz / 1e6:7.3f} Mvox  {best:7.1f} us/iteration", flush=True)
