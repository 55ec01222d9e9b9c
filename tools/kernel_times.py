"""Per-kernel-class device times (CUDA events around every launch) of the loop
at one volume size, per kernel family.

    python tools/kernel_times.py NX NY NZ [iters] [f32|f64]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200 import engine
from paper_2404_01249_b200.engine import Context, OPT_BRICK_MAX, OPT_PERSIST

nx, ny, nz = (int(v) for v in sys.argv[1:4])
iters = int(sys.argv[4]) if len(sys.argv) > 4 else 20
prec = sys.argv[5] if len(sys.argv) > 5 else "f32"
p = synth.make_pair(1, seed=0, shape=(nx, ny, nz), iters=(iters,))
sched = A.PyramidSchedule((1.0,), (iters,))
cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=iters)
for fam, bm in [("stream", 0), ("brick", 1 << 40)][:int(os.environ.get("KT_FAMS", "2"))]:
    ctx = Context(0, prec)
    ctx.set_option(OPT_BRICK_MAX, bm)
    ctx.set_option(OPT_PERSIST, 0)
    for kv in filter(None, os.environ.get("KT_OPTS", "").split(",")):  # e.g. SPLIT_FOLD_MAX=0
        k, v = kv.split("=")
        ctx.set_option(getattr(engine, "OPT_" + k), int(float(v)))
    ctx.set_profiling(True)
    try:
        ctx.register_images(p.grid, p.fixed, p.moving, cfg, sched)
    except A.NumericalError:
        pass  # a single full-resolution level from identity may fold: timings still stand
    kt = ctx.kernel_times()
    parts = []
    for k in ("loss_fwd", "lncc_bwd", "smooth_adam", "compose_smooth"):
        ms, n = kt[k]["ms"], kt[k]["launches"]
        parts.append(f"{k} {1e3 * ms / max(n, 1):7.1f}us")
    print(f"[{prec} {nx}x{ny}x{nz} {fam:6s}] " + "  ".join(parts), flush=True)
    ctx.close()
