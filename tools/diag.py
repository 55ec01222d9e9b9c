"""Diagnostics: per-scale wall time and loss trajectory of one config-1 run."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2404_01249_b200 import synth
from paper_2404_01249_b200.engine import Context

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = synth.make_pair(cfgn, seed=0)
for prec in ("f32", "f64"):
    ctx = Context(0, prec)
    ctx.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    t0 = time.perf_counter()
    fld, log = ctx.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    dt = time.perf_counter() - t0
    print(f"[{prec}] total {dt*1e3:.1f} ms (RunLog total {log.total_ms:.1f}), final loss {log.final_loss:.5f}")
    for s in range(len(p.schedule.scales)):
        rs = [r for r in log.iterations if r.scale_index == s]
        ls = np.array([r.loss for r in rs]); ws = np.array([r.wall_ms for r in rs])
        print(f"  scale {s}: n={len(rs)} wall sum {ws.sum():.2f} ms (per it {np.median(ws)*1e3:.1f} us) "
              f"loss first {ls[0]:.5f} min {ls.min():.5f}@{ls.argmin()} last {ls[-1]:.5f}")
        print("   ", " ".join(f"{v:.4f}" for v in ls[::max(1, len(ls)//12)]))
    ctx.close()
