"""A/B of context options on one pair: per-scale device time and the whole
registration (CUDA events on the library stream), best of 3.

    python tools/opt_ab.py [config] [f32|f64] "KEY=V,KEY=V" ["KEY=V" ...]
KEY is an OPT_* name without the prefix (BRICK_MAX, SPLIT, SPLIT_FOLD_MAX, ...);
an empty spec is the default configuration."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2404_01249_b200 import engine, synth
from paper_2404_01249_b200.engine import Context

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
specs = sys.argv[3:] or [""]
p = synth.make_pair(cfgn, seed=0)
dt = torch.float32 if prec == "f32" else torch.float64
F = torch.from_numpy(p.fixed).cuda().to(dt)
M = torch.from_numpy(p.moving).cuda().to(dt)
for spec in specs:
    ctx = Context(0, prec)
    for kv in filter(None, spec.split(",")):
        k, v = kv.split("=")
        ctx.set_option(getattr(engine, "OPT_" + k), int(float(v)))
    s = torch.cuda.ExternalStream(ctx.stream_ptr)
    best = 1e30
    for rep in range(4):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        log = ctx.register_device(p.grid, F.data_ptr(), M.data_ptr(), p.config, p.schedule)
        e1.record(s)
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    per = []
    for si in range(len(p.schedule.scales)):
        ws = np.array([r.wall_ms for r in log.iterations if r.scale_index == si])
        per.append(f"s{si}: {ws.sum():7.2f} ms ({np.median(ws) * 1e3:6.1f} us/it)")
    print(f"[{prec} {spec or 'default':>28}] best {best:7.2f} ms  loss {log.final_loss:.6f}  "
          + "  ".join(per), flush=True)
    ctx.close()
