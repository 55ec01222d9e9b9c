"""A/B of the kernel families per pyramid level on one config-1 pair:
per-scale device time (sum of the per-iteration globaltimer stamps) and the
whole registration (CUDA events on the library stream).

    python tools/family_ab.py [config] [f32|f64] [brick_max ...]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2404_01249_b200 import synth
from paper_2404_01249_b200.engine import Context, OPT_BRICK_MAX

cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
maxes = [int(float(v)) for v in sys.argv[3:]] or [0, 2_000_000]
p = synth.make_pair(cfgn, seed=0)
dt = torch.float32 if prec == "f32" else torch.float64
F = torch.from_numpy(p.fixed).cuda().to(dt)
M = torch.from_numpy(p.moving).cuda().to(dt)
for bm in maxes:
    ctx = Context(0, prec)
    ctx.set_option(OPT_BRICK_MAX, bm)
    s = torch.cuda.ExternalStream(ctx.stream_ptr)
    for rep in range(3):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        log = ctx.register_device(p.grid, F.data_ptr(), M.data_ptr(), p.config, p.schedule)
        e1.record(s)
        torch.cuda.synchronize()
    per = []
    for si in range(len(p.schedule.scales)):
        ws = np.array([r.wall_ms for r in log.iterations if r.scale_index == si])
        per.append(f"s{si}: {ws.sum():7.2f} ms ({np.median(ws) * 1e3:6.1f} us/it)")
    print(f"[{prec} brick_max={bm:>10}] total {e0.elapsed_time(e1):7.2f} ms  " + "  ".join(per)
          + f"  final loss {log.final_loss:.6f}", flush=True)
    ctx.close()
