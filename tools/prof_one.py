"""Runs `warm` registrations then one more (the one ncu should capture).
python tools/prof_one.py [config] [f32|f64] [warm]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2404_01249_b200 import synth
from paper_2404_01249_b200.engine import Context
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
prec = sys.argv[2] if len(sys.argv) > 2 else "f32"
warm = int(sys.argv[3]) if len(sys.argv) > 3 else 1
p = synth.make_pair(cfgn, seed=0)
ctx = Context(0, prec)
dt = torch.float32 if prec == "f32" else torch.float64
F = torch.from_numpy(p.fixed).cuda().to(dt); M = torch.from_numpy(p.moving).cuda().to(dt)
torch.cuda.synchronize()
for k in range(warm + 1):
    l0 = ctx.launch_count
    log = ctx.register_device(p.grid, F.data_ptr(), M.data_ptr(), p.config, p.schedule)
    print(f"registration {k}: {ctx.launch_count - l0} launches, final loss {log.final_loss:.5f}")
