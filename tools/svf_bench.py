"""SVF-mode registration of one config-1 pair (fp32): device time per level."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context

p = synth.make_pair(1, seed=0)
cfg = p.config
cfg.mode = A.MODE_SVF
cfg.svf_M = 6
F = torch.from_numpy(p.fixed).cuda()
M = torch.from_numpy(p.moving).cuda()
ctx = Context(0, "f32")
s = torch.cuda.ExternalStream(ctx.stream_ptr)
for rep in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    log = ctx.register_device(p.grid, F.data_ptr(), M.data_ptr(), cfg, p.schedule)
    e1.record(s)
    torch.cuda.synchronize()
per = [sum(r.wall_ms for r in log.iterations if r.scale_index == k) for k in range(3)]
print(f"svf M=6 config-1 fp32: {e0.elapsed_time(e1):.1f} ms/pair; per level ms {np.round(per, 1).tolist()}; "
      f"final loss {log.final_loss:.5f}")
