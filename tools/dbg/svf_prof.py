import os, sys
sys.path.insert(0, os.getcwd())
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context
import torch
p = synth.make_pair(1, seed=0, iters=(2, 2, 2))
cfg = p.config; cfg.mode = A.MODE_SVF; cfg.svf_M = 6
F = torch.from_numpy(p.fixed).cuda(); M = torch.from_numpy(p.moving).cuda()
ctx = Context(0, "f32")
log = ctx.register_device(p.grid, F.data_ptr(), M.data_ptr(), cfg, p.schedule)
torch.cuda.synchronize(); print("ok")
