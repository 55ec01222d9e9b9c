import sys, os
sys.path.insert(0, '/root/repo')
os.chdir(os.environ.get('GRAFT_REPO_ROOT', '/root/repo'))
import torch
from paper_2404_01249_b200.synth_gpu import make_config4_pair
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context
n = int(sys.argv[1])
f, m = make_config4_pair("cuda", 0, (n, n, n), n_puncta=int(200000 * (n / 1024) ** 3))
for name, t in (("fixed", f), ("moving", m)):
    print(name, float(t.min()), float(t.max()), bool(torch.isfinite(t).all()), float(t.mean()))
torch.cuda.synchronize(); torch.cuda.empty_cache()
print("mem allocated GB", torch.cuda.memory_allocated() / 1e9, "reserved", torch.cuda.memory_reserved() / 1e9)
g = A.GridMeta.make_3d(n, n, n)
import numpy as np
for sched in (A.PyramidSchedule((8.0, 4.0), (200, 1)), A.PyramidSchedule((8.0, 4.0), (200, 100)), A.PyramidSchedule((8.0, 4.0, 2.0), (200, 100, 50)), A.PyramidSchedule((8.0, 4.0, 2.0, 1.0), (200, 100, 50, 25))):
    ctx = Context(0, "f32")
    cfg = synth.baseline_config(A.LOSS_LNCC, 3, 1.0, max_iters=200)
    try:
        log = ctx.register_device(g, f.data_ptr(), m.data_ptr(), cfg, sched)
        ls = np.array([r.loss for r in log.iterations]); ms = np.array([r.max_step for r in log.iterations])
        print(sched.scales, len(ls), ls[::25].round(4).tolist(), ms[::25].round(3).tolist(), log.final_loss, log.final_singularity_fraction)
    except Exception as e:
        print(sched.scales, "ERR", e)
    ctx.close()
