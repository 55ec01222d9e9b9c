import os, sys, ctypes as C
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2404_01249_b200 import synth, _abi as A
from paper_2404_01249_b200.engine import Context
from oracle import pyoracle
o = pyoracle.port()
p = synth.make_pair(1, seed=0)
g = p.grid
for legacy in (0, 1):
    if legacy: os.environ["DFM_FORCE_LEGACY"] = "1"
    else: os.environ.pop("DFM_FORCE_LEGACY", None)
    ctx = Context(0, "f32")
    s, it = A.schedule_arrays(p.schedule); cap = int(it.sum()) + 1
    recs = (A.dfm_iter_record * cap)(); rl = A.dfm_runlog(); out = np.empty(g.field_shape)
    ci, _ = A.make_init(None, 3); cc = p.config.c()
    f = np.ascontiguousarray(p.fixed); m = np.ascontiguousarray(p.moving)
    rc = ctx.lib.dfm_register(ctx.handle, C.byref(g.c()), f.ctypes.data, m.ctypes.data, A.HOST_F32, C.byref(cc), A._dptr(s),
        it.ctypes.data_as(C.POINTER(C.c_int32)), len(s), C.byref(ci), out.ctypes.data, A.HOST_F64, recs, cap, C.byref(rl))
    det = o.jacobian_det(g, out)
    bad = np.argwhere(det <= 0)
    print("legacy" if legacy else "tma", "rc", rc, "final", rl.final_loss, "sing", rl.final_singularity_fraction,
          "min det", det.min(), "n<=0", (det <= 0).sum(), "n<0.05", (det < 0.05).sum(), "first bad", bad[:5].tolist())
    losses = [recs[i].loss for i in range(rl.n_records)]
    print("  losses at 199/299/349:", losses[199], losses[299], losses[-1], " max_steps last", [recs[i].max_step for i in range(rl.n_records-3, rl.n_records)])

    ctx.close()
