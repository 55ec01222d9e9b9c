"""Max difference between the update variants (see test_update_variants_bit_identical)."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
import numpy as np
import golden_cases as G
from paper_2404_01249_b200 import synth, _abi as A
from paper_2404_01249_b200.engine import Context, OPT_BRICK_MAX, OPT_SPLIT, OPT_SPLIT_FOLD_MAX
prec = sys.argv[1] if len(sys.argv) > 1 else "f32"
z, g, sched = G.register_inputs("lncc")
cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=max(sched.iterations))
out = []
for split, fold_max in ((0, 0), (1, 1 << 40), (1, 0)):
    ctx = Context(0, prec)
    ctx.set_option(OPT_BRICK_MAX, 0); ctx.set_option(OPT_SPLIT, split); ctx.set_option(OPT_SPLIT_FOLD_MAX, fold_max)
    f, log = ctx.register_images(g, z["fixed"], z["moving"], cfg, sched)
    ctx.close()
    out.append((f, np.array([r.loss for r in log.iterations])))
print("shape", g.shape if hasattr(g, "shape") else g, "sched", sched.scales, sched.iterations)
for k in (1, 2):
    d = np.abs(out[k][0] - out[0][0])
    ld = np.abs(out[k][1] - out[0][1])
    first = int(np.argmax(ld > 0)) if (ld > 0).any() else -1
    print(k, "field maxdiff", d.max(), "loss maxdiff", ld.max(), "first differing iter", first)
