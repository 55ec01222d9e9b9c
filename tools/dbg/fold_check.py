import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
from paper_2404_01249_b200 import synth
from paper_2404_01249_b200.engine import Context
p = synth.make_pair(1, seed=int(sys.argv[1]) if len(sys.argv) > 1 else 0)
for prec in ("f32", "f64"):
    for legacy in (0, 1):
        if legacy: os.environ["DFM_FORCE_LEGACY"] = "1"
        else: os.environ.pop("DFM_FORCE_LEGACY", None)
        c = Context(0, prec)
        try:
            f, l = c.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
            print(prec, "legacy" if legacy else "tma", "ok final", l.final_loss)
        except Exception as e:
            print(prec, "legacy" if legacy else "tma", "ERR", e)
        c.close()
