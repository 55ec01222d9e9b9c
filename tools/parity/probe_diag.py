"""Diagnostic (box): error distribution of the per-kernel probe at full size."""
import sys, os, json
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "..", "tests"))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np
import loop_probe
from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context, OPT_SPLIT_FOLD_MAX, OPT_LARGE_MIN, OPT_BRICK_MAX
from oracle import pyoracle

o = pyoracle.best()
cfgn = int(sys.argv[1]) if len(sys.argv) > 1 else 1
p = synth.make_pair(cfgn, seed=0)
g = p.grid
F = p.fixed.astype(np.float64); M = p.moving.astype(np.float64)

def stats(name, a, ref, rel=1e-5, absf=1e-6):
    a = np.asarray(a, np.float64).ravel(); ref = np.asarray(ref, np.float64).ravel()
    peak = np.abs(ref).max()
    r = np.abs(a - ref) / (rel * np.abs(ref) + absf * peak)
    idx = np.argsort(r)[::-1][:5]
    print(name, f"peak {peak:.3e} worst {r.max():.3g} n>1 {(r>1).sum()} n>0.5 {(r>0.5).sum()} n>0.1 {(r>0.1).sum()}")
    for i in idx:
        print("   ", i, f"gpu {a[i]:.6e} ref {ref[i]:.6e} ratio {r[i]:.3g}")

# small forced-large failure message
try:
    q = synth.make_pair(1, seed=0, shape=(56, 48, 40))
    c = Context(0, "f32")
    for k, v in {OPT_LARGE_MIN: 0, OPT_SPLIT_FOLD_MAX: 0, OPT_BRICK_MAX: 0}.items():
        c.set_option(k, v)
    c.register_images(q.grid, q.fixed, q.moving, q.config, A.PyramidSchedule((1.0,), (1,)))
    print("small forced ok")
except Exception as e:
    print("small forced error:", e)
for opts in ({OPT_LARGE_MIN: 0}, {OPT_SPLIT_FOLD_MAX: 0, OPT_BRICK_MAX: 0}, {OPT_LARGE_MIN: 0, OPT_BRICK_MAX: 0}):
    try:
        c = Context(0, "f32")
        for k, v in opts.items():
            c.set_option(k, v)
        c.register_images(q.grid, q.fixed, q.moving, q.config, A.PyramidSchedule((1.0,), (1,)))
        print(opts, "ok")
    except Exception as e:
        print(opts, "error:", e)

for mode in ("default", "folded"):
    ctx = Context(0, "f32")
    if mode == "folded":
        ctx.set_option(OPT_SPLIT_FOLD_MAX, 1 << 40)
    cfg = p.config
    _, l1 = ctx.register_images(g, p.fixed, p.moving, cfg, A.PyramidSchedule((1.0,), (1,)))
    u1 = ctx.debug_field("reg_u1", g); m1 = ctx.debug_field("reg_m", g); nu1 = ctx.debug_field("reg_nu", g)
    _, l2 = ctx.register_images(g, p.fixed, p.moving, cfg, A.PyramidSchedule((1.0,), (2,)))
    m2 = ctx.debug_field("reg_m", g); nu2 = ctx.debug_field("reg_nu", g)
    L1, g1 = o.lncc_eval(g, F, u1, M, 2) if cfg.loss == A.LOSS_LNCC else o.ssd_eval(g, F, u1, M)
    if mode == "folded":
        gg = ctx.debug_field("reg_grad", g)
        stats("grad(fwd+bwd)", gg, g1)
        # smoothing of the GPU grad vs GPU m2
        v = -o.gaussian_smooth_field(g, gg, cfg.sigma_grad)
        stats("smooth+adam m from GPU grad", m2, 0.9 * m1 + 0.1 * v)
    v = -o.gaussian_smooth_field(g, g1, cfg.sigma_grad)
    stats(mode + " m2", m2, 0.9 * m1 + 0.1 * v)
    stats(mode + " nu2", nu2, 0.99 * nu1 + 0.01 * v * v)
    ctx.close()
