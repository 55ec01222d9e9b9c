"""Per-kernel parity of the hot loop at any size, in the precision that runs.

Runs register_images for one and for two iterations on a single scale and
reads the loop's own workspace (dfm_ctx_debug_read) — the outputs of the very
kernels the benchmark launches, captured in the same CUDA graphs — then feeds
each kernel's GPU inputs to the CPU oracle and compares its GPU outputs:

  iteration 0 (u0 = 0)      -> u1, m1, nu1              (1-iteration run)
  iteration 1 (u1 -> u2)    -> losses L0, L1, m2, nu2, step2, c2, u2, G2
  LNCC/SSD fwd+bwd + sigma_grad smoothing + Adam moments:
      m2  = b1 m1  + (1-b1) v,   nu2 = b2 nu1 + (1-b2) v^2,   v = -G_sg * grad(u1)
      (similarity.cpp:81-190, interp.cpp:362-371, diffeo.cpp:11-24, optim.cpp:22-42)
  Adam direction + cap:  step2 = clamp(eta (m2/c1) / (sqrt(nu2/c2) + eps))
      (optim.cpp:27-35, diffeo.cpp:42-55)
  compose:               c2 = step2 + u1(x + step2)          (interp.cpp:269-289)
  sigma_warp smoothing:  u2 = G_sw * c2                       (diffeo.cpp:56-63)
  W/G gather:            W, G = M(x + u2), grad M(x + u2)     (similarity.cpp:25-45)
  loss values:           L0 = loss(u0), L1 = loss(u1)
  monitor:               max_step(1) = max |step2|            (pipeline.cpp:36-41)

Only the split update (its own compose kernel, the step materialised in
"reg_step", the composed field in "reg_grad") is probed; callers set the
context options that select it.  Test infrastructure (imports oracle/).
"""
from __future__ import annotations

import numpy as np

from paper_2404_01249_b200 import _abi as A


def worst(a, ref, rel, absfrac):
    """max over elements of |a - ref| / (rel |ref| + absfrac max|ref|): <= 1 passes"""
    a = np.asarray(a, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    scale = rel * np.abs(ref) + absfrac * max(np.abs(ref).max(), 1e-300)
    return float((np.abs(a - ref) / scale).max())


def probe(ctx, g: A.GridMeta, fixed, moving, cfg: A.RegistrationConfig) -> dict:
    """GPU intermediates of iterations 0 and 1 on one scale (scale 1.0)."""
    out = {}
    _, log1 = ctx.register_images(g, fixed, moving, cfg, A.PyramidSchedule((1.0,), (1,)))
    out["u1"] = ctx.debug_field("reg_u1", g)
    out["m1"] = ctx.debug_field("reg_m", g)
    out["nu1"] = ctx.debug_field("reg_nu", g)
    _, log2 = ctx.register_images(g, fixed, moving, cfg, A.PyramidSchedule((1.0,), (2,)))
    u1b = ctx.debug_field("reg_u1", g)
    assert np.array_equal(u1b, out["u1"]), "iteration 0 not reproducible"
    out["u2"] = ctx.debug_field("reg_u0", g)
    out["m2"] = ctx.debug_field("reg_m", g)
    out["nu2"] = ctx.debug_field("reg_nu", g)
    out["step2"] = ctx.debug_field("reg_step", g)
    out["c2"] = ctx.debug_field("reg_grad", g)
    if cfg.loss == A.LOSS_LNCC:
        out["W2"] = ctx.debug_read("reg_W", g.voxel_count).astype(np.float64).reshape(g.shape)
        out["G2"] = ctx.debug_field("reg_G", g)
    out["losses"] = np.array([r.loss for r in log2.iterations])
    out["max_steps"] = np.array([r.max_step for r in log2.iterations])
    out["loss0_1it"] = log1.iterations[0].loss
    return out


def check(o, g: A.GridMeta, fixed, moving, cfg: A.RegistrationConfig, P: dict,
          rel: float, absfrac: float, loss_rel: float) -> dict:
    """Compares every kernel's GPU output with the oracle fed the GPU's inputs.
    Returns {kernel: worst ratio}; every ratio must be <= 1."""
    F = np.asarray(fixed, dtype=np.float64)
    M = np.asarray(moving, dtype=np.float64)
    r = {}
    zero = np.zeros(g.field_shape)
    lncc = cfg.loss == A.LOSS_LNCC

    def loss_grad(u):
        if lncc:
            return o.lncc_eval(g, F, u, M, cfg.lncc_radius)
        return o.ssd_eval(g, F, u, M)

    L0, _ = loss_grad(zero)
    L1, g1 = loss_grad(P["u1"])
    r["loss(u0)"] = abs(P["losses"][0] - L0) / (loss_rel * abs(L0))
    r["loss(u1)"] = abs(P["losses"][1] - L1) / (loss_rel * abs(L1))
    # fwd + bwd + sigma_grad smoothing + -g + Adam moments at t = 2
    v = -o.gaussian_smooth_field(g, g1, cfg.sigma_grad)
    b1, b2 = cfg.beta1, cfg.beta2
    m2 = b1 * P["m1"] + (1.0 - b1) * v
    nu2 = b2 * P["nu1"] + (1.0 - b2) * v * v
    r["grad+smooth+adam m"] = worst(P["m2"], m2, rel, absfrac)
    r["grad+smooth+adam nu"] = worst(P["nu2"], nu2, rel, absfrac)
    # Adam direction at t = 2 + eta + cap (optim.cpp:27-35 with std::pow bias terms)
    c1 = 1.0 - b1 ** 2
    c2 = 1.0 - b2 ** 2
    d = (P["m2"] / c1) / (np.sqrt(P["nu2"] / c2) + cfg.eps_adam)
    step = np.clip(cfg.eta * d, -cfg.step_cap, cfg.step_cap)
    r["adam step"] = worst(P["step2"], step, rel, absfrac)
    r["max_step"] = abs(P["max_steps"][1] - np.abs(P["step2"]).max()) / (
        rel * np.abs(P["step2"]).max())
    # compose c = step + u1(x + step), then sigma_warp smoothing
    c = o.compose(g, P["u1"], P["step2"])
    r["compose"] = worst(P["c2"], c, rel, absfrac)
    u2 = o.gaussian_smooth_field(g, P["c2"], cfg.sigma_warp)
    r["smooth_warp"] = worst(P["u2"], u2, rel, absfrac)
    if lncc:
        # W/G gather of the compose-smooth kernel: M and grad M at x + u2
        zz, yy, xx = np.meshgrid(*[np.arange(s, dtype=np.float64) for s in g.shape],
                                 indexing="ij")
        pts = np.stack([xx + P["u2"][..., 0], yy + P["u2"][..., 1], zz + P["u2"][..., 2]],
                       axis=-1).reshape(-1, 3)
        vals, grads = o.sample_linear_points(g, M, pts)
        r["W gather"] = worst(P["W2"].ravel(), vals, rel, absfrac)
        r["G gather"] = worst(P["G2"].reshape(-1, 3), grads, rel, absfrac)
    return r
