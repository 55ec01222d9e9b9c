"""Generates tests/golden/*.npz from the UNMODIFIED reference (oracle/_ref).

Run in the container that has /root/reference:

    make -C oracle ref && python tests/golden/make_golden.py

Inputs are seeded numpy arrays (fp32-representable, like the reference's
MET_FLOAT volumes); outputs are whatever the reference computes in fp64.
These vectors pin the plain-C restatement (tests/test_oracle.py) and the CUDA
path (tests/test_parity_gpu.py) without needing /root/reference at run time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import pyoracle  # noqa: E402
from paper_2404_01249_b200 import _abi as A, synth  # noqa: E402


def f32(a):
    return np.asarray(a, dtype=np.float32).astype(np.float64)


def cases():
    rng = np.random.default_rng(1234)
    g3 = A.GridMeta.make_3d(13, 11, 9)
    g2 = A.GridMeta.make_2d(17, 12)
    gm = A.GridMeta.make_3d(10, 14, 8)  # moving on its own grid
    out = {}
    for tag, g in (("3d", g3), ("2d", g2)):
        F = f32(rng.random(g.shape))
        M = f32(ndimage_smooth(rng.random(g.shape)))
        phi = f32(rng.normal(0, 1.6, g.field_shape))   # includes clamp zones
        psi = f32(rng.normal(0, 0.4, g.field_shape))
        v = f32(rng.normal(0, 1e-3, g.field_shape))
        m = f32(rng.normal(0, 1e-3, g.field_shape))
        nu = f32(rng.random(g.field_shape) * 1e-6)
        lab = rng.integers(0, 6, g.shape).astype(np.int32)
        pts = f32(rng.uniform(-2, max(g.dims) + 1, (64, 3)))
        out[tag] = dict(grid=g, F=F, M=M, phi=phi, psi=psi, v=v, m=m, nu=nu, lab=lab, pts=pts)
    Mo = f32(rng.random(gm.shape))
    out["own"] = dict(grid=g3, gm=gm, F=out["3d"]["F"], M=Mo, phi=out["3d"]["phi"])
    return out


def ndimage_smooth(a):
    from scipy import ndimage
    return ndimage.gaussian_filter(a, 1.0)


SVF_MS = (0, 1, 4, 6)


def svf_golden(ref):
    """exp_map / svf_pullback (diffeo.cpp:66-167) and SVF-mode registrations."""
    rng = np.random.default_rng(4321)
    out = {}
    for tag, g in (("3d", A.GridMeta.make_3d(13, 11, 9)), ("2d", A.GridMeta.make_2d(17, 12))):
        v = f32(rng.normal(0, 1.5, g.field_shape))   # large enough to clamp at the faces
        w = f32(rng.normal(0, 1.0, g.field_shape))
        out[f"{tag}_dims"] = np.array(g.dims)
        out[f"{tag}_ndim"] = np.array(g.ndim)
        out[f"{tag}_v"] = v
        out[f"{tag}_w"] = w
        for M in SVF_MS:
            out[f"{tag}_exp{M}"] = ref.exp_map(g, v, M)
            out[f"{tag}_pull{M}"] = ref.svf_pullback(g, v, w, M)
    np.savez_compressed(os.path.join(HERE, "svf.npz"), **out)
    for loss, name in ((A.LOSS_LNCC, "svf_lncc"), (A.LOSS_SSD, "svf_ssd")):
        p = synth.make_pair(0, seed=11, shape=(24, 24, 24), iters=(12, 8, 4))
        cfg = synth.baseline_config(loss, 2, 1.0, max_iters=12)
        cfg.mode = A.MODE_SVF
        cfg.svf_M = 4
        fld, log = ref.register_images(p.grid, p.fixed, p.moving, cfg, p.schedule)
        np.savez_compressed(
            os.path.join(HERE, f"register_{name}.npz"), fixed=p.fixed, moving=p.moving,
            fixed_labels=p.fixed_labels, moving_labels=p.moving_labels,
            dims=np.array(p.grid.dims), scales=np.array(p.schedule.scales),
            iters=np.array(p.schedule.iterations), field=fld, mode=np.array(A.MODE_SVF),
            svf_M=np.array(4), losses=np.array([r.loss for r in log.iterations]),
            max_steps=np.array([r.max_step for r in log.iterations]),
            scale_index=np.array([r.scale_index for r in log.iterations]),
            final_loss=np.array(log.final_loss), sing=np.array(log.final_singularity_fraction))


def affine_moving(p, A, t):
    """the pair's fixed image warped by the affine map x -> A x + t (pre-alignment case)"""
    g = p.grid
    u = pyoracle.reference().affine_to_field(g, A, t)
    return f32(pyoracle.reference().warp_image(g, p.fixed, u))


def affine_golden(ref):
    """affine_to_field / affine_param_gradient / affine_register (affine.cpp:50-183)."""
    rng = np.random.default_rng(777)
    out = {}
    for tag, g in (("3d", A.GridMeta.make_3d(13, 11, 9)), ("2d", A.GridMeta.make_2d(17, 12))):
        d = g.ndim
        Am = np.eye(d) + rng.normal(0, 0.05, (d, d))
        t = rng.normal(0, 0.5, d)
        F = f32(rng.random(g.shape))
        M = f32(ndimage_smooth(rng.random(g.shape)))
        S = (1.3, 1.1, 0.9)
        out.update({f"{tag}_dims": np.array(g.dims), f"{tag}_ndim": np.array(d), f"{tag}_A": Am,
                    f"{tag}_t": t, f"{tag}_F": F, f"{tag}_M": M, f"{tag}_S": np.array(S),
                    f"{tag}_field": ref.affine_to_field(g, Am, t)})
        for loss in (A.LOSS_SSD, A.LOSS_LNCC, A.LOSS_DICE):
            Fm, Mm = (np.clip(F, 0, 1), np.clip(M, 0, 1)) if loss == A.LOSS_DICE else (F, M)
            v, dA, dt = ref.affine_param_gradient(g, Fm, Mm, loss, Am, t, S, 2)
            out[f"{tag}_grad{loss}_val"] = np.array(v)
            out[f"{tag}_grad{loss}_dA"] = dA
            out[f"{tag}_grad{loss}_dt"] = dt
    p = synth.make_pair(0, seed=21, shape=(32, 28, 24))
    Am = np.array([[1.05, 0.03, 0.0], [-0.02, 0.96, 0.04], [0.0, 0.02, 1.03]])
    moving = affine_moving(p, Am, np.array([1.2, -0.8, 0.5]))
    out["reg_dims"] = np.array(p.grid.dims)
    out["reg_fixed"] = p.fixed
    out["reg_moving"] = moving
    for loss in (A.LOSS_SSD, A.LOSS_LNCC):
        r = ref.affine_register(p.grid, p.fixed, moving, loss, [4, 2, 1], [40, 20, 10], 0.01)
        for k in ("A", "t", "loss", "iterations"):
            out[f"reg{loss}_{k}"] = np.array(r[k])
    np.savez_compressed(os.path.join(HERE, "affine.npz"), **out)


def eval_golden(ref):
    """overlap_report / landmark_error (analysis.cpp:169-283)."""
    rng = np.random.default_rng(99)
    out = {}
    gf = A.GridMeta(3, (21, 17, 13), (1.2, 0.9, 1.5), (3.0, -2.0, 10.0))
    gm = A.GridMeta(3, (21, 17, 13), (1.1, 1.0, 1.4), (-1.0, 4.0, 0.5))
    lab_f = rng.integers(-1, 9, gf.shape).astype(np.int32)      # includes 0 / negative
    lab_w = np.where(rng.random(gf.shape) < 0.7, lab_f,
                     rng.integers(0, 12, gf.shape)).astype(np.int32)  # labels only in one map
    r = ref.overlap_report(gf, lab_w, lab_f)
    out["lab_f"], out["lab_w"] = lab_f, lab_w
    for k, v in r.items():
        if k != "regions":
            out[f"ov_{k}"] = np.array(v)
    out["ov_regions"] = np.array([[q[k] for k, _ in A.dfm_region_overlap._fields_]
                                  for q in r["regions"]], dtype=np.float64)
    phi = f32(rng.normal(0, 2.0, gf.field_shape))
    npts = 40
    lo = np.array(gf.origin)
    hi = lo + (np.array(gf.dims) - 1) * np.array(gf.spacing)
    fixed_mm = rng.uniform(lo - 3, hi + 3, (npts, 3))              # some outside the grid
    moving_mm = fixed_mm + rng.normal(0, 2.0, (npts, 3))
    dist, mean, mx = ref.landmark_error(gf, gm, phi, fixed_mm, moving_mm)
    out.update(dict(phi=phi, fixed_mm=fixed_mm, moving_mm=moving_mm, lm_dist=dist,
                    lm_mean=np.array(mean), lm_max=np.array(mx)))
    for tag, g in (("f", gf), ("m", gm)):
        out[f"{tag}_dims"], out[f"{tag}_spacing"], out[f"{tag}_origin"] = (
            np.array(g.dims), np.array(g.spacing), np.array(g.origin))
    np.savez_compressed(os.path.join(HERE, "eval.npz"), **out)


def main():
    ref = pyoracle.reference()
    if "--only-eval" in sys.argv:
        eval_golden(ref)
        print("eval golden vectors written to", HERE)
        return
    if "--only-affine" in sys.argv:
        affine_golden(ref)
        print("affine golden vectors written to", HERE)
        return
    if "--only-svf" in sys.argv:
        svf_golden(ref)
        print("svf golden vectors written to", HERE)
        return
    svf_golden(ref)
    affine_golden(ref)
    eval_golden(ref)
    C = cases()
    for tag in ("3d", "2d"):
        c = C[tag]
        g = c["grid"]
        r = {}
        r["sample_vals"], r["sample_grads"] = ref.sample_linear_points(g, c["M"], c["pts"])
        r["warp"] = ref.warp_image(g, c["M"], c["phi"])
        r["labels"] = ref.warp_labels(g, c["lab"], c["phi"])
        r["compose"] = ref.compose(g, c["phi"], c["psi"])
        r["det"] = ref.jacobian_det(g, c["psi"])
        r["sing"] = np.array(ref.singularity_fraction(g, c["phi"]))
        r["smooth1"] = ref.gaussian_smooth(g, c["F"], 1.0)
        r["smooth_aniso"] = ref.gaussian_smooth(g, c["F"], [0.5, 1.5, 0.7])
        r["smooth_big"] = ref.gaussian_smooth(g, c["F"], 3.2)
        r["smoothf"] = ref.gaussian_smooth_field(g, c["phi"], 1.0)
        r["smoothf05"] = ref.gaussian_smooth_field(g, c["phi"], 0.5)
        for rr in (1, 2, 3):
            val, gr = ref.lncc_eval(g, c["F"], c["phi"], c["M"], rr)
            r[f"lncc{rr}_val"], r[f"lncc{rr}_grad"] = np.array(val), gr
        val, gr = ref.ssd_eval(g, c["F"], c["phi"], c["M"])
        r["ssd_val"], r["ssd_grad"] = np.array(val), gr
        Fm = np.clip(c["F"], 0, 1)
        Mm = np.clip(c["M"], 0, 1)
        val, gr = ref.dice_eval(g, Fm, c["phi"], Mm)
        r["dice_val"], r["dice_grad"] = np.array(val), gr
        d, m2, nu2, t2 = ref.adam_step(g, c["m"], c["nu"], 4, 0.9, 0.99, 1e-8, c["v"])
        r["adam_dir"], r["adam_m"], r["adam_nu"] = d, m2, nu2
        r["euler"] = ref.eulerian_direction(g, c["v"], c["psi"], False)
        r["euler_jac"] = ref.eulerian_direction(g, c["v"], c["psi"], True)
        r["apply"] = ref.apply_update(g, c["psi"], c["v"] * 300, 0.5, 0.5)
        r["apply_nos"] = ref.apply_update(g, c["psi"], c["v"] * 300, 0.5, 0.0, 0.3)
        ng, r["down2"] = ref.downsample_image(g, c["F"], 2.0)
        r["down2_dims"] = np.array(ng.dims)
        ng3, r["down3"] = ref.downsample_image(g, c["F"], 3.0)
        r["down3_dims"] = np.array(ng3.dims)
        big = A.GridMeta(g.ndim, tuple(2 * x - 1 if x > 1 else 1 for x in g.dims))
        r["up"] = ref.upsample_field(g, c["psi"], big)
        r["up_big_dims"] = np.array(big.dims)
        r["up_m"], r["up_nu"] = ref.upsample_state(g, c["m"], c["nu"], big)
        r["resamp_disp"] = ref.resample_displacement(big, r["up"], g)
        np.savez_compressed(os.path.join(HERE, f"funcs_{tag}.npz"),
                            **{k: v for k, v in c.items() if k != "grid"},
                            dims=np.array(g.dims), ndim=np.array(g.ndim), **r)
    c = C["own"]
    val, gr = ref.lncc_eval(c["grid"], c["F"], c["phi"], c["M"], 2, mg=c["gm"])
    sv, sg = ref.ssd_eval(c["grid"], c["F"], c["phi"], c["M"], mg=c["gm"])
    np.savez_compressed(os.path.join(HERE, "own_grid.npz"), F=c["F"], M=c["M"], phi=c["phi"],
                        dims=np.array(c["grid"].dims), mdims=np.array(c["gm"].dims),
                        lncc_val=np.array(val), lncc_grad=gr, ssd_val=np.array(sv), ssd_grad=sg)
    # end-to-end: a config-0-shaped pair at 24^3 with a short schedule
    for loss, name in ((A.LOSS_LNCC, "lncc"), (A.LOSS_SSD, "ssd")):
        p = synth.make_pair(0, seed=7, shape=(24, 24, 24), iters=(30, 20, 10))
        cfg = synth.baseline_config(loss, 2, 1.0, max_iters=30)
        fld, log = ref.register_images(p.grid, p.fixed, p.moving, cfg, p.schedule)
        np.savez_compressed(
            os.path.join(HERE, f"register_{name}.npz"), fixed=p.fixed, moving=p.moving,
            fixed_labels=p.fixed_labels, moving_labels=p.moving_labels,
            dims=np.array(p.grid.dims), scales=np.array(p.schedule.scales),
            iters=np.array(p.schedule.iterations), field=fld,
            losses=np.array([r.loss for r in log.iterations]),
            max_steps=np.array([r.max_step for r in log.iterations]),
            scale_index=np.array([r.scale_index for r in log.iterations]),
            final_loss=np.array(log.final_loss), sing=np.array(log.final_singularity_fraction))
    # default early stopping (window 10, tol 1e-5) on 16^3 self-registration
    p = synth.make_pair(0, seed=3, shape=(16, 16, 16))
    fld, log = ref.register_images(p.grid, p.fixed, p.fixed, A.RegistrationConfig(),
                                   A.PyramidSchedule())
    np.savez_compressed(os.path.join(HERE, "register_self.npz"), fixed=p.fixed, field=fld,
                        losses=np.array([r.loss for r in log.iterations]),
                        final_loss=np.array(log.final_loss))
    print("golden vectors written to", HERE)


if __name__ == "__main__":
    main()
