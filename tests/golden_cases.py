"""Shared recomputation of the golden vectors with any HostAPI backend.

`compute(api, tag)` re-runs, on `api` (the C restatement, the CUDA context, or
the reference), every call that tests/golden/make_golden.py recorded, and
returns {key: (got, want)} pairs.  test_oracle.py requires bit-identity for
the restatement; test_parity_gpu.py applies the fp32/fp64 tolerances.
"""
import os

import numpy as np

from paper_2404_01249_b200 import _abi as A

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return dict(np.load(os.path.join(GOLDEN, name)))


def grid_of(z):
    dims = tuple(int(v) for v in z["dims"])
    nd = int(z["ndim"]) if "ndim" in z else 3
    return A.GridMeta(nd, dims)


def compute(api, tag):
    z = load(f"funcs_{tag}.npz")
    g = grid_of(z)
    out = {}

    def pair(key, got):
        out[key] = (np.asarray(got), z[key])

    vals, grads = api.sample_linear_points(g, z["M"], z["pts"])
    pair("sample_vals", vals)
    pair("sample_grads", grads)
    pair("warp", api.warp_image(g, z["M"], z["phi"]))
    pair("labels", api.warp_labels(g, z["lab"], z["phi"]))
    pair("compose", api.compose(g, z["phi"], z["psi"]))
    pair("det", api.jacobian_det(g, z["psi"]))
    pair("sing", api.singularity_fraction(g, z["phi"]))
    pair("smooth1", api.gaussian_smooth(g, z["F"], 1.0))
    pair("smooth_aniso", api.gaussian_smooth(g, z["F"], [0.5, 1.5, 0.7]))
    pair("smooth_big", api.gaussian_smooth(g, z["F"], 3.2))
    pair("smoothf", api.gaussian_smooth_field(g, z["phi"], 1.0))
    pair("smoothf05", api.gaussian_smooth_field(g, z["phi"], 0.5))
    for r in (1, 2, 3):
        v, gr = api.lncc_eval(g, z["F"], z["phi"], z["M"], r)
        pair(f"lncc{r}_val", v)
        pair(f"lncc{r}_grad", gr)
    v, gr = api.ssd_eval(g, z["F"], z["phi"], z["M"])
    pair("ssd_val", v)
    pair("ssd_grad", gr)
    v, gr = api.dice_eval(g, np.clip(z["F"], 0, 1), z["phi"], np.clip(z["M"], 0, 1))
    pair("dice_val", v)
    pair("dice_grad", gr)
    d, m2, nu2, t2 = api.adam_step(g, z["m"], z["nu"], 4, 0.9, 0.99, 1e-8, z["v"])
    assert t2 == 5
    pair("adam_dir", d)
    pair("adam_m", m2)
    pair("adam_nu", nu2)
    pair("euler", api.eulerian_direction(g, z["v"], z["psi"], False))
    pair("euler_jac", api.eulerian_direction(g, z["v"], z["psi"], True))
    pair("apply", api.apply_update(g, z["psi"], z["v"] * 300, 0.5, 0.5))
    pair("apply_nos", api.apply_update(g, z["psi"], z["v"] * 300, 0.5, 0.0, 0.3))
    ng, d2 = api.downsample_image(g, z["F"], 2.0)
    assert tuple(ng.dims) == tuple(z["down2_dims"])
    pair("down2", d2)
    ng3, d3 = api.downsample_image(g, z["F"], 3.0)
    assert tuple(ng3.dims) == tuple(z["down3_dims"])
    pair("down3", d3)
    big = A.GridMeta(g.ndim, tuple(int(v) for v in z["up_big_dims"]))
    up = api.upsample_field(g, z["psi"], big)
    pair("up", up)
    um, unu = api.upsample_state(g, z["m"], z["nu"], big)
    pair("up_m", um)
    pair("up_nu", unu)
    pair("resamp_disp", api.resample_displacement(big, z["up"], g))
    return out


def compute_own_grid(api):
    z = load("own_grid.npz")
    g = A.GridMeta(3, tuple(int(v) for v in z["dims"]))
    gm = A.GridMeta(3, tuple(int(v) for v in z["mdims"]))
    v, gr = api.lncc_eval(g, z["F"], z["phi"], z["M"], 2, mg=gm)
    sv, sg = api.ssd_eval(g, z["F"], z["phi"], z["M"], mg=gm)
    return {"lncc_val": (np.asarray(v), z["lncc_val"]), "lncc_grad": (gr, z["lncc_grad"]),
            "ssd_val": (np.asarray(sv), z["ssd_val"]), "ssd_grad": (sg, z["ssd_grad"])}


def register_inputs(name):
    z = load(f"register_{name}.npz")
    g = A.GridMeta(3, tuple(int(v) for v in z["dims"]))
    sched = A.PyramidSchedule(tuple(float(s) for s in z["scales"]),
                              tuple(int(i) for i in z["iters"]))
    return z, g, sched


def register_config(name, z, sched):
    """The RegistrationConfig a register_<name>.npz golden was made with."""
    from paper_2404_01249_b200 import synth
    loss = A.LOSS_LNCC if name.endswith("lncc") else A.LOSS_SSD
    cfg = synth.baseline_config(loss, 2, 1.0, max_iters=max(sched.iterations))
    if "mode" in z:
        cfg.mode = int(z["mode"])
        cfg.svf_M = int(z["svf_M"])
    return cfg


SVF_MS = (0, 1, 4, 6)


def compute_svf(api, tag):
    """exp_map / svf_pullback on the svf.npz inputs -> {key: (got, want)}."""
    z = load("svf.npz")
    g = A.GridMeta(int(z[f"{tag}_ndim"]), tuple(int(v) for v in z[f"{tag}_dims"]))
    out = {}
    for M in SVF_MS:
        out[f"exp{M}"] = (api.exp_map(g, z[f"{tag}_v"], M), z[f"{tag}_exp{M}"])
        out[f"pull{M}"] = (api.svf_pullback(g, z[f"{tag}_v"], z[f"{tag}_w"], M),
                           z[f"{tag}_pull{M}"])
    return out


def compute_affine(api, tag):
    """affine_to_field / affine_param_gradient on affine.npz -> {key: (got, want)}."""
    z = load("affine.npz")
    g = A.GridMeta(int(z[f"{tag}_ndim"]), tuple(int(v) for v in z[f"{tag}_dims"]))
    Am, t, S = z[f"{tag}_A"], z[f"{tag}_t"], z[f"{tag}_S"]
    out = {"field": (api.affine_to_field(g, Am, t), z[f"{tag}_field"])}
    for loss in (A.LOSS_SSD, A.LOSS_LNCC, A.LOSS_DICE):
        F, M = z[f"{tag}_F"], z[f"{tag}_M"]
        if loss == A.LOSS_DICE:
            F, M = np.clip(F, 0, 1), np.clip(M, 0, 1)
        v, dA, dt = api.affine_param_gradient(g, F, M, loss, Am, t, S, 2)
        out[f"grad{loss}_val"] = (np.asarray(v), z[f"{tag}_grad{loss}_val"])
        out[f"grad{loss}_dA"] = (dA, z[f"{tag}_grad{loss}_dA"])
        out[f"grad{loss}_dt"] = (dt, z[f"{tag}_grad{loss}_dt"])
    return out


def affine_register_inputs():
    z = load("affine.npz")
    g = A.GridMeta(3, tuple(int(v) for v in z["reg_dims"]))
    return z, g


def eval_inputs():
    z = load("eval.npz")
    gf = A.GridMeta(3, tuple(int(v) for v in z["f_dims"]), tuple(z["f_spacing"]),
                    tuple(z["f_origin"]))
    gm = A.GridMeta(3, tuple(int(v) for v in z["m_dims"]), tuple(z["m_spacing"]),
                    tuple(z["m_origin"]))
    return z, gf, gm


def region_rows(rep):
    return np.array([[q[k] for k, _ in A.dfm_region_overlap._fields_] for q in rep["regions"]],
                    dtype=np.float64)
