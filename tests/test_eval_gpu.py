"""Evaluation epilogue on the device: overlap_report and
landmark_error (analysis.cpp:169-283), and the device-resident warp_labels ->
overlap_report chain after dfm_dev_register.

overlap_report is integer counting, so it is held BIT-EXACT to the reference
(every ratio, every region).  landmark_error samples phi with the fp64 or fp32
trilinear kernel: fp64 within 1e-12 mm, fp32 within 1e-4 mm.
"""
import numpy as np
import pytest

import golden_cases as G
from paper_2404_01249_b200 import _abi as A, synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_overlap_report_bit_exact(request, prec):
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    z, gf, gm = G.eval_inputs()
    r = ctx.overlap_report(gf, z["lab_w"], z["lab_f"])
    for k, v in r.items():
        if k != "regions":
            assert v == float(z[f"ov_{k}"]), k
    assert np.array_equal(G.region_rows(r), z["ov_regions"])


@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_landmark_error_matches_reference(request, prec):
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    z, gf, gm = G.eval_inputs()
    dist, mean, mx = ctx.landmark_error(gf, gm, z["phi"], z["fixed_mm"], z["moving_mm"])
    tol = 1e-12 if prec == "f64" else 1e-4
    assert np.abs(dist - z["lm_dist"]).max() <= tol
    assert abs(mean - float(z["lm_mean"])) <= tol and abs(mx - float(z["lm_max"])) <= tol


def test_overlap_edge_cases(ctx32, oracle_port):
    """empty (all-background) maps, a single label, labels only in one map,
    and a large label id (shared-memory vs global histogram paths)."""
    g = A.GridMeta.make_3d(9, 7, 5)
    zero = np.zeros(g.shape, np.int32)
    cases = [(zero, zero)]
    one = zero.copy()
    one[1:3, 2:4, 3:6] = 5
    cases.append((one, zero))
    cases.append((zero, one))
    big = one.copy()
    big[0, 0, 0] = 70000
    cases.append((big, one))
    for w, f in cases:
        a = ctx32.overlap_report(g, w, f)
        b = oracle_port.overlap_report(g, w, f)
        assert {k: v for k, v in a.items() if k != "regions"} == \
            {k: v for k, v in b.items() if k != "regions"}
        assert G.region_rows(a).tolist() == G.region_rows(b).tolist()
    with pytest.raises(A.InvalidArgument):
        ctx32.overlap_report(g, zero, zero, gf=A.GridMeta.make_3d(9, 7, 6))


def test_device_epilogue_chain(ctx32, oracle_port):
    """register on device -> dev_warp_labels -> dev_overlap_report, no host copy
    of the volumes; equals the host-side warp_labels + overlap_report."""
    import ctypes as C
    import torch
    p = synth.make_pair(0, seed=2, shape=(32, 32, 32), iters=(10, 6, 4))
    g = p.grid
    F = torch.from_numpy(p.fixed).float().cuda()
    M = torch.from_numpy(p.moving).float().cuda()
    fld = torch.empty((3,) + g.shape, dtype=torch.float32, device="cuda")
    ctx32.register_device(g, F.data_ptr(), M.data_ptr(), p.config, p.schedule, fld.data_ptr())
    lab_m = torch.from_numpy(p.moving_labels.astype(np.int32)).cuda()
    lab_f = torch.from_numpy(p.fixed_labels.astype(np.int32)).cuda()
    warped = torch.empty_like(lab_m)
    lib = ctx32.lib
    torch.cuda.synchronize()
    rc = lib.dfm_dev_warp_labels(ctx32.handle, C.byref(g.c()), C.c_void_p(lab_m.data_ptr()),
                                 C.c_void_p(fld.data_ptr()), C.c_void_p(warped.data_ptr()))
    assert rc == 0
    rep = A.dfm_overlap_summary()
    regs = (A.dfm_region_overlap * 256)()
    rc = lib.dfm_dev_overlap_report(ctx32.handle, C.byref(g.c()), C.c_void_p(warped.data_ptr()),
                                    C.c_void_p(lab_f.data_ptr()), C.byref(rep), regs, 256)
    assert rc == 0
    field_aos = fld.permute(1, 2, 3, 0).double().cpu().numpy()
    wl = oracle_port.warp_labels(g, p.moving_labels, field_aos)
    assert np.array_equal(warped.cpu().numpy(), wl)
    ref = oracle_port.overlap_report(g, wl, p.fixed_labels)
    assert rep.mo_mean == ref["mo_mean"] and rep.to_klein == ref["to_klein"]
    assert rep.n_regions == len(ref["regions"])
