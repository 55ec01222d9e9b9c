"""Streaming MHD feed on the device: file -> pinned chunks -> HBM (both
precisions) and HBM field -> file, bit-identical to the host readers/writers;
plus a registration fed from and written to MetaImage files."""
import numpy as np
import pytest

from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200 import mhd as M

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_dev_load_matches_host_reader(request, tmp_path, prec):
    import torch
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    g = A.GridMeta(3, (160, 192, 60), (0.9, 1.0, 1.2), (1.0, 2.0, 3.0))  # 7.4 MB: > 1 chunk? no
    big = A.GridMeta(3, (256, 256, 96), (1.0, 1.0, 1.0))                 # 25 MB: 2 chunks
    for gg in (g, big):
        img = np.random.default_rng(0).normal(size=gg.shape).astype(np.float32)
        p = str(tmp_path / "i.mhd")
        M.write_image(p, gg, img.astype(np.float64))
        dt = torch.float32 if prec == "f32" else torch.float64
        out = torch.empty(gg.shape, dtype=dt, device="cuda")
        got = M.dev_load_image(ctx, p, out.data_ptr())
        assert got == gg
        assert np.array_equal(out.cpu().numpy().astype(np.float32), img)


@pytest.mark.parametrize("prec", ["f32", "f64"])
def test_dev_save_field_matches_host_writer(request, tmp_path, prec):
    import torch
    ctx = request.getfixturevalue("ctx64" if prec == "f64" else "ctx32")
    g = A.GridMeta(3, (200, 180, 90), (1.0, 1.0, 1.0))  # 38.9 MB field: 3 chunks
    dt = torch.float32 if prec == "f32" else torch.float64
    soa = torch.randn((3,) + g.shape, dtype=dt, device="cuda")
    a, b = str(tmp_path / "a.mhd"), str(tmp_path / "b.mhd")
    M.dev_save_field(ctx, a, g, soa.data_ptr())
    M.write_field(b, g, soa.permute(1, 2, 3, 0).double().cpu().numpy())
    assert open(a).read().replace("a.raw", "") == open(b).read().replace("b.raw", "")
    assert open(a[:-4] + ".raw", "rb").read() == open(b[:-4] + ".raw", "rb").read()


def test_registration_fed_from_mhd(ctx32, tmp_path):
    import torch
    p = synth.make_pair(0, seed=4, shape=(48, 40, 32), iters=(8, 6, 4))
    fp, mp_ = str(tmp_path / "f.mhd"), str(tmp_path / "m.mhd")
    M.write_image(fp, p.grid, p.fixed)
    M.write_image(mp_, p.grid, p.moving)
    F = torch.empty(p.grid.shape, dtype=torch.float32, device="cuda")
    Mv = torch.empty_like(F)
    M.dev_load_image(ctx32, fp, F.data_ptr())
    M.dev_load_image(ctx32, mp_, Mv.data_ptr())
    fld = torch.empty((3,) + p.grid.shape, dtype=torch.float32, device="cuda")
    la = ctx32.register_device(p.grid, F.data_ptr(), Mv.data_ptr(), p.config, p.schedule,
                               fld.data_ptr())
    fa, lb = ctx32.register_images(p.grid, p.fixed, p.moving, p.config, p.schedule)
    assert [r.loss for r in la.iterations] == [r.loss for r in lb.iterations]
    out = str(tmp_path / "phi.mhd")
    M.dev_save_field(ctx32, out, p.grid, fld.data_ptr())
    g2, back = M.read_field(out)
    assert g2.dims == p.grid.dims and np.array_equal(back, fa.astype(np.float32))
