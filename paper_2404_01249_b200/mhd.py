"""MetaImage I/O of the reference (io.hpp: read/write_image_mhd,
read/write_labels_mhd, read/write_field_mhd) over the native C-ABI
(csrc/mhd_io.cu), plus the streaming device feed.  Host arrays follow the
reference layout: images (z, y, x) doubles, fields (z, y, x, ndim) doubles,
labels int32."""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _abi as A
from .engine import load_library


def _lib():
    lib = load_library()
    return lib, A.CallTable(lib, "dfm_")


def read_header(path: str) -> dict:
    lib, t = _lib()
    info = A.dfm_mhd_info()
    t.check(lib.dfm_mhd_read_header(path.encode(), C.byref(info)), "mhd_read_header")
    return dict(grid=A.GridMeta.from_c(info.grid), element_type=info.element_type,
                channels=info.channels, element_type_name=info.element_type_name.decode(),
                raw_path=info.raw_path.decode())


def _read(fn: str, path: str, dtype, comps_of):
    lib, t = _lib()
    g = A.dfm_grid()
    f = getattr(lib, fn)
    t.check(f(path.encode(), C.byref(g), None, C.c_int64(0)), fn)
    gm = A.GridMeta.from_c(g)
    n = gm.voxel_count * comps_of(gm)
    out = np.empty(n, dtype=dtype)
    ptr = out.ctypes.data_as(C.POINTER(C.c_double if dtype == np.float64 else C.c_int32))
    t.check(f(path.encode(), C.byref(g), ptr, C.c_int64(n)), fn)
    return gm, out


def read_image(path: str):
    gm, a = _read("dfm_mhd_read_image", path, np.float64, lambda g: 1)
    return gm, a.reshape(gm.shape)


def read_labels(path: str):
    gm, a = _read("dfm_mhd_read_labels", path, np.int32, lambda g: 1)
    return gm, a.reshape(gm.shape)


def read_field(path: str):
    gm, a = _read("dfm_mhd_read_field", path, np.float64, lambda g: g.ndim)
    return gm, a.reshape(gm.field_shape)


def write_image(path: str, g: A.GridMeta, img):
    lib, t = _lib()
    a = A.as_f64(img, g.shape)
    t.check(lib.dfm_mhd_write_image(path.encode(), C.byref(g.c()), A._dptr(a)), "mhd_write_image")


def write_labels(path: str, g: A.GridMeta, labels):
    lib, t = _lib()
    a = np.ascontiguousarray(labels, dtype=np.int32).ravel()
    t.check(lib.dfm_mhd_write_labels(path.encode(), C.byref(g.c()),
                                     a.ctypes.data_as(C.POINTER(C.c_int32))), "mhd_write_labels")


def write_field(path: str, g: A.GridMeta, field):
    lib, t = _lib()
    a = A.as_f64(field, g.field_shape)
    t.check(lib.dfm_mhd_write_field(path.encode(), C.byref(g.c()), A._dptr(a)), "mhd_write_field")


def dev_load_image(ctx, path: str, d_out: int = 0):
    """Streams an MET_FLOAT image into device memory at d_out (context
    precision); d_out = 0 only returns the grid."""
    g = A.dfm_grid()
    ctx.t.check(ctx.lib.dfm_dev_load_image_mhd(ctx.handle, path.encode(), C.byref(g),
                                               C.c_void_p(d_out or None)), "dev_load_image_mhd")
    return A.GridMeta.from_c(g)


def dev_save_field(ctx, path: str, g: A.GridMeta, d_field_soa: int):
    ctx.t.check(ctx.lib.dfm_dev_save_field_mhd(ctx.handle, path.encode(), C.byref(g.c()),
                                               C.c_void_p(d_field_soa)), "dev_save_field_mhd")
