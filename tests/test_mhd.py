"""MetaImage I/O (io.cpp:117-328) of the native library against the
restatement oracle/mhd.py: byte-identical headers and payloads, the reader's
acceptance rules and its "path: byte N: ..." error messages.  Host-only code:
runs without a GPU."""
import os

import numpy as np
import pytest

from oracle import mhd as R
from paper_2404_01249_b200 import _abi as A
from paper_2404_01249_b200 import mhd as M


G3 = A.GridMeta(3, (7, 5, 4), (0.8, 1.25, 2.0 / 3.0), (-3.5, 10.0, 1e-3))
G2 = A.GridMeta(2, (9, 6, 1), (1.1, 0.9, 1.0), (2.0, -1.0, 0.0))


@pytest.mark.parametrize("g", [G3, G2])
def test_writers_byte_identical(tmp_path, g):
    rng = np.random.default_rng(0)
    img = rng.normal(size=g.shape)
    lab = rng.integers(-5, 300, g.shape).astype(np.int32)
    fld = rng.normal(size=g.field_shape)
    for kind, data, et, ch in (("img", img, "MET_FLOAT", 1), ("lab", lab, "MET_SHORT", 1),
                               ("fld", fld, "MET_FLOAT", g.ndim)):
        a = str(tmp_path / f"{kind}_a.mhd")
        b = str(tmp_path / f"{kind}_b.mhd")
        {"img": M.write_image, "lab": M.write_labels, "fld": M.write_field}[kind](a, g, data)
        R.write(b, g.ndim, g.dims, g.spacing, g.origin, data, et, ch)
        ha, hb = open(a).read(), open(b).read()
        assert ha.replace("_a.raw", "") == hb.replace("_b.raw", ""), (ha, hb)
        assert open(a[:-4] + ".raw", "rb").read() == open(b[:-4] + ".raw", "rb").read()


@pytest.mark.parametrize("g", [G3, G2])
def test_round_trips(tmp_path, g):
    rng = np.random.default_rng(1)
    img = rng.normal(size=g.shape).astype(np.float32).astype(np.float64)
    lab = rng.integers(-5, 300, g.shape).astype(np.int32)
    fld = rng.normal(size=g.field_shape).astype(np.float32).astype(np.float64)
    p = str(tmp_path / "x.mhd")
    M.write_image(p, g, img)
    gg, back = M.read_image(p)
    assert gg == g and np.array_equal(back, img)
    M.write_labels(p, g, lab)
    gg, back = M.read_labels(p)
    assert gg == g and np.array_equal(back, lab)
    M.write_field(p, g, fld)
    gg, back = M.read_field(p)
    assert gg == g and np.array_equal(back, fld)
    h = M.read_header(p)
    r = R.read_header(p)
    assert h["channels"] == r["channels"] == g.ndim
    assert h["element_type_name"] == r["element_type"] == "MET_FLOAT"
    assert os.path.samefile(h["raw_path"], r["raw_path"])


def _hdr(tmp_path, text, payload=None, name="h.mhd"):
    p = str(tmp_path / name)
    open(p, "w").write(text)
    if payload is not None:
        payload.tofile(str(tmp_path / "h.raw"))
    return p


GOOD = ("NDims = 3\nDimSize = 4 3 2\nElementType = MET_FLOAT\nElementDataFile = h.raw\n")


def test_reader_acceptance(tmp_path):
    # optional keys absent, extra blank lines / whitespace, CRLF, absolute data path
    data = np.arange(24, dtype=np.float32)
    p = _hdr(tmp_path, "\n  " + GOOD.replace("\n", "\r\n") + "\n\n", data)
    g, img = M.read_image(p)
    assert g.dims == (4, 3, 2) and g.spacing == (1.0, 1.0, 1.0) and g.origin == (0.0, 0.0, 0.0)
    assert np.array_equal(img.ravel(), data)
    absraw = str(tmp_path / "h.raw")
    p = _hdr(tmp_path, GOOD.replace("h.raw", absraw), name="abs.mhd")
    assert np.array_equal(M.read_image(p)[1].ravel(), data)


BAD = [
    ("NDims = 3\nDimSize 4 3 2\n", None),
    ("NDims = 3\n = 4\n", None),
    ("DimSize = 4 3 2\nElementType = MET_FLOAT\nElementDataFile = h.raw\n", None),
    ("NDims = 4\nDimSize = 4 3 2 1\n", None),
    ("NDims = 3\nDimSize = 4 3\nElementType = MET_FLOAT\nElementDataFile = h.raw\n", None),
    ("NDims = 3\nDimSize = 4 x 2\nElementType = MET_FLOAT\nElementDataFile = h.raw\n", None),
    ("NDims = 3\nDimSize = 4 3.5 2\nElementType = MET_FLOAT\nElementDataFile = h.raw\n", None),
    ("NDims = 3\nDimSize = 4 1 2\nElementType = MET_FLOAT\nElementDataFile = h.raw\n", None),
    ("NDims = 3\nDimSize = 4 3 2\nElementSpacing = 1 0 1\nElementType = MET_FLOAT\n"
     "ElementDataFile = h.raw\n", None),
    ("NDims = 3\nDimSize = 4 3 2\nElementDataFile = h.raw\n", None),
    ("NDims = 3\nDimSize = 4 3 2\nElementType = MET_FLOAT\nElementDataFile = LOCAL\n", None),
    ("NDims = 3\nDimSize = 4 3 2\nElementType = MET_FLOAT\nElementNumberOfChannels = 0\n"
     "ElementDataFile = h.raw\n", None),
]


@pytest.mark.parametrize("k", range(len(BAD)))
def test_header_errors_match_reference_messages(tmp_path, k):
    text, _ = BAD[k]
    p = _hdr(tmp_path, text)
    with pytest.raises(R.InvalidArgument) as want:
        R.read_header(p)
    with pytest.raises(A.InvalidArgument) as got:
        M.read_header(p)
    assert str(got.value).endswith(str(want.value)), (str(got.value), str(want.value))


def test_typed_reader_errors(tmp_path):
    data = np.arange(24, dtype=np.float32)
    p = _hdr(tmp_path, GOOD, data[:23])  # short payload
    with pytest.raises(A.InvalidArgument, match="payload is 92 bytes, expected 96"):
        M.read_image(p)
    p = _hdr(tmp_path, GOOD, data)
    with pytest.raises(A.InvalidArgument, match="expected ElementType MET_SHORT, got MET_FLOAT"):
        M.read_labels(p)
    with pytest.raises(A.InvalidArgument, match="field needs 3 channels, got 1"):
        M.read_field(p)
    g = A.GridMeta.make_3d(4, 3, 2)
    with pytest.raises(A.InvalidArgument, match="does not fit MET_SHORT"):
        M.write_labels(str(tmp_path / "l.mhd"), g, np.full(g.shape, 40000, np.int32))
