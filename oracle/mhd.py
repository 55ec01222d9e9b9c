"""oracle/mhd.py — TEST INFRASTRUCTURE ONLY.

Python restatement of the reference's MetaImage writer and header reader
(io.cpp:22-26 fmt, 117-140 write_mhd_header, 152-216 read_mhd_header,
218-226 read_raw_exact, 245-328 typed readers/writers).  The reference's
io.cpp itself is not buildable here (it needs nlohmann/json and OpenSSL, both
absent from the reference tree), so MHD parity is pinned to this restatement.
"""
from __future__ import annotations

import math
import os

import numpy as np


class InvalidArgument(ValueError):
    pass


def fmt17(v: float) -> str:
    return "%.17g" % v


def header_text(mhd_path, ndim, dims, spacing, origin, element_type, channels=1) -> str:
    raw = os.path.splitext(os.path.basename(mhd_path))[0] + ".raw"
    t = "ObjectType = Image\n"
    t += f"NDims = {ndim}\n"
    t += "DimSize =" + "".join(f" {int(d)}" for d in dims[:ndim]) + "\n"
    t += "ElementSpacing =" + "".join(" " + fmt17(s) for s in spacing[:ndim]) + "\n"
    t += "Offset =" + "".join(" " + fmt17(o) for o in origin[:ndim]) + "\n"
    t += f"ElementType = {element_type}\n"
    if channels > 1:
        t += f"ElementNumberOfChannels = {channels}\n"
    t += f"ElementDataFile = {raw}\n"
    return t


def parse_lines(text: str, path: str):
    out, pos = [], 0
    while pos < len(text):
        eol = text.find("\n", pos)
        end = len(text) if eol < 0 else eol
        line = text[pos:end].strip(" \t\r\n")
        if line:
            if "=" not in line:
                raise InvalidArgument(f"{path}: byte {pos}: expected 'Key = value'")
            k, v = line.split("=", 1)
            k, v = k.strip(" \t\r\n"), v.strip(" \t\r\n")
            if not k:
                raise InvalidArgument(f"{path}: byte {pos}: empty key")
            out.append((k, v, pos))
        pos = len(text) if eol < 0 else eol + 1
    return out


def _numbers(h, expect, path):
    k, v, off = h
    vals, toks = [], v.split()
    for i, tok in enumerate(toks):
        try:
            vals.append(float(tok))
        except ValueError:
            raise InvalidArgument(f"{path}: byte {off}: non-numeric token in '{k}'")
    if len(vals) != expect:
        raise InvalidArgument(f"{path}: byte {off}: '{k}' needs {expect} values")
    return vals


def read_header(path: str) -> dict:
    lines = parse_lines(open(path, "rb").read().decode("latin-1"), path)
    find = {k: (k, v, off) for k, v, off in reversed(lines)}

    def need(k):
        if k not in find:
            raise InvalidArgument(f"{path}: byte 0: missing required key '{k}'")
        return find[k]

    nd = need("NDims")
    ndv = _numbers(nd, 1, path)[0]
    if ndv not in (2.0, 3.0):
        raise InvalidArgument(f"{path}: byte {nd[2]}: NDims must be 2 or 3")
    ndim = int(ndv)
    dims, spacing, origin = [1, 1, 1], [1.0, 1.0, 1.0], [0.0, 0.0, 0.0]
    ds = need("DimSize")
    for a, d in enumerate(_numbers(ds, ndim, path)):
        if d < 1 or d != math.floor(d):
            raise InvalidArgument(f"{path}: byte {ds[2]}: DimSize entries must be positive integers")
        dims[a] = int(d)
    if "ElementSpacing" in find:
        spacing[:ndim] = _numbers(find["ElementSpacing"], ndim, path)
    if "Offset" in find:
        origin[:ndim] = _numbers(find["Offset"], ndim, path)
    for a in range(ndim):
        if dims[a] < 2:
            raise InvalidArgument(f"{path}: byte 0: grid dims must be >= 2 per axis")
        if not (spacing[a] > 0.0) or not math.isfinite(spacing[a]):
            raise InvalidArgument(f"{path}: byte 0: grid spacing must be > 0")
    et = need("ElementType")[1]
    channels = 1
    if "ElementNumberOfChannels" in find:
        ch = find["ElementNumberOfChannels"]
        c = _numbers(ch, 1, path)[0]
        if c < 1 or c != math.floor(c):
            raise InvalidArgument(f"{path}: byte {ch[2]}: ElementNumberOfChannels must be a "
                                  "positive integer")
        channels = int(c)
    df = need("ElementDataFile")
    if df[1] in ("", "LOCAL"):
        raise InvalidArgument(f"{path}: byte {df[2]}: embedded payloads are not supported")
    raw = df[1] if os.path.isabs(df[1]) else os.path.join(os.path.dirname(path), df[1])
    return dict(ndim=ndim, dims=tuple(dims), spacing=tuple(spacing), origin=tuple(origin),
                element_type=et, channels=channels, raw_path=raw)


def write(path, ndim, dims, spacing, origin, data, element_type="MET_FLOAT", channels=1):
    with open(path, "w") as f:
        f.write(header_text(path, ndim, dims, spacing, origin, element_type, channels))
    dt = np.float32 if element_type == "MET_FLOAT" else np.int16
    np.ascontiguousarray(data, dtype=dt).tofile(os.path.splitext(path)[0] + ".raw")
