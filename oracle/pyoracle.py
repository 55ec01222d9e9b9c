"""oracle/pyoracle.py — TEST INFRASTRUCTURE ONLY.

Python handles on the two CPU checkers, with the same numpy-level API as the
product's HostAPI (paper_2404_01249_b200/_abi.py):

  * ``port()``      — oracle/_build/liboracle.so, the plain-C fp64 restatement
                      (oracle/difform_oracle.c), always buildable with gcc;
  * ``reference()`` — oracle/_ref/libdifform_ref.so, the UNMODIFIED reference
                      sources compiled in place (oracle/Makefile `ref`); only
                      present when built in the container that has
                      /root/reference (it travels to the GPU box as a file).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

from paper_2404_01249_b200 import _abi as A

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "_build", "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libdifform_ref.so")
REF_FMA_SO = os.path.join(HERE, "_ref", "libdifform_ref_fma.so")


def build(ref: bool = True) -> None:
    """Builds the restatement and, when /root/reference exists, the reference."""
    targets = ["port"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets += ["ref", "ref-fma", "accept"]  # accept: after libdifform_b200.so
    subprocess.check_call(["make", "-s", "-C", HERE] + targets)


class Oracle(A.HostAPI):
    """A CPU checker: HostAPI over a ctx-less C-ABI + register_images."""

    def __init__(self, so_path: str, prefix: str, kind: str):
        lib = C.CDLL(so_path)
        super().__init__(A.CallTable(lib, prefix, ctx=None, err_fn=prefix + "last_error"))
        self.kind = kind  # "port" or "reference"
        self.path = so_path
        reg = getattr(lib, prefix + "register")
        reg.restype = C.c_int
        reg.argtypes = [C.POINTER(A.dfm_grid), C.POINTER(C.c_double), C.POINTER(C.c_double),
                        C.POINTER(A.dfm_config), C.POINTER(C.c_double), C.POINTER(C.c_int32),
                        C.c_int32, C.POINTER(A.dfm_init), C.POINTER(C.c_double),
                        C.POINTER(A.dfm_iter_record), C.c_int64, C.POINTER(A.dfm_runlog)]
        self._reg = reg
        od = getattr(lib, prefix + "overlap_dice")
        od.restype = C.c_int
        od.argtypes = [C.POINTER(A.dfm_grid), C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                       C.POINTER(C.c_double), C.POINTER(C.c_double)]
        self._od = od

    def register_images(self, g: A.GridMeta, fixed, moving, cfg: A.RegistrationConfig,
                        sched: A.PyramidSchedule, init=None):
        """register_images (pipeline.cpp:121-224) -> (field, RunLog)."""
        fixed = A.as_f64(fixed, g.shape)
        moving = A.as_f64(moving, g.shape)
        s, it = A.schedule_arrays(sched)
        cap = int(it.sum()) + 1
        recs = (A.dfm_iter_record * cap)()
        rl = A.dfm_runlog()
        out = np.empty(g.field_shape)
        ci, keep = A.make_init(init, g.ndim)
        cc = cfg.c()
        rc = self._reg(C.byref(g.c()), A._dptr(fixed), A._dptr(moving), C.byref(cc),
                       A._dptr(s), it.ctypes.data_as(C.POINTER(C.c_int32)), len(s),
                       C.byref(ci), A._dptr(out), recs, cap, C.byref(rl))
        self.t.check(rc, "register")
        del keep
        return out, A.records_to_log(recs, rl)

    def overlap_dice(self, g: A.GridMeta, warped, fixed):
        """(MO mean, MO Klein) of overlap_report (analysis.cpp:169-247)."""
        w = np.ascontiguousarray(warped, dtype=np.int32)
        f = np.ascontiguousarray(fixed, dtype=np.int32)
        a, b = C.c_double(), C.c_double()
        rc = self._od(C.byref(g.c()), w.ctypes.data_as(C.POINTER(C.c_int32)),
                      f.ctypes.data_as(C.POINTER(C.c_int32)), C.byref(a), C.byref(b))
        self.t.check(rc, "overlap_dice")
        return a.value, b.value


_cache = {}


def port() -> Oracle:
    if "port" not in _cache:
        if not os.path.exists(PORT_SO):
            build(ref=False)
        _cache["port"] = Oracle(PORT_SO, "orc_", "port")
    return _cache["port"]


def reference_available() -> bool:
    return os.path.exists(REF_SO)


def reference() -> Oracle:
    if "ref" not in _cache:
        if not reference_available():
            raise FileNotFoundError(f"{REF_SO} not built (needs /root/reference at build time)")
        _cache["ref"] = Oracle(REF_SO, "dfmref_", "reference")
    return _cache["ref"]


def reference_fma() -> Oracle:
    """The same unmodified reference built with FMA contraction: a rounding
    change of the reference itself (its divergence from reference() is the
    conditioning envelope of the chaotic LNCC loop)."""
    if "ref_fma" not in _cache:
        if not os.path.exists(REF_FMA_SO):
            raise FileNotFoundError(f"{REF_FMA_SO} not built (make -C oracle ref-fma)")
        _cache["ref_fma"] = Oracle(REF_FMA_SO, "dfmref_", "reference-fma")
    return _cache["ref_fma"]


def best() -> Oracle:
    """The reference itself when built, else the restatement."""
    return reference() if reference_available() else port()
