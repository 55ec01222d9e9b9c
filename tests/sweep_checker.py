"""Drives the CPU checkers' sweep (the restatement's orc_sweep, the reference's
dfmref_sweep) with the product's row layout — test infrastructure only."""
import ctypes as C

import numpy as np

from paper_2404_01249_b200 import _abi as A
from paper_2404_01249_b200.sweep import _marshal, _metric_code, _rows_out


def run_checker(checker, pairs, base, sched, etas, sigma_warps, sigma_grads, metric="loss",
                workers=1):
    """The CPU checkers (restatement `orc_sweep` or the reference
    `dfmref_sweep`) with the same row layout — test infrastructure only."""
    lib = checker.t.lib
    arr, keep = _marshal(pairs)
    s, it = A.schedule_arrays(sched)
    e = np.ascontiguousarray(etas, dtype=np.float64)
    w = np.ascontiguousarray(sigma_warps, dtype=np.float64)
    gsg = np.ascontiguousarray(sigma_grads, dtype=np.float64)
    n_cfg = len(e) * len(w) * len(gsg)
    rows = (A.dfm_sweep_row * max(n_cfg, 1))()
    cc = base.c()
    args = [arr, len(pairs), C.byref(cc), A._dptr(s), it.ctypes.data_as(C.POINTER(C.c_int32)),
            len(s), A._dptr(e), len(e), A._dptr(w), len(w), A._dptr(gsg), len(gsg),
            _metric_code(metric)]
    if checker.kind == "reference":
        rc = lib.dfmref_sweep(*args, int(workers), rows)
    else:
        rc = lib.orc_sweep(*args, rows)
    checker.t.check(rc, "sweep")
    del keep
    return _rows_out(rows, n_cfg)
