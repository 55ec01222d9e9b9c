"""Hyperparameter grid sweep (pipeline.hpp:75-104, pipeline.cpp:226-313) on GPUs.

The paper's sweep use case: every (eta, sigma_warp,
sigma_grad) config registers every pair; metric = final loss or overlap TO
mean.  `sweep()` runs the native dfm_sweep on this process's GPUs (worker
contexts pulling configs from a shared counter); `sweep_distributed()` shards
the config index space over torch.distributed ranks (one per GPU, configs are
independent: no collective on the data path) and gathers the rows on rank 0.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Callable, List, Optional, Sequence

import numpy as np

from . import _abi as A


@dataclass
class SweepPair:
    """difform::SweepPair: fixed/moving on one grid, optional label maps."""
    grid: A.GridMeta
    fixed: np.ndarray
    moving: np.ndarray
    fixed_labels: Optional[np.ndarray] = None
    moving_labels: Optional[np.ndarray] = None
    name: str = ""


@dataclass
class SweepRow:
    eta: float
    sigma_warp: float
    sigma_grad: float
    metric_mean: float = 0.0
    metric_sd: float = 0.0
    wall_ms: float = 0.0
    failed: bool = False
    error: str = ""


@dataclass
class SweepResult:
    rows: List[SweepRow]
    etas: List[float]
    sigma_warps: List[float]
    sigma_grads: List[float]
    heatmaps: list = field(default_factory=list)  # [eta][sigma_warp][sigma_grad]


def config_axes(k: int, n_sw: int, n_sg: int):
    """config k -> (eta, sigma_warp, sigma_grad) indices (pipeline.cpp:254-257)."""
    return k // (n_sg * n_sw), (k // n_sg) % n_sw, k % n_sg


def heatmaps(rows, n_eta, n_sw, n_sg):
    h = [[[0.0] * n_sg for _ in range(n_sw)] for _ in range(n_eta)]
    for k, r in enumerate(rows):
        ei, wi, gi = config_axes(k, n_sw, n_sg)
        h[ei][wi][gi] = r.metric_mean
    return h


def _marshal(pairs: Sequence[SweepPair]):
    keep, arr = [], (A.dfm_sweep_pair * len(pairs))()
    for i, p in enumerate(pairs):
        g = p.grid.c()
        f = A.as_f64(p.fixed, p.grid.shape)
        m = A.as_f64(p.moving, p.grid.shape)
        keep += [g, f, m]
        arr[i].grid = C.cast(C.pointer(g), C.c_void_p)
        arr[i].fixed = A._dptr(f)
        arr[i].moving = A._dptr(m)
        for name in ("fixed_labels", "moving_labels"):
            lab = getattr(p, name)
            if lab is not None:
                la = np.ascontiguousarray(lab, dtype=np.int32).ravel()
                keep.append(la)
                setattr(arr[i], name, la.ctypes.data_as(C.POINTER(C.c_int32)))
    return arr, keep


def _rows_out(crow, n_cfg, only_computed=False):
    out = []
    for k in range(n_cfg):
        r = crow[k]
        if only_computed and not r.computed:
            out.append(None)
            continue
        out.append(SweepRow(r.eta, r.sigma_warp, r.sigma_grad, r.metric_mean, r.metric_sd,
                            r.wall_ms, bool(r.failed), r.error.decode(errors="replace")))
    return out


def _metric_code(metric) -> int:
    return {"loss": A.SWEEP_LOSS, "overlap": A.SWEEP_OVERLAP}.get(metric, metric)


def run_native(pairs, base: A.RegistrationConfig, sched: A.PyramidSchedule, etas, sigma_warps,
               sigma_grads, metric="loss", precision="f32", devices=(0,), workers_per_device=1,
               shard=(0, 1)):
    """dfm_sweep on this process's devices; rows outside the shard are None."""
    from .engine import load_library
    lib = load_library()
    arr, keep = _marshal(pairs)
    s, it = A.schedule_arrays(sched)
    e = np.ascontiguousarray(etas, dtype=np.float64)
    w = np.ascontiguousarray(sigma_warps, dtype=np.float64)
    gsg = np.ascontiguousarray(sigma_grads, dtype=np.float64)
    n_cfg = len(e) * len(w) * len(gsg)
    rows = (A.dfm_sweep_row * max(n_cfg, 1))()
    dev = (C.c_int * len(devices))(*devices)
    prec = {"f32": A.PREC_F32, "f64": A.PREC_F64}[precision]
    cc = base.c()
    f = lib.dfm_sweep
    f.restype = C.c_int
    rc = f(dev, len(devices), int(workers_per_device), prec, arr, len(pairs), C.byref(cc),
           A._dptr(s), it.ctypes.data_as(C.POINTER(C.c_int32)), len(s), A._dptr(e), len(e),
           A._dptr(w), len(w), A._dptr(gsg), len(gsg), _metric_code(metric),
           C.c_int64(shard[0]), C.c_int64(shard[1]), rows)
    A.CallTable(lib, "dfm_").check(rc, "sweep")
    del keep
    return _rows_out(rows, n_cfg, only_computed=True)


def merge_shards(shards: Sequence[Sequence[Optional[SweepRow]]]) -> List[SweepRow]:
    """Union of per-rank row lists (each config computed by exactly one rank)."""
    n = len(shards[0])
    out = [None] * n
    for rows in shards:
        for k, r in enumerate(rows):
            if r is not None:
                if out[k] is not None:
                    raise RuntimeError(f"sweep: config {k} computed by two ranks")
                out[k] = r
    missing = [k for k, r in enumerate(out) if r is None]
    if missing:
        raise RuntimeError(f"sweep: configs {missing} not computed by any rank")
    return out


def sweep(pairs, base, sched, etas, sigma_warps, sigma_grads, metric="loss", precision="f32",
          devices=(0,), workers_per_device=1) -> SweepResult:
    """One process, all of `devices`."""
    rows = run_native(pairs, base, sched, etas, sigma_warps, sigma_grads, metric, precision,
                      devices, workers_per_device)
    res = SweepResult(rows, list(etas), list(sigma_warps), list(sigma_grads))
    res.heatmaps = heatmaps(rows, len(etas), len(sigma_warps), len(sigma_grads))
    return res


def sweep_distributed(pairs, base, sched, etas, sigma_warps, sigma_grads, metric="loss",
                      precision="f32", workers_per_device=1,
                      runner: Optional[Callable] = None) -> Optional[SweepResult]:
    """torch.distributed: rank r computes configs k = r (mod world) on its local
    GPU; rank 0 returns the merged result (None elsewhere).  `runner(shard)`
    replaces the native call (CPU tests of the sharding with gloo)."""
    import os
    import torch.distributed as dist
    rank, world = dist.get_rank(), dist.get_world_size()
    local = int(os.environ.get("LOCAL_RANK", rank))
    if runner is None:
        def runner(shard):
            return run_native(pairs, base, sched, etas, sigma_warps, sigma_grads, metric,
                              precision, (local,), workers_per_device, shard)
    mine = runner((rank, world))
    gathered = [None] * world
    dist.all_gather_object(gathered, mine)
    if rank != 0:
        return None
    rows = merge_shards(gathered)
    res = SweepResult(rows, list(etas), list(sigma_warps), list(sigma_grads))
    res.heatmaps = heatmaps(rows, len(etas), len(sigma_warps), len(sigma_grads))
    return res
