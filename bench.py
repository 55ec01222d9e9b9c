#!/usr/bin/env python
"""Benchmark: full 3-scale LNCC diffeomorphic registration of BASELINE config 1
(160x192x224 fp32 pair, scales 4/2/1 x 200/100/50 iterations, early stop off).

One "step" = one complete registration of one pair.  Under torchrun each rank
registers its own pair (pairs shard with no data-path collective: weak
scaling); `value` = all ranks' voxel-iterations / max-over-ranks device time.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--precision f32|f64]
                    [--impl ours|reference] [--config 1|0|3]

Prints ONE JSON line on rank 0 (contract in the task statement / DESIGN.md §6).
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS = os.path.join(ROOT, "MEASURED_PEAKS.json")
FALLBACK_HBM = 6650.0  # GB/s, B200_PROFILING.md fallback

# algorithmic (compulsory) bytes per voxel per launch of each kernel class of
# the plane-streaming LNCC loop, in elements (fp32 4 B, fp64 8 B); DESIGN.md §4.
ALG_ELEMS = {
    "loss_fwd": 2 + 4,              # read F, W; write 4 window coefficients
    "lncc_bwd": 4 + 1 + 1 + 3 + 3,  # read 4 coef, F, W, G(3); write grad(3)
    "smooth_adam": 3 + 3 + 3 + 3 + 3 + 3,  # read grad m nu; write m nu step
    "compose_smooth": 3 + 3 + 1 + 3 + 1 + 3,  # read step u M; write u' W G(3)
}
# fixed extra bytes per voxel independent of the precision: the forward reads
# the level's precomputed F window statistics (muF, vF as fp64)
ALG_EXTRA_BYTES = {"loss_fwd": 16}
# the iteration's irreducible state traffic: read u m nu F M,
# write u m nu = 20 elements (80 B fp32)
ITER_MIN_ELEMS = 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--precision", default="f32", choices=["f32", "f64"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=1, choices=[0, 1, 3])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-f64", action="store_true",
                    help="skip the fp64 (parity-mode) sub-record")
    ap.add_argument("--pairs-per-gpu", type=int, default=1,
                    help="config-2 style batch: K concurrent pairs per GPU, one context "
                         "(stream) and host thread each; value = aggregate voxel-iter/s")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    return rank, world, local


def voxel_iters(pair) -> int:
    from paper_2404_01249_b200 import engine  # noqa: F401
    from paper_2404_01249_b200 import _abi as A
    import math
    total = 0
    for s, it in zip(pair.schedule.scales, pair.schedule.iterations):
        dims = [math.ceil(d / s) for d in pair.grid.dims]
        total += it * dims[0] * dims[1] * dims[2]
    return total


class ClockSampler:
    """SM clocks + throttle reasons sampled during the timed region: NVML in a
    thread (every 10 ms, plus one sample when the region starts and one when it
    ends, so even a short region is covered); nvidia-smi if NVML is missing."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    # NVML clocks-event reason bits
    BITS = {"hw_slowdown": 0x8, "hw_thermal_slowdown": 0x40, "sw_thermal_slowdown": 0x20,
            "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self.thread = None
        self.nvml = None
        self.stop_evt = threading.Event()

    def _nvml_sample(self):
        nv, h = self.nvml
        sm = nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM)
        mx = nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM)
        try:
            rs = nv.nvmlDeviceGetCurrentClocksEventReasons(h)
        except AttributeError:
            rs = nv.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append((float(sm), float(mx), int(rs)))

    def _nvml_loop(self):
        while not self.stop_evt.wait(0.01):
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001 - sampling must never break the bench
                return

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            vis = [v.strip() for v in os.environ.get("CUDA_VISIBLE_DEVICES", "").split(",")]
            dev = (int(vis[self.device]) if len(vis) > self.device and
                   all(v.isdigit() for v in vis) else self.device)
            self.nvml = (nv, nv.nvmlDeviceGetHandleByIndex(dev))
            self._nvml_sample()
            self.thread = threading.Thread(target=self._nvml_loop, daemon=True)
            self.thread.start()
            return
        except Exception:  # noqa: BLE001
            self.nvml = None
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except OSError:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def stop(self):
        if self.nvml:
            self.stop_evt.set()
            if self.thread:
                self.thread.join(timeout=2)
            try:
                self._nvml_sample()
            except Exception:  # noqa: BLE001
                pass
            sm = [r[0] for r in self.rows]
            reasons = sorted({nm for r in self.rows for nm, bit in self.BITS.items()
                              if r[2] & bit})
            return {"sm_mhz": float(np.median(sm)) if sm else None,
                    "sm_max_mhz": max(r[1] for r in self.rows) if self.rows else None,
                    "reasons": reasons, "samples": len(sm), "source": "nvml"}
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = set()
        for r in self.rows:
            if len(r) >= 8:
                for k, nm in enumerate(names):
                    if r[4 + k].lower() == "active":
                        reasons.add(nm)
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": sorted(reasons),
                "samples": len(sm), "source": "nvidia-smi"}


def hbm_peak():
    try:
        with open(PEAKS) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return FALLBACK_HBM, "fallback"


def cpu_model_name() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.lower().startswith("model name"):
                return line.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return "unknown"


SAMPLE_ITERS = (8, 4, 2)


def cpu_leg(pair, kind_pref="reference", sample_iters=SAMPLE_ITERS):
    """The reference CPU path (oracle/_ref, else the C restatement) on all host
    cores, reported for the SAME schedule as the GPU line: one bounded sample
    registration (same pair, same scales, `sample_iters` iterations) gives
    per-level per-iteration times (the reference's own IterationRecord.wall_ms,
    pipeline.cpp:159-209, median per level) and the one-off work (pyramid,
    level transitions, final full-resolution loss + fold check: RunLog.total_ms
    minus the iterations, pipeline.cpp:140-153, 213-223); the full-schedule
    time is one-offs + sum over levels of iterations x per-iteration time.
    tools/cpu_model_check.py validates this model against real full-schedule
    runs (profiles/r2_cpu_model_check_*.json)."""
    ncores = os.cpu_count() or 1
    os.environ["DIFFORM_THREADS"] = str(ncores)
    from oracle import pyoracle
    o = pyoracle.reference() if (kind_pref == "reference" and
                                 pyoracle.reference_available()) else pyoracle.port()
    from paper_2404_01249_b200 import _abi as A
    sched = A.PyramidSchedule(pair.schedule.scales, sample_iters)
    t0 = time.perf_counter()
    _, log = o.register_images(pair.grid, pair.fixed, pair.moving, pair.config, sched)
    dt = time.perf_counter() - t0
    per_level = []
    for si in range(len(sched.scales)):
        w = [r.wall_ms for r in log.iterations if r.scale_index == si]
        per_level.append(float(np.median(w)) if w else 0.0)
    oneoff_ms = log.total_ms - sum(r.wall_ms for r in log.iterations)
    model_ms = oneoff_ms + sum(n * t for n, t in zip(pair.schedule.iterations, per_level))
    vi = voxel_iters(pair)
    return {"value": vi / (model_ms / 1e3), "unit": "voxel-iter/s",
            "cores": ncores if o.kind == "reference" else 1, "kind": o.kind,
            "cpu_model": cpu_model_name(),
            "s_per_pair": model_ms / 1e3,
            "per_level_iter_ms": per_level, "oneoff_ms": oneoff_ms,
            "schedule": list(pair.schedule.iterations),
            "sample": (f"{pair.name}: same-schedule model from one registration with the same "
                       f"scales and {'/'.join(map(str, sample_iters))} iterations ({dt:.1f} s): "
                       f"one-offs {oneoff_ms / 1e3:.2f} s + "
                       + " + ".join(f"{n} x {t:.1f} ms" for n, t in
                                    zip(pair.schedule.iterations, per_level))
                       + f" = {model_ms / 1e3:.1f} s per pair"),
            "sample_seconds": dt}


def workload_config(pair, world):
    """The `config` object both arms print (same workload, same keys)."""
    from paper_2404_01249_b200 import _abi as A
    cfg = pair.config
    return {"workload": pair.name, "shape_xyz": list(pair.grid.dims),
            "scales": list(pair.schedule.scales), "iterations": list(pair.schedule.iterations),
            "loss": f"lncc r={cfg.lncc_radius}" if cfg.loss == A.LOSS_LNCC else "ssd",
            "sigma_grad": cfg.sigma_grad, "sigma_warp": cfg.sigma_warp, "eta": cfg.eta,
            "early_stop": "off (conv_window > max iterations)",
            "voxel_iters_per_pair": voxel_iters(pair),
            "l2": l2_note(pair)}


def l2_note(pair) -> str:
    """Whether the timed pair's working set exceeds the 126 MB L2 (inputs
    larger than L2 need no flush between timed iterations)."""
    gb = 30 * 4 * pair.grid.voxel_count / 1e9  # ~30 fp32 volumes
    if gb > 0.126:
        return f"working set ~{gb:.2f} GB per pair >> 126 MB L2 (no flush needed)"
    return (f"working set ~{gb * 1e3:.0f} MB per pair fits the 126 MB L2 (coarse levels "
            "are L2-resident by design; no flush between steps)")


def run_reference_arm(args, rank, world):
    """The reference's own CPU implementation (oracle/_ref: the unmodified
    sources compiled in place) on rank 0 with every host core; other ranks
    exit without work.  Each step = one bounded sample registration; value =
    the same-schedule (200/100/50) rate of cpu_leg's model."""
    if rank != 0:
        return
    from paper_2404_01249_b200 import synth
    pair = synth.make_pair(args.config, seed=0)
    vals, secs, pairs_s = [], [], []
    cb = None
    for k in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        cb = cpu_leg(pair, "reference", (4, 2, 1) if k < args.warmup else SAMPLE_ITERS)
        if k >= args.warmup:
            secs.append(time.perf_counter() - t0)
            vals.append(cb["value"])
            pairs_s.append(cb["s_per_pair"])
    v = float(np.mean(vals))
    cb["value"] = v
    cb["s_per_pair"] = float(np.mean(pairs_s))
    cb["sample"] = (f"mean of {len(pairs_s)} samples ({', '.join(f'{x:.1f}' for x in pairs_s)} "
                    f"s per pair); last: " + cb["sample"])
    line = {"impl": "reference", "metric": "voxel-iterations/sec", "value": v,
            "unit": "voxel-iter/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": float(np.mean(secs)) * 1e3,
            "s_per_pair": cb["s_per_pair"],
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config recipe, seeded)",
            "config": workload_config(pair, world),
            "note": ("each timed step is one bounded sample registration "
                     f"({'/'.join(map(str, SAMPLE_ITERS))} iterations, ms_per_step is its wall "
                     "time); value and s_per_pair are the same-schedule model (cpu_baseline)"),
            "cpu_baseline": cb,
            "e2e": {"value": v, "unit": "voxel-iter/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_batch(args, rank, world, local):
    """K independent pairs per GPU registered concurrently (config 2's batch
    of pairs; the reference's sweep worker pattern with streams): device time
    from one start event to the last context's end event, max over ranks."""
    import threading
    import torch
    from paper_2404_01249_b200 import synth
    from paper_2404_01249_b200.engine import Context
    K = args.pairs_per_gpu
    pairs = [synth.make_pair(args.config, seed=rank * K + k) for k in range(K)]
    tdt = torch.float32 if args.precision == "f32" else torch.float64
    dev = f"cuda:{local}"
    bufs = [(torch.from_numpy(p.fixed.astype(np.float32)).to(dev, dtype=tdt),
             torch.from_numpy(p.moving.astype(np.float32)).to(dev, dtype=tdt),
             torch.empty((3,) + p.grid.shape, dtype=tdt, device=dev)) for p in pairs]
    ctxs = [Context(local, args.precision) for _ in range(K)]
    streams = [torch.cuda.ExternalStream(c.stream_ptr, device=dev) for c in ctxs]

    def run(k, n):
        c, p, (F, M, o) = ctxs[k], pairs[k], bufs[k]
        for _ in range(n):
            c.register_device(p.grid, F.data_ptr(), M.data_ptr(), p.config, p.schedule,
                              o.data_ptr())

    def all_threads(n):
        th = [threading.Thread(target=run, args=(k, n)) for k in range(K)]
        for t in th:
            t.start()
        for t in th:
            t.join()

    all_threads(args.warmup)
    vi = voxel_iters(pairs[0])
    clocks = ClockSampler(local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = sum(c.launch_count for c in ctxs)
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for st in streams:
        st.wait_event(e0)
    all_threads(args.steps)
    ends = []
    for st in streams:
        e = torch.cuda.Event(enable_timing=True)
        e.record(st)
        ends.append(e)
    torch.cuda.synchronize()
    ms = max(e0.elapsed_time(e) for e in ends) / args.steps
    launches = sum(c.launch_count for c in ctxs) - l0
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    clk = clocks.stop()
    for c in ctxs:
        c.close()
    if rank == 0:
        line = {"metric": "voxel-iterations/sec", "value": world * K * vi / (ms / 1e3),
                "unit": "voxel-iter/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms,
                "pairs_per_s": world * K / (ms / 1e3), "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": args.precision,
                "data": "synthetic (BASELINE config recipe, seeded per pair)",
                "config": {"workload": pairs[0].name + "_batch", "pairs_per_gpu": K,
                           "shape_xyz": list(pairs[0].grid.dims),
                           "note": "one step = K concurrent pairs per GPU"},
                "gpu_launches": launches, "clocks": clk}
        print(json.dumps(line), flush=True)


def spawn_ranks(args) -> int:
    """`--gpus N` without a launcher: start N ranks (one per GPU) through
    torch.distributed.run on 127.0.0.1 and return their exit code."""
    if args.impl == "ours":
        import torch
        n = torch.cuda.device_count()
        if n < args.gpus:
            print(f"bench.py --gpus {args.gpus}: only {n} CUDA device(s) visible",
                  file=sys.stderr)
            return 2
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args))
    rank, world, local = dist_env()
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        # the reference is a CPU library: rank 0 alone runs, the others exit
        run_reference_arm(args, rank, world)
        return
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")

    import torch
    torch.cuda.set_device(local)
    from paper_2404_01249_b200 import synth, _abi as A
    from paper_2404_01249_b200.engine import Context

    if args.pairs_per_gpu > 1:
        return run_batch(args, rank, world, local)
    pair = synth.make_pair(args.config, seed=rank)
    g = pair.grid
    cfg = pair.config
    sched = pair.schedule
    ctx = Context(local, args.precision)
    tdt = torch.float32 if args.precision == "f32" else torch.float64
    F = torch.from_numpy(pair.fixed.astype(np.float32)).to(f"cuda:{local}", dtype=tdt)
    M = torch.from_numpy(pair.moving.astype(np.float32)).to(f"cuda:{local}", dtype=tdt)
    out = torch.empty((3,) + g.shape, dtype=tdt, device=f"cuda:{local}")
    torch.cuda.synchronize()
    stream = torch.cuda.ExternalStream(ctx.stream_ptr, device=f"cuda:{local}")

    def step():
        return ctx.register_device(g, F.data_ptr(), M.data_ptr(), cfg, sched, out.data_ptr())

    for _ in range(args.warmup):
        log = step()
    vi = voxel_iters(pair)

    # ---- timed region: device-resident inputs
    clocks = ClockSampler(local)
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    torch.cuda.synchronize()
    clocks.start()
    l0 = ctx.launch_count
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(args.steps):
        log = step()
    e1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launch_count - l0
    ms = e0.elapsed_time(e1) / args.steps
    if world > 1:
        import torch.distributed as dist
        t = torch.tensor([ms], device=f"cuda:{local}")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    clk = clocks.stop()
    value = world * vi / (ms / 1e3)

    # ---- end to end through the host C-ABI (pinned host buffers, H2D + D2H inside)
    e2e = None
    if not args.no_e2e:
        hf = torch.from_numpy(pair.fixed.astype(np.float32)).pin_memory()
        hm = torch.from_numpy(pair.moving.astype(np.float32)).pin_memory()
        hout = torch.empty(g.field_shape, dtype=torch.float32).pin_memory()
        import ctypes as C
        s, it = A.schedule_arrays(sched)
        cap = int(it.sum()) + 1
        recs = (A.dfm_iter_record * cap)()
        rl = A.dfm_runlog()
        cc = cfg.c()
        ci, _ = A.make_init(None, 3)
        gc = g.c()

        def e2e_step():
            rc = ctx.lib.dfm_register(ctx.handle, C.byref(gc), hf.data_ptr(), hm.data_ptr(),
                                      A.HOST_F32, C.byref(cc), A._dptr(s),
                                      it.ctypes.data_as(C.POINTER(C.c_int32)), len(s),
                                      C.byref(ci), hout.data_ptr(), A.HOST_F32, recs, cap,
                                      C.byref(rl))
            ctx.t.check(rc, "register")
        e2e_step()
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            e2e_step()
        torch.cuda.synchronize()
        ems = (time.perf_counter() - t0) * 1e3 / args.steps
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ems], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        e2e = {"value": world * vi / (ems / 1e3), "unit": "voxel-iter/s",
               "h2d_bytes_per_step": int(hf.numel() * 4 + hm.numel() * 4),
               "d2h_bytes_per_step": int(hout.numel() * 4 + cap * C.sizeof(A.dfm_iter_record)),
               "ms_per_step": ems, "s_per_pair": ems / 1e3}

    # ---- per-kernel roofline (full-resolution launches, CUDA events on the
    # library stream, separate untimed pass with per-kernel events)
    ctx.set_profiling(True)
    step()
    kt = ctx.kernel_times()
    ctx.set_profiling(False)
    esz = 4 if args.precision == "f32" else 8
    peak, peak_kind = hbm_peak()
    per = {}
    for k, elems in ALG_ELEMS.items():
        if kt[k]["launches"]:
            avg_ms = kt[k]["ms"] / kt[k]["launches"]
            vox = kt[k]["voxels"] / kt[k]["launches"]
            bytes_launch = vox * (elems * esz + ALG_EXTRA_BYTES.get(k, 0))
            per[k] = {"avg_ms": avg_ms, "launches": kt[k]["launches"],
                      "alg_bytes": bytes_launch, "gbs": bytes_launch / (avg_ms * 1e6)}
    dom = max(per, key=lambda k: per[k]["avg_ms"] * per[k]["launches"]) if per else None
    roof = None
    if dom:
        roof = {"bound": "hbm", "kernel": dom, "achieved": per[dom]["gbs"], "peak": peak,
                "peak_kind": peak_kind, "unit": "GB/s", "frac": per[dom]["gbs"] / peak,
                "traffic": None,
                "per_kernel_frac": {k: v["gbs"] / peak for k, v in per.items()},
                "per_kernel_ms": {k: v["avg_ms"] for k, v in per.items()}}
        it_ms = sum(v["avg_ms"] for v in per.values()) + (
            kt["monitor"]["ms"] / kt["monitor"]["launches"] if kt["monitor"]["launches"] else 0)
        vox = per[dom]["alg_bytes"] / (ALG_ELEMS[dom] * esz + ALG_EXTRA_BYTES.get(dom, 0))
        roof["iteration"] = {"ms": it_ms, "min_bytes_per_voxel": ITER_MIN_ELEMS * esz,
                             "achieved": vox * ITER_MIN_ELEMS * esz / (it_ms * 1e6),
                             "frac": vox * ITER_MIN_ELEMS * esz / (it_ms * 1e6) / peak}
        tr = os.path.join(ROOT, "profiles", "traffic.json")
        if os.path.exists(tr):
            try:
                with open(tr) as f:
                    roof["traffic"] = json.load(f).get(args.precision, {}).get(dom)
                roof["traffic_unit"] = "DRAM bytes per launch (ncu, profiles/traffic.json)"
                roof["alg_bytes_per_launch"] = per[dom]["alg_bytes"]
            except (OSError, ValueError):
                pass

    # ---- parity-mode (fp64 context) time of the same pair, device-timed
    f64 = None
    if args.precision == "f32" and not args.no_f64:
        ctx64 = Context(local, "f64")
        F64, M64 = F.double(), M.double()
        o64 = torch.empty((3,) + g.shape, dtype=torch.float64, device=f"cuda:{local}")
        s64 = torch.cuda.ExternalStream(ctx64.stream_ptr, device=f"cuda:{local}")

        def step64():
            return ctx64.register_device(g, F64.data_ptr(), M64.data_ptr(), cfg, sched,
                                         o64.data_ptr())
        step64()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n64 = max(1, min(args.steps, 5))
        a.record(s64)
        for _ in range(n64):
            log64 = step64()
        b.record(s64)
        torch.cuda.synchronize()
        ms64 = a.elapsed_time(b) / n64
        if world > 1:
            import torch.distributed as dist
            t = torch.tensor([ms64], device=f"cuda:{local}")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms64 = float(t.item())
        f64 = {"value": world * vi / (ms64 / 1e3), "unit": "voxel-iter/s", "ms_per_step": ms64,
               "steps": n64, "dtype": "f64", "final_loss": log64.final_loss,
               "note": "fp64 context (parity mode), same pair and schedule, device-resident"}
        ctx64.close()

    # ---- CPU reference beside it (rank 0; the other ranks wait on a gloo
    # barrier, which sleeps in a socket read instead of spinning a core)
    cpu = None
    cpu_group = None
    if world > 1:
        import torch.distributed as dist
        cpu_group = dist.new_group(backend="gloo")
    if rank == 0 and not args.no_cpu_baseline:
        try:
            cpu = cpu_leg(pair)
        except Exception as e:  # keep the GPU line even if the checker is missing
            cpu = {"error": str(e)}
    if cpu_group is not None:
        import torch.distributed as dist
        dist.barrier(group=cpu_group)

    if rank == 0:
        line = {"metric": "voxel-iterations/sec", "value": value, "unit": "voxel-iter/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "s_per_pair": ms / 1e3, "pairs_per_step": world,
                "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f32" if args.precision == "f32" else "f64",
                "data": "synthetic (BASELINE config recipe, seeded per pair)",
                "config": workload_config(pair, world),
                "gpu_launches": launches,
                "final_loss": log.final_loss,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk, "f64": f64}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
