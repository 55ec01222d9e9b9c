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


def cpu_leg(pair, kind_pref="reference", sample_iters=(8, 4, 2)):
    """Times the reference CPU path (oracle/_ref, else the C restatement) on a
    bounded sample of the same workload; returns the cpu_baseline dict."""
    ncores = os.cpu_count() or 1
    os.environ["DIFFORM_THREADS"] = str(ncores)
    from oracle import pyoracle
    o = pyoracle.reference() if (kind_pref == "reference" and
                                 pyoracle.reference_available()) else pyoracle.port()
    from paper_2404_01249_b200 import _abi as A
    sched = A.PyramidSchedule(pair.schedule.scales, sample_iters)
    cfg = pair.config
    t0 = time.perf_counter()
    o.register_images(pair.grid, pair.fixed, pair.moving, cfg, sched)
    dt = time.perf_counter() - t0

    class _P:
        pass
    pp = _P()
    pp.grid, pp.schedule = pair.grid, sched
    vi = voxel_iters(pp)
    return {"value": vi / dt, "unit": "voxel-iter/s",
            "cores": ncores if o.kind == "reference" else 1, "kind": o.kind,
            "sample": (f"{pair.name}: one registration with the same scales and "
                       f"{'/'.join(map(str, sample_iters))} iterations (incl. pyramid and "
                       f"final full-res loss + fold check), {dt:.1f} s"),
            "seconds": dt}


def run_reference_arm(args, rank, world):
    if rank != 0:
        return
    from paper_2404_01249_b200 import synth
    pair = synth.make_pair(args.config, seed=0)
    vals = []
    cb = None
    for k in range(args.warmup + args.steps):
        cb = cpu_leg(pair, "reference", (4, 2, 1) if k < args.warmup else (8, 4, 2))
        if k >= args.warmup:
            vals.append(cb["value"])
    v = float(np.mean(vals))
    cb["value"] = v
    s_pair_est = voxel_iters(pair) / v
    line = {"impl": "reference", "metric": "voxel-iterations/sec", "value": v,
            "unit": "voxel-iter/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": s_pair_est * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic (BASELINE config recipe, seeded)",
            "config": {"workload": pair.name, "shape_xyz": list(pair.grid.dims),
                       "schedule": list(pair.schedule.iterations),
                       "note": "each step times a bounded sample (8/4/2 iterations); "
                               "ms_per_step = full-schedule estimate at that rate"},
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


def main():
    args = parse()
    rank, world, local = dist_env()
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl" if args.impl == "ours" else "gloo")
    if args.impl == "reference":
        run_reference_arm(args, rank, world)
        if world > 1:
            import torch.distributed as dist
            dist.barrier()
            dist.destroy_process_group()
        return

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

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_leg(pair)
        except Exception as e:  # keep the GPU line even if the checker is missing
            cpu = {"error": str(e)}

    if rank == 0:
        line = {"metric": "voxel-iterations/sec", "value": value, "unit": "voxel-iter/s",
                "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
                "ms_per_step": ms, "s_per_pair": ms / 1e3, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None,
                "dtype": "f32" if args.precision == "f32" else "f64",
                "data": "synthetic (BASELINE config recipe, seeded per pair)",
                "config": {"workload": pair.name, "shape_xyz": list(g.dims),
                           "scales": list(sched.scales), "iterations": list(sched.iterations),
                           "loss": "lncc r=2" if cfg.loss == A.LOSS_LNCC else "ssd",
                           "early_stop": "off (conv_window > max iterations)",
                           "pairs_per_step": world, "voxel_iters_per_pair": vi,
                           "l2": "working set ~0.7 GB per pair >> 126 MB L2 (no flush needed)"},
                "gpu_launches": launches,
                "final_loss": log.final_loss,
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk}
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
