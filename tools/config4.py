"""BASELINE config 4 on one B200: a 1024^3 fp32 microscopy-like pair (device-
generated, synth_gpu.py), LNCC kernel 7 (r = 3), scales 8/4/2/1 x 200/100/50/25,
registered (a) monolithically and (b) as `--slabs` emulated z-slabs (the exact
plan the NCCL multi-GPU path runs, halos exchanged by device copies), and the
two fields compared bit for bit.

    python tools/config4.py [--size 1024] [--slabs 8] [--no-slab]
Prints one JSON line.
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_01249_b200 import _abi as A, synth
from paper_2404_01249_b200.engine import Context, register_slab
from paper_2404_01249_b200.synth_gpu import make_config4_pair

ap = argparse.ArgumentParser()
ap.add_argument("--size", type=int, default=1024)
ap.add_argument("--slabs", type=int, default=8)
ap.add_argument("--no-slab", action="store_true")
ap.add_argument("--iters", default="200,100,50,25")
args = ap.parse_args()

n = args.size
shape = (n, n, n)
t0 = time.perf_counter()
puncta = int(200_000 * (n / 1024) ** 3)
fixed, moving = make_config4_pair("cuda", seed=0, shape=shape, n_puncta=max(puncta, 1000))
torch.cuda.synchronize()
t_gen = time.perf_counter() - t0
torch.cuda.empty_cache()

g = A.GridMeta.make_3d(n, n, n)
iters = tuple(int(v) for v in args.iters.split(","))
sched = A.PyramidSchedule((8.0, 4.0, 2.0, 1.0)[-len(iters):], iters)
cfg = synth.baseline_config(A.LOSS_LNCC, 3, 1.0, max_iters=max(iters))
vox_iters = 0
for s, it in zip(sched.scales, sched.iterations):
    m = -(-n // int(s))
    vox_iters += it * m ** 3

ctx = Context(0, "f32")
s = torch.cuda.ExternalStream(ctx.stream_ptr)
out = torch.empty((3,) + shape, dtype=torch.float32, device="cuda")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(s)
log = ctx.register_device(g, fixed.data_ptr(), moving.data_ptr(), cfg, sched, out.data_ptr())
e1.record(s)
torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
per_scale = {}
for si in range(len(sched.scales)):
    ws = [r.wall_ms for r in log.iterations if r.scale_index == si]
    ls = [r.loss for r in log.iterations if r.scale_index == si]
    per_scale[f"{int(sched.scales[si])}x"] = {"ms": sum(ws), "iters": len(ws),
                                              "loss_first": ls[0], "loss_last": ls[-1]}
res = {"workload": f"cfg4_{n}cube_puncta_lncc7", "shape": [n, n, n], "scales": list(sched.scales),
       "iterations": list(iters), "dtype": "f32", "gen_s": t_gen, "s_per_pair": ms / 1e3,
       "voxel_iters": vox_iters, "voxel_iter_per_s": vox_iters / (ms / 1e3),
       "final_loss": log.final_loss, "singularity": log.final_singularity_fraction,
       "per_scale": per_scale, "peak_mem_gb": torch.cuda.max_memory_allocated() / 1e9}
ctx.close()
print(json.dumps(res), flush=True)


def plane_sums(f):
    """per (component, z) exact integer checksum of the fp32 bit patterns"""
    out = torch.empty((3, f.shape[1]), dtype=torch.int64, device=f.device)
    for c in range(3):
        for z0 in range(0, f.shape[1], 64):
            blk = f[c, z0:z0 + 64].contiguous().view(torch.int32).to(torch.int64)
            out[c, z0:z0 + 64] = blk.sum(dim=(1, 2))
    return out


sums = plane_sums(out)
mono_losses = [r.loss for r in log.iterations]
del out
torch.cuda.empty_cache()

if not args.no_slab:
    ctx = Context(0, "f32")
    out2 = torch.empty((3,) + shape, dtype=torch.float32, device="cuda")
    s = torch.cuda.ExternalStream(ctx.stream_ptr)
    torch.cuda.synchronize()
    e0.record(s)
    zlo, zhi, log2 = register_slab(ctx, g, fixed.data_ptr(), moving.data_ptr(), cfg, sched,
                                   emulate=args.slabs, d_out=out2.data_ptr())
    e1.record(s)
    torch.cuda.synchronize()
    res["slabs"] = {"n": args.slabs, "s_per_pair": e0.elapsed_time(e1) / 1e3,
                    "bit_identical_field": bool(torch.equal(sums, plane_sums(out2))),
                    "check": "per-(component, z-plane) integer sums of the fp32 bit patterns",
                    "final_loss": log2.final_loss,
                    "max_loss_rel_diff": max(abs(a - b) / abs(a) for a, b in
                                             zip(mono_losses, [r.loss for r in log2.iterations]))}
    ctx.close()
    print(json.dumps(res))
