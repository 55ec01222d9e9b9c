"""One rank of a 2-process z-slab registration on ONE GPU (test helper for
tests/test_slab_transport_gpu.py): the world > 1 call sequence of the slab
loop with rank-local slab views and offsets, its collectives host-staged over
torch.distributed gloo (dfm_dev_register_slab_tp) — kernels never wait on
another process, the hosts exchange between launches.

    python tests/slab_worker.py RANK WORLD PORT OUTDIR PREC [REPL_MAX]
"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, HERE)

import numpy as np  # noqa: E402


def case():
    from paper_2404_01249_b200 import _abi as A, synth
    p = synth.make_pair(0, seed=5, shape=(64, 40, 48))  # z, y, x
    sched = A.PyramidSchedule((4.0, 2.0, 1.0), (12, 8, 4))
    cfg = synth.baseline_config(A.LOSS_LNCC, 2, 1.0, max_iters=12)
    return p, sched, cfg


def main(rank, world, port, outdir, prec, repl_max=0):
    import torch
    import torch.distributed as dist
    from paper_2404_01249_b200.engine import (Context, OPT_SLAB_REPL_MAX, TorchDistTransport,
                                              register_slab_tp)
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world)
    p, sched, cfg = case()
    g = p.grid
    dt = torch.float32 if prec == "f32" else torch.float64
    ctx = Context(0, prec)
    ctx.set_option(OPT_SLAB_REPL_MAX, repl_max)
    F = torch.from_numpy(p.fixed).cuda().to(dt)
    M = torch.from_numpy(p.moving).cuda().to(dt)
    out = torch.zeros((3,) + g.shape, dtype=dt, device="cuda")
    torch.cuda.synchronize()
    tp = TorchDistTransport()
    zlo, zhi, log = register_slab_tp(ctx, g, F.data_ptr(), M.data_ptr(), cfg, sched, rank, world,
                                     tp, out.data_ptr())
    nout = (zhi - zlo) * g.dims[0] * g.dims[1]  # component c at c * nout (difform_gpu.h)
    owned = out.reshape(-1)[:3 * nout].reshape(3, nout).cpu().numpy()
    np.savez(os.path.join(outdir, f"rank{rank}.npz"), zlo=zlo, zhi=zhi, field=owned,
             losses=np.array([r.loss for r in log.iterations]), final_loss=log.final_loss,
             sing=log.final_singularity_fraction, launches=ctx.launch_count)
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5],
         int(sys.argv[6]) if len(sys.argv) > 6 else 0)
