"""Aggregate pair throughput on one GPU with K concurrent contexts (config-2
style batch of independent pairs): K host threads, one dfm_ctx (stream) each,
each registering its own config-1 pair repeatedly.

    python tools/concurrency.py [K ...]
"""
import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2404_01249_b200 import synth
from paper_2404_01249_b200.engine import Context

ks = [int(v) for v in sys.argv[1:]] or [1, 2, 3, 4]
pairs = [synth.make_pair(1, seed=s) for s in range(max(ks))]
dev = [(torch.from_numpy(p.fixed).cuda(), torch.from_numpy(p.moving).cuda()) for p in pairs]
reps = 3
for K in ks:
    ctxs = [Context(0, "f32") for _ in range(K)]
    for c, (F, M), p in zip(ctxs, dev, pairs):  # warm up (graphs, workspaces)
        c.register_device(p.grid, F.data_ptr(), M.data_ptr(), p.config, p.schedule)
    torch.cuda.synchronize()

    def work(i):
        c, (F, M), p = ctxs[i], dev[i], pairs[i]
        for _ in range(reps):
            c.register_device(p.grid, F.data_ptr(), M.data_ptr(), p.config, p.schedule)

    th = [threading.Thread(target=work, args=(i,)) for i in range(K)]
    t0 = time.perf_counter()
    for t in th:
        t.start()
    for t in th:
        t.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"K={K}: {K * reps} pairs in {dt:.3f} s -> {dt / (K * reps) * 1e3:.1f} ms/pair aggregate",
          flush=True)
    for c in ctxs:
        c.close()
