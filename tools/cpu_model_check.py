"""Validates bench.py's same-schedule CPU model against real full-schedule
runs of the reference (oracle/_ref, all host cores) on this host:

    python tools/cpu_model_check.py [config ...]   -> profiles/r2_cpu_model_check_<host>.json

For each config: the model (one bounded sample registration: per-level
per-iteration wall times + one-offs, combined for the full schedule) and the
measured RunLog.total_ms of one complete registration with the full schedule.
"""
import json
import os
import socket
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from oracle import pyoracle  # noqa: E402
from paper_2404_01249_b200 import synth  # noqa: E402

configs = [int(c) for c in sys.argv[1:]] or [0, 1]
rows = []
for c in configs:
    pair = synth.make_pair(c, seed=0)
    model = bench.cpu_leg(pair)
    t0 = time.perf_counter()
    _, log = pyoracle.reference().register_images(pair.grid, pair.fixed, pair.moving,
                                                  pair.config, pair.schedule)
    wall = time.perf_counter() - t0
    rows.append({"config": pair.name, "model_s_per_pair": model["s_per_pair"],
                 "measured_s_per_pair": log.total_ms / 1e3, "measured_wall_s": wall,
                 "model_over_measured": model["s_per_pair"] / (log.total_ms / 1e3),
                 "per_level_iter_ms": model["per_level_iter_ms"],
                 "oneoff_ms": model["oneoff_ms"], "cores": model["cores"],
                 "cpu_model": model["cpu_model"], "records": len(log.iterations)})
    print(json.dumps(rows[-1]), flush=True)
host = socket.gethostname().split(".")[0]
out = os.path.join(ROOT, "profiles", f"r2_cpu_model_check_{host}.json")
with open(out, "w") as f:
    json.dump(rows, f, indent=1)
print("wrote", out)
