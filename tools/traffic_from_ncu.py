"""DRAM bytes per launch of each kernel class from an ncu --set full report of
the full-resolution loop (tools/box/profiles.sh), into profiles/traffic.json
(bench.py's roofline.traffic).
    python tools/traffic_from_ncu.py rep.ncu-rep [source-note]"""
import csv
import json
import os
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data = rows[0], rows[2:]
ki, rd, wr = (hdr.index("Kernel Name"), hdr.index("dram__bytes_read.sum"),
              hdr.index("dram__bytes_write.sum"))
unit = rows[1][rd]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[unit]
CLASSES = [("LnccFwd3", "loss_fwd"), ("LnccBwd2", "lncc_bwd"), ("SmoothAdam2", "smooth_adam"),
           ("Compose2<float, 0", "compose_smooth"), ("ComposeS2", "compose_smooth")]
per = defaultdict(list)
for r in data:
    name = r[ki].replace("(int)", "").replace("(bool)", "")
    for key, cls in CLASSES:
        if key in name:
            b = (float(r[rd].replace(",", "")) + float(r[wr].replace(",", ""))) * scale
            per[(cls, key)].append(b)
            break
res = defaultdict(float)
for (cls, key), v in per.items():
    res[cls] += sum(v) / len(v)  # mean per launch; compose_smooth = pointwise + smoothing kernels
note = sys.argv[2] if len(sys.argv) > 2 else os.path.basename(rep)
doc = {"_source": f"{note}: ncu --set full of the full-resolution loop kernels (config-1 phantom "
                  "at 160x192x224, fp32); DRAM bytes per launch (dram__bytes_read.sum + "
                  "dram__bytes_write.sum), mean over the captured launches; compose_smooth = the "
                  "radius-0 compose + the smoothing/W-G kernel of the split update",
       "f32": {k: int(v) for k, v in res.items()}}
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "traffic.json"), "w") as f:
    json.dump(doc, f, indent=1)
print(json.dumps(doc["f32"]))
