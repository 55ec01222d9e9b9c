"""Top SASS instructions (by executed count and by stall samples) per kernel of an
ncu report: python tools/ncu_hot.py rep.ncu-rep [kernel-substring] [topn]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]; sub = sys.argv[2] if len(sys.argv) > 2 else ""; topn = int(sys.argv[3]) if len(sys.argv) > 3 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
cur = None; rows = collections.defaultdict(list); hdr = None
for ln in lines:
    if ln.startswith('"Kernel Name"'):
        cur = next(csv.reader([ln]))[1]; hdr = None; continue
    r = next(csv.reader([ln]))
    if r and r[0] == "Address": hdr = r; continue
    if cur and hdr: rows[cur].append(dict(zip(hdr, r)))
for k, rs in rows.items():
    if sub not in k: continue
    tot = sum(int(r["Instructions Executed"] or 0) for r in rs)
    samp = sum(int(r["Warp Stall Sampling (All Samples)"] or 0) for r in rs)
    ops = collections.Counter()
    for r in rs:
        op = r["Source"].strip().split()[0] if r["Source"].strip() else "?"
        if op.startswith("@"): op = r["Source"].strip().split()[1]
        ops[op.split(".")[0]] += int(r["Instructions Executed"] or 0)
    print(f"=== {k[:100]}\n  warp-instructions {tot}  stall samples {samp}")
    print("  by opcode:", ", ".join(f"{o}:{c/tot*100:.1f}%" for o, c in ops.most_common(14)))
    top = sorted(rs, key=lambda r: -int(r["Warp Stall Sampling (All Samples)"] or 0))[:topn]
    for r in top:
        print(f"   {r['Warp Stall Sampling (All Samples)']:>6} {r['Instructions Executed']:>10}  {r['Source'].strip()[:90]}")
