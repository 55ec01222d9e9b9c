"""Per-source-line executed-instruction attribution for one kernel of an ncu
report: joins ncu's SASS source page (instructions executed per address) with
nvdisasm -g line info of the cubin.
python tools/ncu_lines.py rep.ncu-rep obj.o kernel-substring [mangled-substring] [topn]"""
import csv, os, re, subprocess, sys, tempfile, collections
rep, obj, sub = sys.argv[1], sys.argv[2], sys.argv[3]
msub = sys.argv[4] if len(sys.argv) > 4 else sub
topn = int(sys.argv[5]) if len(sys.argv) > 5 and sys.argv[5].isdigit() else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
cur = None; hdr = None; rows = []
for ln in out.splitlines():
    r = next(csv.reader([ln]))
    if r and r[0] == "Kernel Name":
        cur = r[1]; hdr = None; continue
    if r and r[0] == "Address": hdr = r; continue
    if cur and hdr and sub in cur: rows.append(dict(zip(hdr, r)))
base = int(rows[0]["Address"], 16)
cnt = {int(r["Address"], 16) - base: int(r["Instructions Executed"] or 0) for r in rows}
stl = {int(r["Address"], 16) - base: int(r.get("Warp Stall Sampling (All Samples)") or 0)
       for r in rows}
d = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
dis = subprocess.run(["nvdisasm", "-g", os.path.join(d, cub)], capture_output=True, text=True).stdout
# find the function
lines = dis.splitlines(); in_fn = False; curline = None; per = collections.Counter(); src = {}
pst = collections.Counter()
for ln in lines:
    if ln.startswith("\t.text.") or ".text." in ln and ln.strip().endswith(":"):
        in_fn = msub in ln
    m = re.search(r'//## File "(.*)", line (\d+)', ln)
    if m and in_fn: curline = (os.path.basename(m.group(1)), int(m.group(2)))
    m2 = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if m2 and in_fn and curline:
        off = int(m2.group(1), 16)
        per[curline] += cnt.get(off, 0)
        pst[curline] += stl.get(off, 0)
tot = sum(per.values())
stot = max(sum(pst.values()), 1)
by_stall = "--stalls" in sys.argv
print(f"{sub}: attributed {tot} warp-instructions, {stot} stall samples")
files = {}
for (f, l), n in (pst if by_stall else per).most_common(topn):
    p = os.path.join("/root/repo/paper_2404_01249_b200/csrc", f)
    if f not in files and os.path.exists(p): files[f] = open(p).read().splitlines()
    txt = files[f][l - 1].strip()[:80] if f in files and l - 1 < len(files[f]) else ""
    print(f"{per[(f, l)]/tot*100:5.1f}%i {pst[(f, l)]/stot*100:5.1f}%s {f}:{l:<5} {txt}")
