"""Join an ncu SASS source page (CSV) with nvdisasm line info: stall samples and executed
instructions per CUDA source line.  usage: ncu_lines.py <sass.csv> <lib.so> <mangled-substring> [n]"""
import csv
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

csv_path, lib, fname = sys.argv[1], sys.argv[2], sys.argv[3]
topn = int(sys.argv[4]) if len(sys.argv) > 4 else 40
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(lib)], cwd=tmp, capture_output=True)
lines_by_off = {}
for cub in os.listdir(tmp):
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(tmp, cub)], capture_output=True, text=True).stdout
    cur = None
    infn = False
    for ln in dis.split("\n"):
        if ln.startswith("//---------------------") and ".text." in ln:
            infn = fname in ln
            continue
        if not infn:
            continue
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            lines_by_off[int(m.group(1), 16)] = cur
    if lines_by_off:
        break
rows = list(csv.reader(open(csv_path)))
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
ei = hdr.index("Instructions Executed")
addrs = [int(r[0], 16) for r in data]
base = min(addrs)
samp, execd = defaultdict(float), defaultdict(float)
for r, a in zip(data, addrs):
    key = lines_by_off.get(a - base, ("?", 0))
    samp[key] += float(r[si] or 0)
    execd[key] += float(r[ei] or 0)
ts, te = sum(samp.values()), sum(execd.values())
print(f"samples {ts:.0f}  warp-instr {te:.3g}")
for k, v in sorted(samp.items(), key=lambda x: -x[1])[:topn]:
    print(f"{k[0]:>20s}:{k[1]:<5d} samples {v/ts*100:5.1f}%  instr {execd[k]/te*100:5.1f}%")

if len(sys.argv) > 5:
    want = set(int(x) for x in sys.argv[5].split(","))
    for r, a in zip(data, addrs):
        k = lines_by_off.get(a - base, ("?", 0))
        if k[1] in want and k[0].startswith(sys.argv[6] if len(sys.argv) > 6 else ""):
            print(f"{k[1]:5d} {a-base:6x} exec={float(r[ei] or 0):10.3g} samp={float(r[si] or 0):7.0f}  {r[1][:70]}")
