"""Summarise an ncu source page (SASS) CSV: top instructions by warp-stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = None
data = []
for r in rows:
    if len(r) > 3 and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(r)
si = hdr.index("Warp Stall Sampling (All Samples)")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(float(r[si] or 0) for r in data)
print("total samples", tot)
for idx, r in sorted(enumerate(data), key=lambda x: -float(x[1][si] or 0))[:n]:
    st = sorted(((float(r[i] or 0), hdr[i]) for i in stall_cols), reverse=True)[:3]
    print(f"{idx:5d} {float(r[si] or 0)/tot*100:5.1f}% {r[1][:60]:60s} " + " ".join(f"{h[6:]}={v:.0f}" for v, h in st))

tot_by = {}
for r in data:
    for i in stall_cols:
        tot_by[hdr[i]] = tot_by.get(hdr[i], 0) + float(r[i] or 0)
print("stall totals:", ", ".join(f"{k[6:]}={v/tot*100:.1f}%" for k, v in sorted(tot_by.items(), key=lambda x: -x[1])[:10]))
ops = {}
ei = hdr.index("Instructions Executed")
for r in data:
    op = r[1].split()[0] if not r[1].strip().startswith("@") else r[1].split()[1]
    op = op.split(".")[0]
    ops[op] = ops.get(op, 0) + float(r[ei] or 0)
te = sum(ops.values())
print("executed warp-instructions:", f"{te:.3g}", ", ".join(f"{k}={v/te*100:.1f}%" for k, v in sorted(ops.items(), key=lambda x: -x[1])[:14]))
