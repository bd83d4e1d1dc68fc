"""Pick metrics from an ncu --page raw --csv export: python ncu_raw.py file.csv metric [metric...]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
units = rows[1] if len(rows) > 2 else None
for r in rows[1:]:
    if len(r) != len(hdr) or not r[0].isdigit():
        continue
    out = {}
    for m in sys.argv[2:]:
        if m in hdr:
            i = hdr.index(m)
            out[m] = r[i] + (" " + units[i] if units and units[i] else "")
    print(r[4][:50], out)
