#!/usr/bin/env python3
"""Record K1's DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum from an
ncu --set full capture exported with --page raw --csv) in profiles/k1_traffic.json, which
bench.py reports as roofline.traffic.   usage: update_traffic.py CONFIG raw.csv"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def main(cfg, path):
    rows = list(csv.reader(open(path)))
    hdr, units = rows[0], rows[1]
    data = [r for r in rows[2:] if len(r) == len(hdr)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for m in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(m)
        tot += float(data[0][i].replace(",", "")) * scale[units[i]]
    out = os.path.join(ROOT, "profiles", "k1_traffic.json")
    d = json.load(open(out)) if os.path.exists(out) else {}
    d[cfg] = int(tot)
    json.dump(d, open(out, "w"), indent=1)
    print(cfg, int(tot))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
