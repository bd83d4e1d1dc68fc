"""Print the key lines of an ncu --page details --csv export."""
import csv
import sys

WANT = ['Duration', 'Elapsed Cycles', 'Issue Slots Busy', 'Executed Ipc Active', 'DRAM Throughput',
        'Memory Throughput', 'Registers Per Thread', 'Achieved Occupancy', 'Executed Instructions',
        'L1/TEX Hit Rate', 'L2 Hit Rate', 'Eligible Warps Per Scheduler', 'No Eligible',
        'Warp Cycles Per Issued Instruction', 'Compute (SM) Throughput', 'L2 Cache Throughput',
        'L1/TEX Cache Throughput', 'Mem Busy', 'Mem Pipes Busy']
rows = list(csv.reader(open(sys.argv[1])))
h = rows[0]
si, mi, vi, ui = (h.index(k) for k in ('Section Name', 'Metric Name', 'Metric Value', 'Metric Unit'))
for r in rows[1:]:
    if len(r) > vi and r[mi] in WANT:
        print(f"{r[si][:32]:32s} | {r[mi]} = {r[vi]} {r[ui]}")
