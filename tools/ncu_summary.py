"""Print the key metrics of an ncu report (details page): python tools/ncu_summary.py REP [filter]"""
import csv
import subprocess
import sys

KEYS = ["Duration", "Elapsed Cycles", "Throughput", "Registers Per", "Achieved Occupancy",
        "Theoretical Occupancy", "Warp Cycles Per Issued", "Issued Ipc", "Executed Ipc",
        "L1/TEX Hit", "L2 Hit", "Mem Busy", "Max Bandwidth", "Issue Slots Busy", "No Eligible",
        "Active Warps Per", "Eligible Warps", "Shared Memory Configuration", "Dynamic Shared",
        "Waves Per SM", "Block Limit"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "details", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
ki, si, ni, ui, vi = (hdr.index(x) for x in ("Kernel Name", "Section Name", "Metric Name",
                                             "Metric Unit", "Metric Value"))
flt = sys.argv[2] if len(sys.argv) > 2 else None
seen = set()
for r in rows[1:]:
    name = r[ni]
    if (flt and flt not in name) or (not flt and not any(k in name for k in KEYS)):
        continue
    key = (r[ki], r[si], name)
    if key in seen:
        continue
    seen.add(key)
    print(f"{r[si][:30]:30s} {name[:50]:50s} {r[ui]:>8s} {r[vi]}")
