"""Per-launch table of an ncu --csv launch list (last N launches = one step).
usage: python tools/launch_table.py launches.csv [N]"""
import csv
import sys
from collections import OrderedDict

rows = list(csv.reader(open(sys.argv[1])))
h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
hdr = rows[h]
ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
gi = hdr.index("Grid Size")
launches = OrderedDict()
for r in rows[h + 1:]:
    d = launches.setdefault(r[ii], {"name": r[ki], "grid": r[gi]})
    d[r[mi]] = float(r[vi].replace(",", ""))
L = list(launches.values())
n = int(sys.argv[2]) if len(sys.argv) > 2 else len(L)
tot = 0
for d in L[-n:]:
    t = d.get("gpu__time_duration.sum", 0) / 1000
    tot += t
    dr = (d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)) / 1e6
    lt = d.get("lts__t_bytes.sum", 0) / 1e6
    print(f"{d['name'][:44]:44s} {d['grid']:>16s} {t:9.1f} us  dram {dr:8.1f} MB  L2 {lt:9.1f} MB")
print(f"total {tot:.1f} us")
