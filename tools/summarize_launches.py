"""Summarise an ncu launch list (gpu__time_duration + dram bytes per launch).

usage: python tools/summarize_launches.py launches.csv KEY OUT_DIR
Writes OUT_DIR/<csv-stem>_summary.json (per-kernel launches, avg us, share of
device time, dram bytes per launch) and merges {KEY: {kernel: dram bytes per
launch}} into OUT_DIR/traffic.json, which bench.py reads for roofline.traffic.
"""
import csv
import json
import os
import sys
from collections import OrderedDict


def main():
    path, key, out_dir = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(open(path)))
    h = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[h]
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    launches = OrderedDict()
    for r in rows[h + 1:]:
        d = launches.setdefault(r[ii], {"name": r[ki]})
        d[r[mi]] = float(r[vi].replace(",", ""))
    agg = OrderedDict()
    for d in launches.values():
        name = d["name"].split("(")[0].replace("void ", "").split("<")[0].replace("wino::", "")
        a = agg.setdefault(name, {"kernel": name, "launches": 0, "total_us": 0.0, "dram": 0.0})
        a["launches"] += 1
        a["total_us"] += d.get("gpu__time_duration.sum", 0) / 1000
        a["dram"] += d.get("dram__bytes_read.sum", 0) + d.get("dram__bytes_write.sum", 0)
    total = sum(a["total_us"] for a in agg.values()) or 1.0
    out = []
    for a in sorted(agg.values(), key=lambda a: -a["total_us"]):
        out.append({"kernel": a["kernel"], "launches": a["launches"],
                    "total_us": round(a["total_us"], 1),
                    "avg_us": round(a["total_us"] / a["launches"], 2),
                    "share": round(a["total_us"] / total, 3),
                    "dram_bytes_per_launch": int(a["dram"] / a["launches"])})
    stem = os.path.splitext(os.path.basename(path))[0]
    with open(os.path.join(out_dir, stem + "_summary.json"), "w") as f:
        json.dump(out, f, indent=1)
    tpath = os.path.join(out_dir, "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    traffic[key] = {o["kernel"]: o["dram_bytes_per_launch"] for o in out}
    with open(tpath, "w") as f:
        json.dump(traffic, f, indent=1)
    for o in out:
        print(o)


if __name__ == "__main__":
    main()
