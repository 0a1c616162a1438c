"""Append raw-metric lines (DRAM bytes, tensor-pipe activity, grid) and the
top warp-stall reasons of an ncu report to stdout (used with ncu_summary.py by
tools/evidence.sh).  usage: python tools/ncu_raw_summary.py REP"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, u, v = rows[0], rows[1], rows[2]
for w in ("dram__bytes_read.sum", "dram__bytes_write.sum",
          "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
          "l1tex__m_xbar2l1tex_read_bytes.sum", "launch__grid_size", "launch__block_size"):
    if w in h:
        print("raw", w, u[h.index(w)], v[h.index(w)])
st = []
for i, n in enumerate(h):
    if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued"):
        try:
            st.append((float(v[i]), n.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
tot = sum(x for x, _ in st) or 1.0
print("stalls (pc samples)", " ".join(f"{n}:{100 * x / tot:.0f}%" for x, n in sorted(st, reverse=True)[:8]))
