"""GEMM timeline per CTA (WINO_GEMM_DBG=64 globaltimer stamps; diagnostic).

usage: WINO_BUILD_TRACE=1 python paper_1509_09308_b200/build.py   (trace build)
       WINO_GEMM_DBG=64 python tools/gemm_trace.py LABEL M PREC BATCH [WORKSPACE_MB]
Stamps: 0 entry, 1 after griddepcontrol.wait, 2 first stage at the MMA warp,
3 last commit issued, 4 first accumulator at the epilogue, 5 epilogue done, 6 exit.
"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from paper_1509_09308_b200 import _lib  # noqa: E402
from paper_1509_09308_b200.suites import VGG_E_ROWS  # noqa: E402

assert os.environ.get("WINO_GEMM_DBG") == "64"
label, m, prec, batch = sys.argv[1], int(sys.argv[2]), sys.argv[3], int(sys.argv[4])
_, C, H, K, _ = [r for r in VGG_E_ROWS if r[0] == label][0]
cfg = wb.LayerConfig(N=batch, C=C, H=H, W=H, K=K, pad=1)
ws_mb = int(sys.argv[5]) if len(sys.argv) > 5 else 0
plan = wb.WinogradPlan(cfg, m, prec, workspace_limit=ws_mb << 20)
d = torch.rand((batch, C, H, H), device="cuda") * 2 - 1
g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
ws = plan.alloc_workspace()
y = torch.empty(plan.out_shape, device="cuda")
for _ in range(5):
    plan.forward(d, y=y, g=g, workspace=ws)
torch.cuda.synchronize()
lib = _lib.lib
buf = (ctypes.c_ulonglong * (16 * 1024))()
lib.wino_debug_gemm_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
lib.wino_debug_gemm_trace(ctypes.addressof(buf), 1024)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
rel = (a[:, :8] - t0) / 1000.0
print(label, prec, batch, "bn", plan.info["gemm_bn"], "splits", plan.info["gemm_splits"], "chunks", plan.info["num_chunks"], "ctas", len(a))
names = ["entry", "gdwait", "stage0@mma", "last_commit", "acc@epi", "epi_done", "exit", "full0@split"]
for i, nme in enumerate(names):
    col = rel[:, i]
    col = col[a[:, i] > 0]
    if col.size == 0:
        continue
    print(f"  {nme:12s} min {col.min():7.2f}  med {np.median(col):7.2f}  max {col.max():7.2f} us")
waits = ["prod_wait_empty", "mma_wait_full", "mma_wait_tempty", "epi_wait_tfull"]
for i, nme in enumerate(waits):
    col = a[:, 8 + i] / 1000.0
    print(f"  {nme:16s} med {np.median(col):7.2f}  max {col.max():7.2f} us (total per CTA)")
