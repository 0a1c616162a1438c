import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1509_09308_b200 as wb
from oracle import winograd_oracle as O
os.environ["WINO_PATH"] = "staged"
for (N, C, H, K) in [(4, 96, 40, 80), (2, 256, 28, 256), (1, 64, 112, 64)]:
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    dn = O.fill_uniform((N, C, H, H), 61); gn = O.fill_uniform((K, C, 3, 3), 62)
    d, g = torch.from_numpy(dn).cuda(), torch.from_numpy(gn).cuda()
    ref = O.direct_forward(dn, gn, 1)
    for m in (2, 4):
        res = {}
        for mode in ("bf16M", "fp32M"):
            if mode == "fp32M": os.environ["WINO_M_FP32"] = "1"
            else: os.environ.pop("WINO_M_FP32", None)
            plan = wb.WinogradPlan(cfg, m, "bf16")
            y = plan.forward(d, g=g).cpu().numpy().astype(np.float64)
            e = y - ref
            res[mode] = (np.abs(e).max(), np.sqrt((e**2).mean()), plan.info["m_bytes_per_elem"], plan.info["gemm_splits"])
        s = np.abs(ref).max()
        print(f"N{N} C{C} H{H} K{K} F{m}: bf16M max {res['bf16M'][0]/s:.3e} rms {res['bf16M'][1]/s:.3e} (mb {res['bf16M'][2]}, sp {res['bf16M'][3]}) | fp32M max {res['fp32M'][0]/s:.3e} rms {res['fp32M'][1]/s:.3e} | ratio max {res['bf16M'][0]/res['fp32M'][0]:.2f} rms {res['bf16M'][1]/res['fp32M'][1]:.2f}")
