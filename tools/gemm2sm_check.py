"""Check the fp32 (3xTF32) forward against the oracle on a few shapes; run with
WINO_GEMM_2SM=1 (read once per process) to check the CTA-pair GEMM variant.
Gates: vs the oracle's fp32 Winograd 2e-5 (F2) / 5e-5 (F4) of 1 + max|y|, vs
the fp64 direct conv 5e-4 / 5e-3.  usage: python tools/gemm2sm_check.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from oracle import winograd_oracle as O  # noqa: E402

for (N, C, H, K, m) in [(1, 64, 16, 64, 2), (1, 256, 28, 256, 2), (4, 64, 64, 64, 2),
                        (1, 512, 14, 512, 4), (2, 96, 30, 80, 4)]:
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    dn = O.fill_uniform((N, C, H, H), 5)
    gn = O.fill_uniform((K, C, 3, 3), 6)
    d, g = torch.from_numpy(dn).cuda(), torch.from_numpy(gn).cuda()
    plan = wb.WinogradPlan(cfg, m, "fp32")
    y = plan.forward(d, g=g).cpu().numpy()
    yo = O.winograd_forward(dn, gn, m, 1)
    err = np.abs(y - yo).max() / (1 + np.abs(yo).max())
    derr = O.max_abs_error(y, O.direct_forward(dn, gn, 1))
    ok = err <= (2e-5 if m == 2 else 5e-5) and derr < (5e-4 if m == 2 else 5e-3)
    print(f"N={N} C={C} H={H} K={K} F{m}: bn {plan.info['gemm_bn']} splits {plan.info['gemm_splits']} "
          f"rel err vs oracle fp32 {err:.2e}, vs fp64 direct {derr:.2e} {'OK' if ok else 'FAIL'}",
          flush=True)
