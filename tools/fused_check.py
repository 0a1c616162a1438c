"""Fused vs staged path vs fp64 direct conv on a few shapes (GPU box).

python tools/fused_check.py            -- prints one line per case
"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1509_09308_b200 as wb  # noqa: E402
from oracle import winograd_oracle as O  # noqa: E402

CASES = [  # N, C, H, W, K, pad
    (1, 16, 8, 8, 16, 1),
    (2, 32, 20, 18, 48, 1),
    (1, 64, 56, 56, 64, 1),
    (2, 96, 13, 17, 130, 1),
    (1, 128, 28, 28, 256, 0),
    (3, 40, 9, 31, 200, 2),
]
PRECS = ["fp32", "tf32", "bf16", "fp16"]


def run(cfg, m, prec, d, g, path):
    os.environ["WINO_PATH"] = path
    plan = wb.WinogradPlan(cfg, m, prec)
    y = plan.forward(d, g=g)
    torch.cuda.synchronize()
    return y.cpu().numpy(), plan.info


def main():
    bad = 0
    for (N, C, H, W, K, pad) in CASES:
        cfg = wb.LayerConfig(N=N, C=C, H=H, W=W, K=K, pad=pad)
        dn = O.fill_uniform((N, C, H, W), 7)
        gn = O.fill_uniform((K, C, 3, 3), 8)
        t0 = time.time()
        ref = O.direct_forward(dn.astype(np.float64), gn.astype(np.float64), pad)
        scale = np.abs(ref).max()
        d = torch.from_numpy(dn).cuda()
        g = torch.from_numpy(gn).cuda()
        for m in (2, 4):
            for prec in PRECS:
                try:
                    yf, info = run(cfg, m, prec, d, g, os.environ.get("CHECK_PATH", "fused"))
                    yu, _ = run(cfg, m, prec, d, g, "staged")
                except Exception as e:  # noqa: BLE001
                    print(f"{(N, C, H, W, K, pad)} F{m} {prec}: ERROR {e}")
                    bad += 1
                    continue
                ef = np.abs(yf - ref).max() / scale
                eu = np.abs(yu - ref).max() / scale
                dfu = np.abs(yf - yu).max() / scale
                ok = ef <= max(2 * eu, 1e-6)
                bad += not ok
                print(f"{(N, C, H, W, K, pad)} F{m} {prec:5s} fused={info['fused']} "
                      f"splits={info['fused_splits']} rel err fused {ef:.2e} staged {eu:.2e} "
                      f"|fused-staged| {dfu:.2e} {'OK' if ok else 'MISMATCH'}", flush=True)
        print(f"  ({time.time() - t0:.1f}s)", flush=True)
    print("BAD", bad)


if __name__ == "__main__":
    main()
