"""Accuracy of the fp32 (3xTF32) GEMM variants against the fp64 direct conv on
VGG-E shapes (diagnostic).  usage: python tools/acc_probe.py"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402
from oracle import winograd_oracle as O  # noqa: E402
from paper_1509_09308_b200 import _lib  # noqa: E402

VARIANTS = [("default", {}), ("no_tmem_a", {"WINO_NO_TMEM_A": "1"}),
            ("splits1", {"WINO_SPLITS": "1"}), ("usplit_off", {"WINO_NO_USPLIT": "1"}),
            ("fused", {"WINO_PATH": "fused"}), ("bn64", {"WINO_GEMM_BN": "64"})]
for (lbl, C, H, K, i) in (("conv2.2", 128, 112, 128, 3), ("conv4.1", 256, 28, 512, 6),
                          ("conv5", 512, 14, 512, 8)):
    for N in (1, 8):
        d, g = O.layer_inputs(N, C, H, H, K, 0, i)
        dd, gg = torch.from_numpy(d).cuda(), torch.from_numpy(g).cuda()
        d64, g64 = dd.double(), gg.double()
        y64 = torch.empty((N, K, H, H), dtype=torch.float64, device="cuda")
        desc = _lib.LayerDesc(N, C, H, H, K, 3, 3, 1)
        _lib.check(_lib.lib.wino_direct_forward(ctypes.byref(desc), _lib.PREC_FP64, _lib.PREC_FP64,
                                                d64.data_ptr(), g64.data_ptr(), y64.data_ptr(),
                                                torch.cuda.current_stream().cuda_stream))
        for m in (2, 4):
            out = []
            for name, env in VARIANTS:
                old = {k: os.environ.get(k) for k in env}
                os.environ.update(env)
                try:
                    plan = wb.WinogradPlan(wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1), m, "fp32")
                    y = plan.forward(dd, g=gg)
                    torch.cuda.synchronize()
                    err = float((y.double() - y64).abs().max())
                    out.append(f"{name} {err:.2e} (sp{plan.info['gemm_splits']})")
                finally:
                    for k, v in old.items():
                        if v is None:
                            os.environ.pop(k, None)
                        else:
                            os.environ[k] = v
            print(f"{lbl} N={N} F{m}: " + "  ".join(out), flush=True)
