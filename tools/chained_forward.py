"""Run the chained VGG-E stack a few times (for ncu captures).

usage: python tools/chained_forward.py M PREC N [--no-fuse-act]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1509_09308_b200.network import VGGEStack  # noqa: E402

m, prec, n = int(sys.argv[1]), sys.argv[2], int(sys.argv[3])
net = VGGEStack(n, m, prec, seed=0, fuse_act="--no-fuse-act" not in sys.argv)
x = torch.rand(net.in_shape, device="cuda") * 2 - 1
for _ in range(2):
    net.forward(x)
torch.cuda.synchronize()
