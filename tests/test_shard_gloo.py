"""Multi-process (world_size 2, gloo, CPU) coverage of the batch-shard driver's
host logic: each rank computes its contiguous shard of the minibatch with the
replicated filters and no collective on the forward; the optional verification
all_gather reassembles exactly the single-process result.  The driver object
(sharding.ShardedForward: shard bounds, per-rank plan, local slice) is the one
bench.py --global-batch runs under torchrun; the per-rank compute here is the
CPU oracle (test infrastructure) standing in for the GPU kernel, which needs a
B200 (every rank's plan.forward is the C-ABI forward the GPU tests cover)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1509_09308_b200 as wb
        from oracle import winograd_oracle as O
        from paper_1509_09308_b200 import sharding

        cfg = wb.LayerConfig(N=5, C=6, H=9, W=7, K=4, pad=1)
        d_full = O.fill_uniform((cfg.N, cfg.C, cfg.H, cfg.W), 21)
        g = O.fill_uniform((cfg.K, cfg.C, 3, 3), 22)  # replicated filters
        start, count = sharding.shard_bounds(cfg.N, world, rank)
        lcfg = sharding.local_config(cfg, world, rank)
        assert lcfg.N == count
        # the batch-shard driver's host side: per-rank plan over the local shard
        # (plan creation is host-only), its slice of the global batch
        sf = sharding.ShardedForward(cfg, 4, "fp32", world, rank)
        assert (sf.start, sf.count) == (start, count) and sf.cfg == lcfg
        assert sf.plan.info["P"] == count * sf.plan.info["tiles_h"] * sf.plan.info["tiles_w"]
        assert sf.plan.out_shape == (count, cfg.K, cfg.out_h, cfg.out_w)
        d_local = sf.local_slice(d_full)
        assert d_local.shape[0] == count
        with pytest.raises(ValueError):
            sf.forward(None)  # no filters set and no g: refused before any launch
        y_local = torch.from_numpy(O.winograd_forward(d_local, g, 4, cfg.pad))
        y_all = sharding.gather_outputs(y_local, cfg)
        ref = O.winograd_forward(d_full, g, 4, cfg.pad)
        q.put((rank, bool(np.array_equal(y_all.numpy(), ref))))
    finally:
        dist.destroy_process_group()


def test_sharded_forward_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
    results = dict(q.get(timeout=10) for _ in range(2))
    assert results == {0: True, 1: True}
    assert all(p.exitcode == 0 for p in procs)
