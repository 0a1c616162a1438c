#!/usr/bin/env python
"""Benchmark: effective conv TFLOPS + images/s on the VGG-E 3x3 layers.

One "step" = one forward pass of every VGG-E conv layer instance (9 shapes,
16 layers depth-weighted, suites.py:68-78) over one batch of synthetic data,
exactly what the reference's `cmd_bench` TOTAL row measures
(commands.py:136-178).  Effective TFLOPS = direct-conv FLOPs (39.02 GFLOP per
image) / time.

  python bench.py [--gpus N --steps K --warmup W] [--algo f2x2|f4x4|f2x2-fx|f4x4-fx]
                  [--prec fp32|tf32|bf16|fp16] [--batch B]    # B = images per GPU
  torchrun ... bench.py --gpus N                            # batch-sharded, no collective
  python bench.py --impl reference                          # CPU reference arm

Default workload = BASELINE.json configs[1]: F(2x2,3x3), fp32, all VGG-E
layers, N=1 on one B200.  The fp32 GEMM is 3xTF32 on tcgen05 (fp32-accurate,
parity-tested against the reference tolerances).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "effective conv TFLOPS + images/sec, VGG-E 3x3 layers, N=1..64, 1/2/4/8 B200"
# Paper Table: F(2x2,3x3) VGG-E total effective
# TFLOPS on Titan X, keyed by (prec, N).  Only F(2x2) was published.
PUBLISHED_F2 = {"fp32": {1: 7.03, 2: 7.89, 4: 8.81, 8: 9.43, 16: 9.49, 32: 9.43, 64: 9.37}}
VGG_E = (("conv1.1", 3, 224, 64, 1), ("conv1.2", 64, 224, 64, 1), ("conv2.1", 64, 112, 128, 1),
         ("conv2.2", 128, 112, 128, 1), ("conv3.1", 128, 56, 256, 1), ("conv3.2", 256, 56, 256, 3),
         ("conv4.1", 256, 28, 512, 1), ("conv4.2", 512, 28, 512, 3), ("conv5", 512, 14, 512, 4))
STAGES = ("filter_transform", "input_transform", "batched_gemm", "output_transform")


def gflop_direct(N, C, H, K):
    return 2.0 * N * C * K * H * H * 9 / 1e9  # pad 1: out = H


def load_traffic(algo, prec, batch, stage):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu launch
    list for this workload (profiles/*/traffic.json), or None."""
    import glob
    kerns = {"batched_gemm": ["wgemm_tc_kernel"],
             "input_transform": ["input_transform_tma_kernel", "input_transform_kernel"],
             "output_transform": ["output_transform_tma_kernel", "output_transform_kernel"],
             "filter_transform": ["filter_transform_kernel"]}[stage]
    for path in sorted(glob.glob(os.path.join(ROOT, "profiles", "*", "traffic.json")), reverse=True):
        try:
            with open(path) as fh:
                tab = json.load(fh)
            row = tab.get(f"{algo}:{prec}:N{batch}", {})
            for kern in kerns:
                if row.get(kern) is not None:
                    return row[kern]
        except Exception:
            pass
    return None


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            pk = json.load(fh)
        return float(pk["hbm_gbs"]), float(pk["bf16_tflops"]), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled (every 20 ms) while the
    timed region runs; one long-lived `nvidia-smi -lms` process."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "20"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the sampler start before the timed region
        except Exception:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.05)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except Exception:
            self._p.kill()
            out = ""
        for line in out.strip().splitlines():
            self.samples.append([x.strip() for x in line.split(",")])

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        num = lambda x: x.replace(".", "", 1).isdigit()
        sm = [float(s[0]) for s in self.samples if num(s[0])]
        mx = [float(s[1]) for s in self.samples if len(s) > 1 and num(s[1])]
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 2 + i and s[2 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ============================================================== reference arm

def cpu_reference_pass(batch: int, m: int, fx: bool, use_ref: bool, seed: int = 0,
                       layers=VGG_E, budget_s: float | None = None):
    """One VGG-E pass on the host CPU: the reference package from baseline/_ref if
    installed (kind 'reference'), else the oracle port (kind 'port').  Returns
    (seconds of compute, direct GFLOP done, layers done)."""
    sec = gf = 0.0
    done = []
    if use_ref:
        from winoconv.direct import LayerConfig
        from winoconv.engine import FilterCache, winograd_forward
        from winoconv.tensors import Tensor4, fill_uniform
        from winoconv.winograd import builtin
        alg = builtin(m, 3)
        for i, (lbl, C, H, K, depth) in enumerate(layers):
            cfg = LayerConfig(N=batch, C=C, H=H, W=H, K=K, pad=1)
            d = fill_uniform(Tensor4.zeros((batch, C, H, H)), seed + 2 * i, -1.0, 1.0)
            g = fill_uniform(Tensor4.zeros((K, C, 3, 3)), seed + 2 * i + 1, -1.0, 1.0)
            cache = FilterCache()
            if fx:
                winograd_forward(d, g, cfg, alg, cache_filters=True, cache=cache)
            for _ in range(depth):
                t0 = time.perf_counter()
                winograd_forward(d, g, cfg, alg, cache_filters=fx, cache=cache)
                sec += time.perf_counter() - t0
                gf += gflop_direct(batch, C, H, K)
            done.append(lbl)
            if budget_s and sec > budget_s:
                break
    else:
        from oracle import winograd_oracle as O
        for i, (lbl, C, H, K, depth) in enumerate(layers):
            d, g = O.layer_inputs(batch, C, H, H, K, seed, i)
            U = O.filter_transform(g, m) if fx else None
            for _ in range(depth):
                t0 = time.perf_counter()
                O.winograd_forward(d, g, m, 1, U=U)
                sec += time.perf_counter() - t0
                gf += gflop_direct(batch, C, H, K)
            done.append(lbl)
            if budget_s and sec > budget_s:
                break
    return sec, gf, done


def _ref_available() -> bool:
    ref = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isdir(os.path.join(ref, "winoconv")):
        if ref not in sys.path:
            sys.path.insert(0, ref)
        try:
            import winoconv  # noqa: F401
            return True
        except Exception:
            return False
    return False


def _cpu_threads() -> int:
    try:
        import numba
        n = os.cpu_count() or 1
        numba.set_num_threads(min(n, numba.config.NUMBA_NUM_THREADS))
        return numba.get_num_threads()
    except Exception:
        return 1


def cpu_baseline(batch: int, m: int, fx: bool, budget_s: float = 20.0) -> dict:
    """Bounded CPU sample (rank 0, N=1 only): the full VGG-E pass at batch 1,
    stopping after ~budget_s of compute; reported as effective TFLOPS."""
    use_ref = _ref_available()
    cores = _cpu_threads()
    # JIT warm-up on a tiny layer (not timed)
    cpu_reference_pass(1, m, fx, use_ref, layers=(("warm", 3, 8, 4, 1),))
    sec, gf, done = cpu_reference_pass(batch, m, fx, use_ref, budget_s=budget_s)
    return {"value": gf / sec / 1e3 if sec else None, "unit": "TFLOPS",
            "cores": cores, "kind": "reference" if use_ref else "port",
            "sample": f"VGG-E layers {done[0]}..{done[-1]} ({len(done)}/9 shapes, depth-weighted) "
                      f"at N={batch}, {('f%dx%d' % (m, m)) + ('-fx' if fx else '')}, fp32, "
                      f"{sec:.1f} s of compute; numba threads={cores}"}


def run_reference_arm(args) -> None:
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    m, fx = (2 if args.algo.startswith("f2x2") else 4), args.algo.endswith("-fx")
    batch = args.global_batch if args.global_batch > 0 else args.batch * world
    use_ref = _ref_available()
    cores = _cpu_threads()
    cpu_reference_pass(1, m, fx, use_ref, layers=(("warm", 3, 8, 4, 1),))
    # each step is one full VGG-E pass at the arm's global batch; bound the run
    budget_total = float(os.environ.get("WINO_REF_BUDGET_S", "240"))
    times = []
    t_start = time.perf_counter()
    total_steps = args.warmup + args.steps
    for s in range(total_steps):
        sec, gf, done = cpu_reference_pass(batch, m, fx, use_ref)
        if s >= args.warmup or total_steps == 1:
            times.append((sec, gf))
        if time.perf_counter() - t_start > budget_total and times:
            break
    sec = sum(t for t, _ in times) / len(times)
    gf = times[0][1]
    value = gf / sec / 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "TFLOPS",
        "images_per_s": batch / sec, "n_gpus": world, "steps": len(times),
        "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp32", "data": "synthetic",
        "config": {"workload": f"VGG-E 16 conv layers (9 shapes, depth-weighted), {args.algo}, "
                               f"fp32, N={batch}", "algo": args.algo, "global_batch": batch,
                   "parallelism": "host CPU"},
        "cpu_baseline": {"value": value, "unit": "TFLOPS", "cores": cores,
                         "kind": "reference" if use_ref else "port",
                         "sample": f"full VGG-E pass per step at N={batch}; "
                                   f"{len(times)} timed steps (run budget {budget_total:.0f} s)"},
        "e2e": {"value": value, "unit": "TFLOPS", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def stage_roofline(entries, prec, fx, stream, flush, algo, batch):
    """Live per-stage kernel timing (CUDA events on the launch stream, L2 flushed
    before every layer) of the layer forwards in `entries` = (cfg, plan, d, y,
    workspace, U, g, depth); the dominant stage's algorithmic bytes or flops per
    launch over its average launch time, against the measured peak."""
    import torch

    from paper_1509_09308_b200 import engine as weng
    stage_bytes = [0.0] * 4  # algorithmic HBM bytes
    stage_flops = [0.0] * 4
    timer = weng.StageTimer()
    for (c, plan, d, y, ws, U, g, depth) in entries:
        info = plan.info
        a2 = info["alpha"] ** 2
        es, ns = info["op_bytes"], info["op_splits"]
        for _ in range(depth):
            with torch.cuda.stream(stream):
                flush.fill_(1)  # also gives the host a head start: no launch gaps timed
            timer.gap()
            plan.forward_timed(d, y, timer, U=U, g=None if fx else g, workspace=ws,
                               stream=stream)
            P, C, K = info["P"], c.C, c.K
            if not fx:
                stage_bytes[0] += 4 * 9 * K * C + ns * es * a2 * K * C
            stage_bytes[1] += 4 * c.N * C * c.H * c.W + ns * es * a2 * C * P
            stage_bytes[2] += ns * es * a2 * (C * P + K * C) + 4 * a2 * K * P
            stage_bytes[3] += 4 * a2 * K * P + 4 * c.N * K * c.out_h * c.out_w
            stage_flops[2] += 2.0 * a2 * K * C * P * (3 if prec == "fp32" else 1)
    stage_ms, stage_n = timer.read()
    hbm_peak, bf16_peak, peak_src = load_peaks()
    tensor_peak = bf16_peak if prec in ("bf16", "fp16") else bf16_peak / 2  # tf32 = bf16/2
    dom = max(range(4), key=lambda j: stage_ms[j])
    avg_ms = stage_ms[dom] / max(stage_n[dom], 1)
    if dom == 2:
        achieved = stage_flops[2] / max(stage_n[2], 1) / (avg_ms / 1e3) / 1e12
        roof = {"bound": "tensor", "achieved": achieved, "peak": tensor_peak, "unit": "TFLOP/s",
                "frac": achieved / tensor_peak, "traffic": None}
    else:
        achieved = stage_bytes[dom] / max(stage_n[dom], 1) / (avg_ms / 1e3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "traffic": None}
    traffic = load_traffic(algo, prec, batch, STAGES[dom])
    if traffic is not None:
        roof["traffic"] = traffic
        roof["traffic_source"] = "ncu dram__bytes_read.sum+write.sum per launch (profiles/)"
    roof.update({"kernel": STAGES[dom], "peak_source": f"{peak_src} (MEASURED_PEAKS.json)"
                 if peak_src == "measured" else "fallback (B200_PROFILING.md)",
                 "avg_launch_ms": avg_ms, "launches": stage_n[dom],
                 "stage_share": {STAGES[j]: stage_ms[j] / max(sum(stage_ms), 1e-9)
                                 for j in range(4)}})
    if prec not in ("bf16", "fp16") and dom == 2:
        roof["peak_note"] = "tf32 dense peak taken as measured bf16 / 2"
    if prec == "fp32" and dom == 2:
        roof["flops_note"] = "3xTF32: achieved counts all three tf32 MMA passes"
    return roof


# ============================================================== GPU arm

def run_gpu(args) -> None:
    import torch
    import torch.distributed as dist

    import paper_1509_09308_b200 as wb
    from paper_1509_09308_b200 import engine as weng

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    m, fx, prec = wb.parse_algo(args.algo)
    prec = args.prec or prec or "fp32"
    strong = args.global_batch > 0
    if strong:
        # strong scaling (config 4): a fixed global batch split contiguously over
        # the ranks by the batch-shard driver (sharding.ShardedForward)
        from paper_1509_09308_b200 import sharding
        _, B = sharding.shard_bounds(args.global_batch, world, rank)
        if B < 1:
            raise SystemExit(f"--global-batch {args.global_batch} leaves rank {rank} empty")
    else:
        B = args.batch  # images per GPU (weak scaling: per-GPU work fixed)
    gen = torch.Generator(device="cpu").manual_seed(1234 + rank)

    layers = []
    for i, (lbl, C, H, K, depth) in enumerate(VGG_E):
        if strong:
            gcfg = wb.LayerConfig(N=args.global_batch, C=C, H=H, W=H, K=K, pad=1)
            shard = sharding.ShardedForward(gcfg, m, prec, world, rank,
                                            workspace_limit=args.workspace)
            cfg, plan = shard.cfg, shard.plan
        else:
            cfg = wb.LayerConfig(N=B, C=C, H=H, W=H, K=K, pad=1)
            plan = weng.WinogradPlan(cfg, m, prec, workspace_limit=args.workspace)
        # synthetic U[-1,1) data (this rank's shard) and replicated filters.  Every
        # instance of a repeated layer (conv3.2 x3, conv4.2 x3, conv5 x4) has its own
        # input and filters, as in the network (the reference's cmd_bench re-runs
        # one input; --reuse-depth-inputs restores that, which reads the repeats'
        # filters from warm L2)
        ninst = 1 if args.reuse_depth_inputs else depth
        inst = []
        for j in range(ninst):
            d_host = (torch.rand((B, C, H, H), generator=gen) * 2 - 1).pin_memory()
            g_host = torch.rand((K, C, 3, 3),
                                generator=torch.Generator().manual_seed(100 * i + j)) * 2 - 1
            d = d_host.to(dev)
            g = g_host.to(dev)
            y = torch.empty(plan.out_shape, dtype=torch.float32, device=dev)
            y_host = torch.empty(plan.out_shape, dtype=torch.float32).pin_memory()
            if strong and fx:
                sh = sharding.ShardedForward(gcfg, m, prec, world, rank,
                                             workspace_limit=args.workspace)
                sh.set_filters(g)
                inst.append(dict(d=d, g=g, y=y, U=sh.U, shard=sh, d_host=d_host, y_host=y_host))
            else:
                inst.append(dict(d=d, g=g, y=y, U=plan.filter_transform(g) if fx else None,
                                 shard=shard if strong else None, d_host=d_host, y_host=y_host))
        ws = plan.alloc_workspace(dev)
        calls = [inst[j % ninst] for j in range(depth)]
        layers.append(dict(lbl=lbl, C=C, H=H, K=K, depth=depth, cfg=cfg, plan=plan,
                           d=inst[0]["d"], g=inst[0]["g"], y=inst[0]["y"], U=inst[0]["U"],
                           shard=shard if strong else None, ws=ws, calls=calls,
                           d_host=inst[0]["d_host"], y_host=inst[0]["y_host"],
                           gf=gflop_direct(B, C, H, K)))
    gf_step = sum(L["gf"] * L["depth"] for L in layers)  # this rank's share
    # whole-job GFLOP per step: every rank's shard (weak: world x B images;
    # strong: the fixed global batch)
    gf_job = (sum(gflop_direct(args.global_batch, C, H, K) * dep for (_, C, H, K, dep) in VGG_E)
              if strong else gf_step * world)
    images_job = args.global_batch if strong else B * world
    launches_step = sum(L["depth"] * (L["plan"].info["launches_per_forward"] +
                                      (0 if fx or L["plan"].info["combined_transforms"] else 1))
                        for L in layers)

    stream = torch.cuda.Stream(device=dev)

    def step_body(s):
        for L in layers:
            for c in L["calls"]:
                if c["shard"] is not None:  # batch-shard driver (strong scaling)
                    c["shard"].forward(c["d"], y_local=c["y"], workspace=L["ws"], stream=s,
                                       g=None if fx else c["g"])
                else:
                    L["plan"].forward(c["d"], y=c["y"], U=c["U"], g=None if fx else c["g"],
                                      workspace=L["ws"], stream=s)

    # capture the whole step in one CUDA graph (launch-bound at N=1)
    with torch.cuda.stream(stream):
        step_body(stream)  # warm (sets kernel attributes, outside capture)
    torch.cuda.synchronize()
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            step_body(torch.cuda.current_stream())
        torch.cuda.synchronize()

    def run_step():
        if graph is not None:
            graph.replay()
        else:
            with torch.cuda.stream(stream):
                step_body(stream)

    flush = torch.empty(int(args.flush_mb) << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up
    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            run_step()
    torch.cuda.synchronize()

    # ---- timed region: K steps, L2 flushed between steps (outside the events)
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        with torch.cuda.stream(stream):
            for a, b in evs:
                flush.fill_(1)
                a.record(stream)
                run_step()
                b.record(stream)
        torch.cuda.synchronize()
    barrier()
    step_ms = [a.elapsed_time(b) for a, b in evs]
    t_local = sum(step_ms) / 1e3
    t = torch.tensor([t_local], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    ms_per_step = t_max / args.steps * 1e3
    total_gf = gf_job * args.steps
    value = total_gf / t_max / 1e3  # TFLOPS, whole job
    images_per_s = images_job * args.steps / t_max

    roof = stage_roofline([(L["cfg"], L["plan"], L["d"], L["y"], L["ws"], L["U"], L["g"],
                            L["depth"]) for L in layers], prec, fx, stream, flush,
                          args.algo, B)

    # ---- e2e through the C ABI with pinned host buffers (H2D + compute + D2H)
    h2d = sum(L["d_host"].numel() * 4 * L["depth"] for L in layers)
    d2h = sum(L["y_host"].numel() * 4 * L["depth"] for L in layers)
    e2e_steps = max(1, min(args.steps, 5))

    # The layer invocations of a step are independent calls (each with its own
    # input, like the reference's cmd_bench), so they are pipelined the way a
    # server pipelines requests: round-robin over E2E_STREAMS streams, each with
    # its own device and pinned-host buffers, so one call's H2D copy, another's
    # kernels and a third's D2H copy overlap.  Every call still copies its full
    # input in and its full output out inside the timed region.
    E2E_STREAMS = int(os.environ.get("WINO_E2E_STREAMS", "4"))
    e2e_streams = [stream] + [torch.cuda.Stream(device=dev) for _ in range(E2E_STREAMS - 1)]
    e2e_bufs = []
    for si in range(E2E_STREAMS):
        row = []
        for L in layers:
            if si == 0:
                row.append((L["d"], L["y"], L["ws"], L["y_host"]))
            else:
                row.append((torch.empty_like(L["d"]), torch.empty_like(L["y"]),
                            torch.empty_like(L["ws"]), torch.empty_like(L["y_host"]).pin_memory()))
        e2e_bufs.append(row)

    def e2e_step():
        call = 0
        for li, L in enumerate(layers):
            for c in L["calls"]:
                si = call % E2E_STREAMS
                call += 1
                d_dev, y_dev, ws, y_host = e2e_bufs[si][li]
                L["plan"].forward_host(c["d_host"], y_host, d_dev, y_dev, U=c["U"],
                                       g=None if fx else c["g"], workspace=ws,
                                       stream=e2e_streams[si])

    def e2e_fork(ev):
        for st in e2e_streams[1:]:
            st.wait_event(ev)

    def e2e_join():
        for st in e2e_streams[1:]:
            ev = torch.cuda.Event()
            ev.record(st)
            stream.wait_event(ev)

    e2e_step()
    torch.cuda.synchronize()
    barrier()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ea.record(stream)
    e2e_fork(ea)
    for _ in range(e2e_steps):
        e2e_step()
    e2e_join()
    eb.record(stream)
    eb.synchronize()
    barrier()
    te = torch.tensor([ea.elapsed_time(eb) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = gf_job * e2e_steps / float(te.item()) / 1e3

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(1, m, fx, budget_s=args.cpu_budget)

    if rank == 0:
        pub = PUBLISHED_F2.get(prec, {}).get(images_job) if (m == 2 and not fx) else None
        clocks = sampler.summary()
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS",
            "images_per_s": images_per_s, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": (value / pub) if pub else None,
            "vs_baseline_ref": ("paper F(2x2) VGG-E Titan X, PAPER.md:565-607" if pub else None),
            "dtype": prec, "data": "synthetic",
            "config": {"workload": f"VGG-E 16 conv layers (9 shapes, depth-weighted), "
                                   f"{args.algo} F({m}x{m},3x3), GEMM {prec}"
                                   f"{' (3xTF32)' if prec == 'fp32' else ''}, "
                                   + (f"global N={args.global_batch} split over {world} GPU(s)"
                                      if strong else f"N={B} per GPU"),
                       "algo": args.algo, "global_batch": images_job, "batch_per_gpu": B,
                       "parallelism": f"dp{world} batch-shard (no collective)"
                                      + (", sharding.ShardedForward" if strong else ""),
                       "workspace_limit": args.workspace,
                       "l2": f"flushed between timed steps ({args.flush_mb} MB write)",
                       "layer_instances": ("one input/filter set per shape, re-run depth times"
                                           if args.reuse_depth_inputs else
                                           "distinct input and filters for each of the 16 layers"),
                       "cuda_graph": graph is not None},
            "roofline": roof,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_val, "unit": "TFLOPS", "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h, "steps": e2e_steps, "streams": E2E_STREAMS,
                    "path": f"wino_forward_host (C ABI), pinned host buffers, independent layer calls round-robin over {E2E_STREAMS} streams"},
            "gpu_launches": launches_step * args.steps,
            "clocks": clocks,
            "step_ms": step_ms,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_chained(args) -> None:
    """--chained: the VGG-E conv stack run as a network (network.VGGEStack):
    each layer's output feeds the next through ReLU and 2x2 max-pool.  One step
    = one forward of the 16-layer stack at N = --batch (per GPU); e2e copies
    only the network input in and its output out.  Effective TFLOPS counts the
    16 convolutions' direct-conv FLOPs (ReLU / pooling add none)."""
    import torch
    import torch.distributed as dist

    import paper_1509_09308_b200 as wb
    from paper_1509_09308_b200.network import VGGEStack

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    m, fx, prec = wb.parse_algo(args.algo)
    prec = args.prec or prec or "fp32"
    strong = args.global_batch > 0  # config 4: a fixed global batch split over the ranks
    if strong:
        from paper_1509_09308_b200 import sharding
        _, B = sharding.shard_bounds(args.global_batch, world, rank)
        if B <= 0:
            raise SystemExit(f"--global-batch {args.global_batch} leaves rank {rank} empty")
    else:
        B = args.batch
    images_job = args.global_batch if strong else B * world
    net = VGGEStack(B, m, prec, seed=0, workspace_limit=args.workspace,
                    fuse_act=not args.no_fuse_act, fx=fx)
    gen = torch.Generator(device="cpu").manual_seed(1234 + rank)
    x_host = (torch.rand(net.in_shape, generator=gen) * 2 - 1).pin_memory()
    x = x_host.to(dev)
    out = torch.empty(net.out_shape, device=dev)
    out_host = torch.empty(net.out_shape).pin_memory()
    stream = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(stream):
        net.forward(x, out=out, stream=stream)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=stream):
        net.forward(x, out=out, stream=torch.cuda.current_stream())
    torch.cuda.synchronize()
    flush = torch.empty(int(args.flush_mb) << 20, dtype=torch.uint8, device=dev)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        with torch.cuda.stream(stream):
            graph.replay()
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        with torch.cuda.stream(stream):
            for a, b in evs:
                flush.fill_(1)
                a.record(stream)
                graph.replay()
                b.record(stream)
        torch.cuda.synchronize()
    barrier()
    t = torch.tensor([sum(a.elapsed_time(b) for a, b in evs) / 1e3], dtype=torch.float64,
                     device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    t_max = float(t.item())
    gf_job = net.gflop / B * images_job  # direct-conv GFLOP of the whole job per step
    value = gf_job * args.steps / t_max / 1e3

    # per-layer stage roofline on the stack's own layer inputs
    entries = []
    for i, (name, cfg, plan, g, pool) in enumerate(net.layers):
        d = torch.rand((cfg.N, cfg.C, cfg.H, cfg.W), device=dev)
        y = torch.empty(plan.out_shape, device=dev)
        entries.append((cfg, plan, d, y, net._ws, net._U[i] if fx else None, g, 1))
    roof = stage_roofline(entries, prec, fx, stream, flush, args.algo, B)

    # e2e: pinned input -> device, the stack, output -> pinned host, every step
    e2e_steps = max(1, min(args.steps, 10))
    barrier()
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(stream):
        ea.record(stream)
        for _ in range(e2e_steps):
            x.copy_(x_host, non_blocking=True)
            graph.replay()
            out_host.copy_(out, non_blocking=True)
        eb.record(stream)
    eb.synchronize()
    barrier()
    te = torch.tensor([ea.elapsed_time(eb) / 1e3], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_val = gf_job * e2e_steps / float(te.item()) / 1e3
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "TFLOPS",
            "images_per_s": images_job * args.steps / t_max, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": t_max / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": prec,
            "data": "synthetic",
            "config": {"workload": f"VGG-E conv stack chained as a network (16 conv + ReLU, "
                                   f"2x2 max-pool per block), {args.algo} F({m}x{m},3x3), "
                                   f"GEMM {prec}, "
                                   + (f"global N={args.global_batch} split over {world} GPU(s)"
                                      if strong else f"N={B} per GPU"),
                       "algo": args.algo, "global_batch": images_job, "batch_per_gpu": B,
                       "parallelism": f"dp{world} batch-shard (no collective)",
                       "l2": f"flushed between timed steps ({args.flush_mb} MB write)",
                       "cuda_graph": True, "chained": True,
                       "relu_pool": "separate pass" if args.no_fuse_act else
                       "fused into the output transform (wino_forward_act)",
                       "filters": "transformed once (FX, FilterCache semantics)" if fx else
                       "transformed every step (non-FX)"},
            "roofline": roof,
            "cpu_baseline": None,
            "e2e": {"value": e2e_val, "unit": "TFLOPS",
                    "h2d_bytes_per_step": x_host.numel() * 4,
                    "d2h_bytes_per_step": out_host.numel() * 4, "steps": e2e_steps,
                    "path": "VGGEStack.forward (C ABI per layer) captured in a graph; pinned "
                            "input copied in and output copied out every step"},
            "gpu_launches": net.launches() * args.steps,
            "clocks": sampler.summary(),
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--algo", default="f2x2")
    ap.add_argument("--prec", default=None, choices=(None, "fp32", "tf32", "bf16", "fp16"))
    ap.add_argument("--batch", type=int, default=1, help="images per GPU")
    ap.add_argument("--workspace", type=int, default=0,
                    help="transform-space staging budget in bytes (0 = planner default 128 MiB; "
                         "16777216 = the paper's 16 MB)")
    ap.add_argument("--global-batch", type=int, default=0,
                    help="strong scaling: this global N is split over the ranks "
                         "(default: --batch images per GPU, weak scaling)")
    ap.add_argument("--flush-mb", type=int, default=256)
    ap.add_argument("--no-graph", action="store_true")
    ap.add_argument("--no-fuse-act", action="store_true",
                    help="--chained: ReLU / max-pool as a separate pass, not in the output transform")
    ap.add_argument("--chained", action="store_true",
                    help="run the 16 layers as a network (ReLU + max-pool between blocks)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--reuse-depth-inputs", action="store_true",
                    help="repeated layers (conv3.2 x3 ...) re-run one input and filter set, as "
                         "the reference's cmd_bench does (default: distinct per instance)")
    ap.add_argument("--cpu-budget", type=float, default=20.0)
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3  # timing rule: at least 3 warm-up steps
    if args.impl == "reference":
        run_reference_arm(args)
    elif args.chained:
        run_chained(args)
    else:
        run_gpu(args)


if __name__ == "__main__":
    main()
