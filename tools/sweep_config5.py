"""BASELINE config 5: transform / GEMM roofline sweep on one B200.

C = K in {64, 128, 256, 512}, H = W in {14, 28, 56, 112, 224}, N in {1, 8, 64},
F(2x2) fp32 (3xTF32) and F(4x4) fp16, pad 1.  Per layer: CUDA-graph time of one
forward (effective TFLOPS), the per-stage device times (stage timer) and each
stage's roofline fraction:
  * input / output transform: algorithmic bytes (d + V / M + y) / time vs the
    measured HBM copy bandwidth (MEASURED_PEAKS.json);
  * GEMM: alpha^2 K C P multiply-adds x 2 (x 3 passes for 3xTF32) / time vs the
    dense tensor peak (bf16 measured; tf32 = bf16 / 2);
  * layer: compulsory bytes (d + g + y) / time vs HBM.
The reference CPU package (baseline/_ref, numba on all host cores) is timed on
the small N = 1 shapes for the "vs CPU oracle" column.

usage: python tools/sweep_config5.py OUT.md [OUT.jsonl]
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1509_09308_b200 as wb  # noqa: E402

peaks = {}
try:
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
except Exception:
    pass
HBM = peaks.get("hbm_gbs", 6455.0) * 1e9
BF16 = peaks.get("bf16_tflops", 1669.0) * 1e12

ref = None
ref_path = os.path.join(ROOT, "baseline", "_ref")
if os.path.isdir(ref_path):
    sys.path.insert(0, ref_path)
    try:
        import winoconv as ref  # noqa: E402
    except Exception:
        ref = None


def ref_time(N, C, H, K, m):
    if ref is None:
        return None
    from winoconv import commands as rc
    cfg = ref.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    d = ref.Tensor4.zeros((N, C, H, H), ref.Precision.FP32)
    g = ref.Tensor4.zeros((K, C, 3, 3), ref.Precision.FP32)
    d = ref.fill_uniform(d, 0, -1.0, 1.0)
    g = ref.fill_uniform(g, 1, -1.0, 1.0)
    alg = ref.builtin(m, 3)
    ref.winograd_forward(d, g, cfg, alg)  # warm-up (numba compile)
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        ref.winograd_forward(d, g, cfg, alg)
        best = min(best, time.perf_counter() - t0)
    return best


def one(N, C, H, K, m, prec, reps=10):
    cfg = wb.LayerConfig(N=N, C=C, H=H, W=H, K=K, pad=1)
    plan = wb.WinogradPlan(cfg, m, prec)
    d = torch.rand((N, C, H, H), device="cuda") * 2 - 1
    g = torch.rand((K, C, 3, 3), device="cuda") * 2 - 1
    ws = plan.alloc_workspace()
    y = torch.empty(plan.out_shape, device="cuda")
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for _ in range(2):
            plan.forward(d, y=y, g=g, workspace=ws, stream=s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=s):
        plan.forward(d, y=y, g=g, workspace=ws, stream=s)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        gr.replay()
        a.record(s)
        for _ in range(reps):
            gr.replay()
        b.record(s)
    b.synchronize()
    t = a.elapsed_time(b) / reps * 1e-3
    timer = wb.engine.StageTimer()
    with torch.cuda.stream(s):
        for _ in range(3):
            timer.gap()
            plan.forward_timed(d, y, timer, g=g, workspace=ws, stream=s)
    st, _ = timer.read()
    st = [v / 3 * 1e-3 for v in st]  # seconds per forward
    i = plan.info
    a2 = (m + 2) ** 2
    P = i["P"]
    ob = 4 if prec in ("fp32", "tf32") else 2
    passes = 3 if prec == "fp32" else 1
    gemm_flop = 2.0 * a2 * K * C * P * passes
    peak = BF16 / 2 if prec in ("fp32", "tf32") else BF16
    d_b, y_b = 4.0 * N * C * H * H, 4.0 * N * K * H * H
    v_b, m_b = float(a2) * P * C * ob, float(a2) * P * K * i["m_bytes_per_elem"]
    eff = 2.0 * N * C * K * H * H * 9 / t
    row = dict(N=N, C=C, H=H, K=K, m=m, prec=prec, us=t * 1e6, eff_tflops=eff / 1e12,
               img_s=N / t, chunks=i["num_chunks"], small_c=i["fused_small_c"],
               stage_us=[v * 1e6 for v in st],
               gemm_frac=(gemm_flop / st[2] / peak) if st[2] > 0 else None,
               in_frac=((d_b + v_b) / st[1] / HBM) if st[1] > 0 else None,
               out_frac=((m_b + y_b) / st[3] / HBM) if st[3] > 0 else None,
               layer_hbm_frac=(d_b + 36.0 * K * C + y_b) / t / HBM)
    del ws, y, d, g, gr
    torch.cuda.empty_cache()
    return row


def main():
    out_md = sys.argv[1]
    out_jl = sys.argv[2] if len(sys.argv) > 2 else None
    rows = []
    for (m, prec) in ((2, "fp32"), (4, "fp16")):
        for C in (64, 128, 256, 512):
            for H in (14, 28, 56, 112, 224):
                for N in (1, 8, 64):
                    if N * C * H * H * 4 > 3.3e9:  # N=64 C>=256 H=224: > 3 GB per tensor
                        continue
                    r = one(N, C, H, C, m, prec)
                    if N == 1 and H <= 28 and C <= 128 and m == 2:
                        rt = ref_time(N, C, H, C, m)
                        if rt:
                            r["ref_cpu_us"] = rt * 1e6
                            r["vs_ref"] = rt / (r["us"] * 1e-6)
                    rows.append(r)
                    print(json.dumps(r), flush=True)
    if out_jl:
        with open(out_jl, "w") as fh:
            for r in rows:
                fh.write(json.dumps(r) + "\n")
    f = lambda v: "—" if v is None else f"{v:.2f}"  # noqa: E731
    with open(out_md, "w") as fh:
        fh.write("# Config 5: transform / GEMM roofline sweep (one B200)\n\n")
        fh.write("`tools/sweep_config5.py`; C = K, pad 1; time = CUDA-graph replay of one forward "
                 "(non-FX: filter transform included). Fractions: transforms = algorithmic bytes / "
                 f"stage time / {HBM / 1e9:.0f} GB/s; GEMM = MMA flops (x3 for 3xTF32) / stage time "
                 f"/ {BF16 / 2e12:.0f} (tf32) or {BF16 / 1e12:.0f} (fp16) TF/s; layer = (d + g + y) "
                 "/ time / HBM. small-C layers (C <= 8) run one fused kernel (none here).\n\n")
        fh.write("| F, prec | C=K | H=W | N | µs | eff TFLOPS | img/s | filter / input / GEMM / output µs "
                 "| input frac | GEMM frac | output frac | layer HBM frac | ref CPU (×) |\n")
        fh.write("|---|---|---|---|---|---|---|---|---|---|---|---|---|\n")
        for r in rows:
            st = " / ".join(f"{v:.1f}" for v in r["stage_us"])
            rc = f"{r['ref_cpu_us'] / 1e3:.1f} ms ({r['vs_ref']:.0f}×)" if "ref_cpu_us" in r else "—"
            fh.write(f"| F{r['m']} {r['prec']} | {r['C']} | {r['H']} | {r['N']} | {r['us']:.1f} | "
                     f"{r['eff_tflops']:.1f} | {r['img_s']:.0f} | {st} | {f(r['in_frac'])} | "
                     f"{f(r['gemm_frac'])} | {f(r['out_frac'])} | {f(r['layer_hbm_frac'])} | {rc} |\n")


if __name__ == "__main__":
    main()
