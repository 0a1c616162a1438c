"""Command line for the GPU path: ``python -m paper_1509_09308_b200 bench ...``.

Mirrors the ``bench`` and ``accuracy`` commands of the reference CLI
(winoconv/cli.py:38-83, 110-159): same flags, same reports
(commands.cmd_bench / cmd_accuracy, commands.py:64-178) and exit codes (0 ok,
1 usage / domain error, 2 runtime failure).  Algorithm names are the
reference's (Winograd names optionally with a GEMM precision suffix,
``f4x4-fx:bf16``).  The CLI runs in-process;
``serve`` runs the HTTP service (service/app.py) under uvicorn.
"""
from __future__ import annotations

import argparse
import sys
from typing import Optional


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="python -m paper_1509_09308_b200",
                                description="B200 Winograd convolution layer benchmark")
    sub = p.add_subparsers(dest="command", required=True)
    pb = sub.add_parser("bench", help="device-time layers, report effective GFLOPS")
    pb.add_argument("--suite", default="vgg-e")
    pb.add_argument("--algo", default="f2x2")
    pb.add_argument("--batch", type=int, default=1)
    pb.add_argument("--repeats", type=int, default=3)
    pb.add_argument("--seed", type=int, default=0)
    pb.add_argument("--scale", type=float, default=1.0)
    pb.add_argument("--format", choices=("csv", "text"), default="csv")
    pb.add_argument("--out", metavar="FILE", default=None,
                    help="write the report here instead of stdout")
    pa = sub.add_parser("accuracy", help="max abs error vs the fp64 direct oracle (GPU)")
    pa.add_argument("--suite", default="vgg-e-accuracy")
    pa.add_argument("--algos", default="direct-fp32,f2x2,f4x4,fft",
                    help="comma-separated algorithm names")
    pa.add_argument("--precision", choices=("fp32", "fp16"), default="fp32")
    pa.add_argument("--seed", type=int, default=0)
    pa.add_argument("--scale", type=float, default=1.0)
    pa.add_argument("--format", choices=("csv", "text"), default="csv")
    pa.add_argument("--out", metavar="FILE", default=None)
    ps = sub.add_parser("serve", help="run the HTTP service (uvicorn)")
    ps.add_argument("--host", default="127.0.0.1")
    ps.add_argument("--port", type=int, default=8000)
    return p


def main(argv: Optional[list] = None) -> int:
    args = build_parser().parse_args(argv)
    from .commands import BENCH_ALGOS, WINOGRAD_ALGOS, cmd_accuracy, cmd_bench
    if args.command == "serve":  # cli.py `winoconv serve`
        import uvicorn

        from .service import create_app
        uvicorn.run(create_app(), host=args.host, port=args.port)
        return 0
    try:
        if args.command == "accuracy":
            rep = cmd_accuracy(suite=args.suite, algos=[a for a in args.algos.split(",") if a],
                               precision=args.precision, seed=args.seed, scale=args.scale)
        else:
            if (args.algo not in BENCH_ALGOS
                    and args.algo.partition(":")[0] not in WINOGRAD_ALGOS):
                raise ValueError(f"unknown algorithm {args.algo!r}; known: "
                                 f"{', '.join(BENCH_ALGOS)}")
            if args.batch < 1:
                raise ValueError(f"batch must be >= 1, got {args.batch}")
            rep = cmd_bench(suite=args.suite, algo=args.algo, batch=args.batch,
                            repeats=args.repeats, scale=args.scale, seed=args.seed)
    except (ValueError, KeyError) as e:
        sys.stderr.write(f"paper_1509_09308_b200: error: {e}\n")
        return 1
    except RuntimeError as e:
        sys.stderr.write(f"paper_1509_09308_b200: error: {e}\n")
        return 2
    payload = rep.to_csv() if args.format == "csv" else rep.to_text()
    if args.out:
        with open(args.out, "w", encoding="utf-8") as fh:
            fh.write(payload)
    else:
        sys.stdout.write(payload)
    return 0


if __name__ == "__main__":
    sys.exit(main())
