"""Latency sweep and time-to-first-run harness (reference cli.py:63-67, 234-336).

``bench_sweep`` emits the reference's ``bench`` CSV schema row for row
(engine x stage over the N/K/d/B grid, stages assign / update / e2e, one
counter snapshot per row), timed on the device: every sample is one call
bracketed by CUDA events with a synchronize, the median of ``reps`` samples
after one discarded warm-up (cli.py:234-242).  The flash engine is the fused
sm_100a path; the baseline engine is the materializing foil (N x K distances
in HBM, baseline.py).

``time_to_first_run`` measures what the paper's compile heuristic targets
(PAPER.md:326-394): for each new shape, the wall time of the very first
assign+update call (tiling heuristic, workspace allocation, tensor-map
encoding, first launch -- the kernels are ahead-of-time compiled, so there is
no JIT) against the steady-state latency, and the exhaustive tile search the
heuristic replaces (``tuner.exhaustive_tune``).

CLI: ``python -m paper_2603_09229_b200.benchmark bench --n 65536 --k 1024
--d 128 --dtype bf16 --out bench.csv`` (also ``tune`` and ``ttfr``); exit
codes follow cli.py:1-6 (1 usage, 2 data format, 3 internal).
"""

from __future__ import annotations

import argparse
import statistics
import sys
import time
from itertools import product

import torch

from .baseline import argmin_rows, baseline_iteration, compute_distance_matrix, normalize, scatter_update
from .core import (Counters, DataFormatError, ResourceLimitError, dtype_for, generate_dataset,
                   init_centroids, worker_count)
from .fileio import atomic_write_text
from .flash_assign import flash_assign
from .sort_inverse import sort_inverse_update
from .tuner import CacheModel, ProblemShape, enumerate_candidates, exhaustive_tune, heuristic_config

__all__ = ["BENCH_COLUMNS", "bench_sweep", "time_to_first_run", "main"]

BENCH_COLUMNS = (
    "engine,stage,n,k,d,b,reps,median_latency_ns,"
    "intermediate_bytes_written,intermediate_bytes_read,"
    "synchronized_merges,elements_streamed,b_n,b_k,update_chunk"
)
TTFR_COLUMNS = "n,k,d,b,dtype,heuristic_ns,first_call_ns,steady_ns,b_n,b_k,update_chunk"


def _device_median_ns(fn, reps: int) -> int:
    fn()  # warm-up discarded
    torch.cuda.synchronize()
    samples = []
    for _ in range(reps):
        s = torch.cuda.Event(enable_timing=True)
        e = torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        e.synchronize()
        samples.append(int(s.elapsed_time(e) * 1e6))
    return int(statistics.median(samples))


def _stage(engine: str, stage: str, x, c, tiling):
    """(callable(counters), counter snapshot of one call) -- cli.py:245-284."""
    k = c.clusters
    if engine == "baseline":
        if stage == "assign":
            def run(counters):
                argmin_rows(compute_distance_matrix(x, c, counters, dot_mode="fast"))
        elif stage == "update":
            a = argmin_rows(compute_distance_matrix(x, c, Counters(), dot_mode="fast"))

            def run(counters):
                scatter_update(x, a, k, counters)
        else:
            def run(counters):
                baseline_iteration(x, c, counters, dot_mode="fast")
    else:
        if stage == "assign":
            def run(counters):
                flash_assign(x, c, tiling, counters, dot_mode="fast")
        elif stage == "update":
            a, _, _ = flash_assign(x, c, tiling, Counters(), dot_mode="fast")

            def run(counters):
                sort_inverse_update(x, a, k, tiling.update_chunk, counters)
        else:
            def run(counters):
                a2, _, _ = flash_assign(x, c, tiling, counters, dot_mode="fast")
                stats, _ = sort_inverse_update(x, a2, k, tiling.update_chunk, counters)
                normalize(stats, c)
    snap = Counters()
    run(snap)
    return run, snap


def _problem(n, k, d, b, seed, dtype):
    x = generate_dataset(b, n, k, d, 1.0, seed, precision=dtype)
    x = type(x)(x.data.cuda(), check_finite=False)
    return x, init_centroids(x, k, seed)


def bench_sweep(n: list[int], k: list[int], d: list[int], b: list[int] = (1,),
                engines: tuple[str, ...] = ("baseline", "flash"), reps: int = 5, seed: int = 0,
                dtype: str = "single") -> list[str]:
    """CSV lines (header first) of the reference's bench sweep (cli.py:287-336)."""
    for e in engines:
        if e not in ("baseline", "flash"):
            raise ValueError(f"unknown engine {e!r}")
    if not engines:
        raise ValueError("at least one engine is required")
    if reps < 1:
        raise ValueError("reps must be >= 1")
    if max(k) > min(n):
        raise ValueError(f"every K must be <= every N; got max K {max(k)} vs min N {min(n)}")
    elem = torch.empty((), dtype=dtype_for(dtype)).element_size()
    workers = worker_count()
    lines = [BENCH_COLUMNS]
    for nn, kk, dd, bb in product(n, k, d, b):
        x, c = _problem(nn, kk, dd, bb, seed, dtype)
        tiling = heuristic_config(ProblemShape(nn, kk, dd, bb), CacheModel(elem_bytes=elem, workers=workers))
        for engine, stage in product(engines, ("assign", "update", "e2e")):
            run, snap = _stage(engine, stage, x, c, tiling)
            med = _device_median_ns(lambda: run(Counters()), reps)
            tiles = (f"{tiling.point_tile},{tiling.centroid_tile},{tiling.update_chunk}"
                     if engine == "flash" else ",,")
            lines.append(f"{engine},{stage},{nn},{kk},{dd},{bb},{reps},{med},"
                         f"{snap.intermediate_bytes_written},{snap.intermediate_bytes_read},"
                         f"{snap.synchronized_merges},{snap.elements_streamed},{tiles}")
        del x, c
        torch.cuda.empty_cache()
    return lines


def time_to_first_run(shapes: list[tuple[int, int, int, int]], dtype: str = "bf16", reps: int = 5,
                      seed: int = 0) -> list[str]:
    """Per new shape: heuristic wall time, first assign+update call wall time
    (host clock, synchronized), steady-state device latency (CSV lines)."""
    elem = torch.empty((), dtype=dtype_for(dtype)).element_size()
    workers = worker_count()
    lines = [TTFR_COLUMNS]
    for n, k, d, b in shapes:
        x, c = _problem(n, k, d, b, seed, dtype)
        torch.cuda.synchronize()
        t0 = time.perf_counter_ns()
        tiling = heuristic_config(ProblemShape(n, k, d, b), CacheModel(elem_bytes=elem, workers=workers))
        t_h = time.perf_counter_ns() - t0

        def step():
            a, _, _ = flash_assign(x, c, tiling, Counters())
            sort_inverse_update(x, a, k, tiling.update_chunk, Counters())

        t0 = time.perf_counter_ns()
        step()
        torch.cuda.synchronize()
        t_first = time.perf_counter_ns() - t0
        t_steady = _device_median_ns(step, reps)
        lines.append(f"{n},{k},{d},{b},{dtype},{t_h},{t_first},{t_steady},"
                     f"{tiling.point_tile},{tiling.centroid_tile},{tiling.update_chunk}")
        del x, c
        torch.cuda.empty_cache()
    return lines


# ------------------------------------------------------------------ CLI
def _int_list(text: str) -> list[int]:
    try:
        values = [int(v) for v in text.split(",") if v.strip() != ""]
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected comma-separated integers, got {text!r}")
    if not values:
        raise argparse.ArgumentTypeError("list must be non-empty")
    return values


class _Parser(argparse.ArgumentParser):
    def error(self, message):  # usage errors exit 1 (cli.py:70-79)
        self.print_usage(sys.stderr)
        print(f"{self.prog}: error: {message}", file=sys.stderr)
        raise SystemExit(1)


def build_parser() -> argparse.ArgumentParser:
    p = _Parser(prog="paper_2603_09229_b200.benchmark", description=__doc__.splitlines()[0])
    sub = p.add_subparsers(dest="command", required=True)
    dtypes = ("single", "double", "bf16", "fp16")
    b = sub.add_parser("bench", help="kernel latency sweep to CSV (reference schema)")
    b.add_argument("--n", type=_int_list, required=True)
    b.add_argument("--k", type=_int_list, required=True)
    b.add_argument("--d", type=_int_list, required=True)
    b.add_argument("--b", type=_int_list, default=[1])
    b.add_argument("--engines", default="baseline,flash")
    b.add_argument("--reps", type=int, default=5)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--dtype", choices=dtypes, default="single")
    b.add_argument("--out", required=True)
    t = sub.add_parser("tune", help="exhaustive tile search vs the cache heuristic")
    t.add_argument("--n", type=int, required=True)
    t.add_argument("--k", type=int, required=True)
    t.add_argument("--d", type=int, required=True)
    t.add_argument("--b", type=int, default=1)
    t.add_argument("--reps", type=int, default=5)
    t.add_argument("--seed", type=int, default=0)
    t.add_argument("--dtype", choices=dtypes, default="single")
    t.add_argument("--out", required=True)
    f = sub.add_parser("ttfr", help="time-to-first-run per new shape")
    f.add_argument("--shapes", required=True, help="n:k:d:b,... e.g. 65536:1024:128:1")
    f.add_argument("--dtype", choices=dtypes, default="bf16")
    f.add_argument("--reps", type=int, default=5)
    f.add_argument("--out", required=True)
    return p


def main(argv=None) -> int:
    try:
        args = build_parser().parse_args(argv)
        if args.command == "bench":
            engines = tuple(e.strip() for e in args.engines.split(",") if e.strip())
            lines = bench_sweep(args.n, args.k, args.d, args.b, engines, args.reps, args.seed, args.dtype)
            atomic_write_text(args.out, "\n".join(lines) + "\n")
            print(f"wrote {args.out}: {len(lines) - 1} rows")
        elif args.command == "tune":
            if args.k > args.n:
                raise ValueError(f"K ({args.k}) must be <= N ({args.n})")
            shape = ProblemShape(points=args.n, clusters=args.k, dims=args.d, batch=args.b)
            elem = torch.empty((), dtype=dtype_for(args.dtype)).element_size()
            x = generate_dataset(args.b, args.n, args.k, args.d, 1.0, args.seed, precision=args.dtype)
            x = type(x)(x.data.cuda(), check_finite=False)
            rep = exhaustive_tune(shape, x, enumerate_candidates(shape), reps=args.reps,
                                  cache=CacheModel(elem_bytes=elem, workers=worker_count()),
                                  seed=args.seed)
            atomic_write_text(args.out, rep.csv_text())
            h, c = rep.heuristic, rep.chosen
            print(f"heuristic=({h.point_tile},{h.centroid_tile},{h.update_chunk}) "
                  f"tuned=({c.point_tile},{c.centroid_tile},{c.update_chunk}) "
                  f"candidates={len(rep.candidates)} "
                  f"latency_ratio={rep.heuristic_latency_ns / max(rep.chosen_latency_ns, 1):.3f} "
                  f"time_ratio={rep.tuning_wall_ns / max(rep.heuristic_wall_ns, 1):.1f}")
        else:
            shapes = [tuple(int(v) for v in s.split(":")) for s in args.shapes.split(",") if s]
            if not shapes or any(len(s) != 4 for s in shapes):
                raise ValueError("shapes must be n:k:d:b,...")
            lines = time_to_first_run(shapes, args.dtype, args.reps)
            atomic_write_text(args.out, "\n".join(lines) + "\n")
            print("\n".join(lines))
        return 0
    except SystemExit as e:
        return e.code if isinstance(e.code, int) else 1
    except DataFormatError as e:
        print(f"error: data format: {e}", file=sys.stderr)
        return 2
    except (ResourceLimitError, MemoryError, OSError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except ValueError as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    raise SystemExit(main())
