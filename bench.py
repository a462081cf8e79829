#!/usr/bin/env python
"""Benchmark: one Lloyd iteration of flash-kmeans at BASELINE config 3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, NCCL)

``--gpus N`` without torchrun re-launches itself under torch.distributed.run
with N ranks (and refuses to run if fewer than N GPUs are visible).

Workload (BASELINE.json metric): N=8,388,608 points, d=128, K=4096, bf16,
synthetic Gaussian blobs (generate_dataset's distribution, drawn on the GPU),
random_distinct init.  A "step" is one full Lloyd iteration of the hot path:
FlashAssign (tcgen05) -> objective -> sort-inverse update -> [NCCL all-reduce
when N > 1] -> normalize -> the one 16-byte host read that decides
termination.  Points are sharded across ranks (strong scaling: the 8M points
are split N ways) and every rank keeps replicated centroids.

Printed JSON (rank 0, one line): value = points/s of the whole job (points /
max-over-ranks iteration time), plus ms_per_step, the assign kernel's
roofline, the update kernel's HBM fraction, clocks sampled during the timed
region, a parity check of the last timed iteration against the oracle, an
end-to-end figure through the public out_of_core_iteration from pinned host
buffers, and the CPU oracle timed on this host's cores.
"""

from __future__ import annotations

import argparse
import datetime
import glob
import json
import os
import socket
import statistics
import subprocess
import sys
import tempfile
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Lloyd iteration latency (ms) & points/s at N=8M,d=128,K=4096; % TC/HBM roofline"
N_TOTAL = 1 << 23
DIMS = 128
CLUSTERS = 4096
PARITY_ROWS = 1 << 16


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=p["hbm_gbs"], tc_burst=p["bf16_tflops"], tc_sustained=p["bf16_tflops_sustained"],
                    src="measured (MEASURED_PEAKS.json)")
    except Exception:
        return dict(hbm=6650.0, tc_burst=1590.0, tc_sustained=1400.0,
                    src="fallback (B200_PROFILING.md)")


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernels from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except Exception:
        return {}


def update_traffic(tr):
    """DRAM bytes of one update (every update kernel in the ncu capture), or None."""
    keys = [k for k, v in tr.items() if isinstance(v, dict) and k.startswith("k_")
            and any(p in k for p in ("hist", "scan", "scatter", "segsum"))]
    return sum(tr[k]["dram_bytes"] for k in keys) if keys else None


class ClockSampler:
    """nvidia-smi clocks + throttle reasons, sampled every 20 ms; ``summary``
    keeps only the samples whose timestamps fall inside the timed region."""

    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == 8:
                try:
                    parts[0] = datetime.datetime.strptime(parts[0], "%Y/%m/%d %H:%M:%S.%f")
                except ValueError:
                    continue
                self.rows.append(parts)

    def mark(self, start: bool):
        now = datetime.datetime.now()
        if start:
            self.window = [now, now]
        else:
            self.window[1] = now

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.1)  # let the sampler flush the last in-window samples
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        rows = self.rows
        note = "samples inside the timed region"
        if self.window is not None:
            lo, hi = self.window
            inside = [r for r in rows if lo <= r[0] <= hi]
            if not inside:  # region shorter than one sample period: the nearest samples
                pad = datetime.timedelta(milliseconds=100)
                inside = [r for r in rows if lo - pad <= r[0] <= hi + pad]
                note = "timed region shorter than the sampling period: samples within 100 ms of it"
            rows = inside
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        sm = [v for v in (num(r[1]) for r in rows) if v is not None]
        mx = [v for v in (num(r[2]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(rows), "window": note}


def make_shard(n_local: int, seed: int, device):
    """Gaussian blobs like core.generate_dataset (centers U(-10,10), unit noise), on the GPU."""
    import torch

    g = torch.Generator(device=device).manual_seed(1234)  # same centers on every rank
    centers = (torch.rand((CLUSTERS, DIMS), generator=g, device=device) * 20 - 10)
    g.manual_seed(1000 + seed)
    labels = torch.randint(0, CLUSTERS, (n_local,), generator=g, device=device)
    x = centers[labels] + torch.randn((n_local, DIMS), generator=g, device=device)
    return x.to(torch.bfloat16).reshape(1, n_local, DIMS).contiguous()


def cpu_oracle_rate(sample_points: int, threads: int):
    """The reference algorithm (oracle/, exact mode) on this host's cores: points/s per iteration."""
    import numpy as np
    import torch

    from oracle import oracle as O

    O.build()
    g = torch.Generator().manual_seed(7)
    centers = torch.rand((CLUSTERS, DIMS), generator=g) * 20 - 10
    lab = torch.randint(0, CLUSTERS, (sample_points,), generator=g)
    x = (centers[lab] + torch.randn((sample_points, DIMS), generator=g)).to(torch.bfloat16).float()
    x = x.numpy().reshape(1, sample_points, DIMS)
    k = min(CLUSTERS, sample_points)
    c = np.ascontiguousarray(x[:, np.random.default_rng(0).choice(sample_points, k, replace=False)])
    t0 = time.perf_counter()
    a, m = O.assign(x, c, threads)
    sums, counts, _ = O.sort_inverse_update(x, a, k, sample_points)
    O.normalize(sums, counts, c)
    dt = time.perf_counter() - t0
    return sample_points / dt, dt


def run_reference(args):
    """The reference arm: the reference's exact Lloyd iteration (the oracle port of
    flashmeans' lloyd_run path; the Numba package itself cannot travel to the
    GPU box) on every host core, timed on a 2^20-point sample of config 3 per
    step and extrapolated linearly in N (assign cost is exactly linear in N,
    BASELINE.md §2)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    sample = args.cpu_sample
    for _ in range(args.warmup):  # warm caches / thread pool on a small sample
        cpu_oracle_rate(1 << 13, threads)
    vals = [cpu_oracle_rate(sample, threads)[0] for _ in range(args.steps)]
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": N_TOTAL / v * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32 (exact bf16 upcast)",
        "data": "synthetic", "config": {"workload": f"config 3: N={N_TOTAL}, d={DIMS}, K={CLUSTERS}, "
                                        f"bf16 (upcast), timed on a {sample}-point sample per step",
                                        "engine": "oracle port of flashmeans exact Lloyd iteration"},
        "extrapolated": True,
        "extrapolation": f"ms_per_step = {N_TOTAL} / (median points/s of {args.steps} timed "
                         f"{sample}-point iterations); warm-up steps ran on 8192 points",
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} points x K={CLUSTERS} x d={DIMS}, one exact Lloyd iteration "
                                   "per step"},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def parity_check(eng, x, rank: int):
    """The last timed iteration's ids vs the oracle on a sample of rows, with the
    operand centroids that iteration used: equal except documented near-ties
    (|d64(a_gpu) - d64(a_ref)| <= 1e-3 d64(a_ref)); counts of the sample exact."""
    import numpy as np

    from oracle import oracle as O

    O.build()
    slot = (eng.it - 1) & 1
    c = eng.operand[eng.cur ^ 1][0].float().cpu().numpy()[None]
    n = x.shape[1]
    rows = np.linspace(0, n - 1, min(PARITY_ROWS, n)).astype(np.int64)
    xs = x[0, rows].float().cpu().numpy()[None]
    a_gpu = eng.ids[slot][0].cpu().numpy()[rows]
    a_ref, _ = O.assign(np.ascontiguousarray(xs), np.ascontiguousarray(c), os.cpu_count() or 1)
    mism = np.flatnonzero(a_gpu != a_ref[0])
    xs64, c64 = xs[0].astype(np.float64), c[0].astype(np.float64)
    dg = ((xs64[mism] - c64[a_gpu[mism]]) ** 2).sum(-1)
    dr = ((xs64[mism] - c64[a_ref[0][mism]]) ** 2).sum(-1)
    near = np.abs(dg - dr) <= 1e-3 * dr
    return {"rows": int(rows.size), "rank": rank, "mismatches": int(mism.size),
            "near_ties": int(near.sum()), "ok": bool(near.all()),
            "rule": "ids equal to the oracle except |d64(gpu)-d64(ref)| <= 1e-3 d64(ref)"}


def nccl_summary(log_dir):
    """nranks / NVLS / channel lines from this run's NCCL_DEBUG=INFO logs."""
    out = {"nranks": None, "nvls": None, "lines": []}
    for f in sorted(glob.glob(os.path.join(log_dir, "nccl.*.log"))):
        try:
            text = open(f, errors="replace").read().splitlines()
        except OSError:
            continue
        for line in text:
            low = line.lower()
            if "nranks" in low and out["nranks"] is None:
                try:
                    out["nranks"] = int(low.split("nranks")[1].split()[0])
                except (IndexError, ValueError):
                    pass
                out["lines"].append(line.strip()[-160:])
            if "nvls" in low:
                if out["nvls"] is None:
                    out["nvls"] = "disab" not in low and "not support" not in low
                if len(out["lines"]) < 6:
                    out["lines"].append(line.strip()[-160:])
    return out


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_09229_b200 import LloydEngine
    from paper_2603_09229_b200.distributed import make_allreduce, shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # FK_BENCH_SHARE_GPU=1 + FK_DIST_BACKEND=gloo: every rank on cuda:0 (a
    # one-GPU rehearsal of the multi-rank code path; numbers are not scaling data)
    share = os.environ.get("FK_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    elif torch.cuda.device_count() <= local:
        raise SystemExit(f"rank {rank}: LOCAL_RANK={local} but only {torch.cuda.device_count()} GPUs visible")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    backend = None
    if world > 1:
        backend = os.environ.get("FK_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        group = dist.group.WORLD
    lo, hi = shard_bounds(N_TOTAL, world, rank)
    n_local = hi - lo
    x = make_shard(n_local, rank, dev)
    # random_distinct init over the global range (core.py:375-377); rows from the owning shard
    idx = np.random.default_rng((0, 0)).choice(N_TOTAL, size=CLUSTERS, replace=False)
    c0 = torch.zeros((1, CLUSTERS, DIMS), dtype=torch.float32, device=dev)
    sel = np.flatnonzero((idx >= lo) & (idx < hi))
    c0[0, torch.from_numpy(sel).to(dev)] = x[0, torch.from_numpy(idx[sel] - lo).to(dev)].float()
    allreduce = make_allreduce() if world > 1 else None
    if world > 1:
        dist.all_reduce(c0)
    eng = LloydEngine(x, CLUSTERS, update_chunk=N_TOTAL, allreduce=allreduce)
    eng.set_centroids(c0)

    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # One step = one Lloyd iteration as lloyd_run executes it (LloydEngine.run):
    # the next assign is queued before the host reads this iteration's flags,
    # so the GPU does not idle on the poll.  Phases are timed live with events
    # on the launching stream (eager launches, no graphs, so events can sit
    # between the kernels).
    eng.use_graphs = False

    def run_steps(n, timers=None):
        def t(s, k):
            if timers is not None:
                timers[s][k].record(stream)
        t(0, 0)
        eng.enq_assign(eng.it & 1, eng.it > 0, eng.cur)
        t(0, 1)
        for s in range(n):
            slot = eng.it & 1
            eng.enq_rest(slot, None, None if timers is None else timers[s][2:4])
            eng.it += 1
            if s + 1 < n:  # speculative: the run continues unless the flags say stop
                t(s + 1, 0)
                eng.enq_assign(eng.it & 1, True, eng.cur ^ 1)
                t(s + 1, 1)
            eng.wait_flags()  # the poll (changed, shift) every iteration reads
            eng.cur ^= 1  # commit

    run_steps(args.warmup)
    torch.cuda.synchronize()
    # this library's kernels per step, counted (not assumed) over one extra
    # untimed step with the CUDA activity profiler
    per_step = count_launches(lambda: run_steps(1))
    if world > 1:
        dist.barrier()
    timers = [[ev() for _ in range(4)] for _ in range(args.steps)]
    t0, t1 = ev(), ev()
    with ClockSampler(local) as clk:
        time.sleep(0.3)  # the sampler is running before the timed region starts
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        clk.mark(True)
        t0.record(stream)
        run_steps(args.steps, timers)
        t1.record(stream)
        torch.cuda.synchronize()
        clk.mark(False)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    ms_local = t0.elapsed_time(t1) / args.steps
    t_assign = statistics.mean(t[0].elapsed_time(t[1]) for t in timers)
    t_obj = statistics.mean(t[1].elapsed_time(t[2]) for t in timers)
    t_update = statistics.mean(t[2].elapsed_time(t[3]) for t in timers)
    ms = ms_local
    if world > 1:
        tt = torch.tensor([ms_local], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())

    parity = parity_check(eng, x, rank) if rank == 0 and not args.no_parity else None

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, x, eng, world, rank, dev, group)

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    pk = peaks()
    flops = 2.0 * n_local * CLUSTERS * DIMS
    ach = flops / (t_assign * 1e-3) / 1e12
    upd_bytes = n_local * DIMS * 2 + 4 * n_local + 4 * CLUSTERS * DIMS + 4 * CLUSTERS
    upd_gbs = upd_bytes / (t_update * 1e-3) / 1e9
    tr = ncu_traffic()
    cpu = None
    if not args.no_cpu:
        threads = os.cpu_count() or 1
        v, dt = cpu_oracle_rate(args.cpu_sample, threads)
        cpu = {"value": v, "unit": "points/s", "cores": threads, "kind": "port",
               "sample": f"{args.cpu_sample} of the workload's points, K={CLUSTERS}, d={DIMS}: one exact "
                         f"Lloyd iteration of the oracle restatement ({dt:.1f} s), rank 0"}
    launches = per_step
    line = {
        "metric": METRIC,
        "value": N_TOTAL / (ms * 1e-3),
        "unit": "points/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": "synthetic (Gaussian blobs drawn on device, random-init centroids)",
        "config": {"workload": f"config 3: N={N_TOTAL}, d={DIMS}, K={CLUSTERS} bf16, one Lloyd iteration "
                               f"per step", "points_per_gpu": n_local, "parallelism": f"point-sharded dp{world}",
                   "comm": (f"{backend} all-reduce of one packed f64 buffer per iteration"
                            if world > 1 else "none"),
                   "l2": "inputs (2 GiB X per GPU at dp1) larger than the 126 MB L2; no flush needed"},
        "gpu_launches": launches * args.steps,
        "roofline": {"bound": "tensor", "kernel": "fk_assign_tc2_kernel", "achieved": ach,
                     "peak": pk["tc_burst"], "unit": "TFLOP/s", "frac": ach / pk["tc_burst"],
                     "frac_of_sustained": ach / pk["tc_sustained"],
                     "peak_source": pk["src"] + " bf16_tflops (burst: the timed region is short)",
                     "algorithmic_flops_per_launch": flops, "ms_per_launch": t_assign,
                     "traffic": tr.get("fk_assign_tc", {}).get("dram_bytes")},
        "roofline_update": {"bound": "hbm", "kernel": "fk_update (colscan+scatter+segsum; the block histogram is built in the assign epilogue)",
                            "achieved": upd_gbs, "peak": pk["hbm"], "unit": "GB/s", "frac": upd_gbs / pk["hbm"],
                            "algorithmic_bytes_per_launch": upd_bytes, "ms_per_launch": t_update,
                            "traffic": update_traffic(tr)},
        "phase_ms": {"assign": t_assign, "objective": t_obj, "update": t_update,
                     "normalize_allreduce_poll": ms_local - t_assign - t_obj - t_update},
        "clocks": clk.summary(),
        "parity": parity,
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    if world > 1 and backend == "nccl":
        line["nccl"] = nccl_summary(os.environ.get("FK_NCCL_LOG_DIR", ""))
        for ln in line["nccl"]["lines"]:
            print("nccl:", ln, file=sys.stderr)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, x, eng, world, rank, dev, group):
    """Same metric through the public API with HOST buffers: every step calls
    ``out_of_core_iteration`` (the drop-in for pipeline.py:385-417), which
    copies the step's centroids and every X chunk of this rank's shard from
    pinned host memory (H2D overlapped with compute on a copy stream), and the
    new centroids are read back to the host.  Sharded runs pass the process
    group: each rank streams its whole chunks, one packed all-reduce per pass."""
    import torch
    import torch.distributed as dist

    from paper_2603_09229_b200 import (Centroids, Counters, DeviceAssignmentStore, HostStream,
                                       KMeansConfig, TilingConfig, out_of_core_iteration)

    # this rank streams whole chunks of the global chunk grid (pipeline.stream_shard);
    # at the bench sizes they coincide with its in-core rows
    n_chunks = -(-N_TOTAL // args.e2e_chunk)
    c_lo, c_hi = n_chunks * rank // world, n_chunks * (rank + 1) // world
    r_lo, r_hi = c_lo * args.e2e_chunk, min(N_TOTAL, c_hi * args.e2e_chunk)
    lo = N_TOTAL * rank // world
    if r_lo == lo and r_hi - r_lo == x.shape[1]:
        host = x.cpu().pin_memory()
    else:
        host = make_shard(r_hi - r_lo, rank, dev).cpu().pin_memory()
    stream = HostStream(host, args.e2e_chunk, pin=False, row_offset=r_lo, total_points=N_TOTAL)
    cfg = KMeansConfig(CLUSTERS, precision="bf16", tiling=TilingConfig(1024, 1024, N_TOTAL))
    c_host = eng.centroids.cpu().pin_memory()
    store = DeviceAssignmentStore(1, r_hi - r_lo, dev, row_offset=r_lo)
    steps = max(1, args.e2e_steps)

    def one():
        new_c, _, _ = out_of_core_iteration(stream, Centroids(c_host, check_finite=False), cfg, Counters(),
                                            store=store, device=dev, group=group)
        return new_c.data.cpu()                                 # D2H of the step's result

    one()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / steps
    if world > 1:
        tt = torch.tensor([dt], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        dt = float(tt.item())
    h2d = (r_hi - r_lo) * DIMS * 2 + CLUSTERS * DIMS * 4
    d2h = CLUSTERS * DIMS * 4
    return {"value": N_TOTAL / dt, "unit": "points/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "h2d_gbs": h2d / dt / 1e9, "steps": steps,
            "api": "paper_2603_09229_b200.out_of_core_iteration over a pinned HostStream of "
                   f"{args.e2e_chunk}-point chunks (copy stream + 2 device buffers)"
                   + (", process group = the bench ranks" if world > 1 else "")}


def relaunch(args) -> int:
    """``--gpus N`` outside torchrun: start N ranks under torch.distributed.run."""
    import torch

    have = torch.cuda.device_count()
    if os.environ.get("FK_BENCH_SHARE_GPU") != "1" and have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} GPUs, {have} visible", file=sys.stderr)
        return 2
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=os.environ.copy())


def count_launches(fn) -> int:
    """Kernels of libflashkmeans.so (namespace fk::) launched by fn, counted with
    torch's CUDA activity profiler; torch's own kernels are excluded."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        fn()
        torch.cuda.synchronize()
    return sum(1 for e in prof.events() if e.device_type.name == "CUDA" and "fk::" in e.name)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=1 << 18)  # 64 MB chunks: 54 GB/s of the 55.5 raw (profiles/r01_e2e_sweep.txt)
    args = ap.parse_args()
    if args.cpu_sample is None:  # reference arm: BASELINE.md §2's 2^20 points; cpu_baseline: ~8 s of host work
        args.cpu_sample = (1 << 20) if args.impl == "reference" else 524288
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch(args))
    if args.gpus > 1 and "NCCL_DEBUG" not in os.environ:
        # NCCL's init report (nranks, NVLS) for the driver: to stderr and a log per rank
        log_dir = os.environ.setdefault("FK_NCCL_LOG_DIR", tempfile.mkdtemp(prefix="fk_nccl_"))
        os.environ["NCCL_DEBUG"] = "INFO"
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", os.path.join(log_dir, "nccl.%h.%p.log"))
    run_ours(args)


if __name__ == "__main__":
    main()
