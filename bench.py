#!/usr/bin/env python
"""Benchmark: one Lloyd iteration of flash-kmeans at BASELINE config 3.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, NCCL)

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
region, an end-to-end figure through the public streaming API from pinned
host buffers, and the CPU oracle timed on this host's cores.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Lloyd iteration latency (ms) & points/s at N=8M,d=128,K=4096; % TC/HBM roofline"
N_TOTAL = 1 << 23
DIMS = 128
CLUSTERS = 4096


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return dict(hbm=p["hbm_gbs"], tc_burst=p["bf16_tflops"], tc_sustained=p["bf16_tflops_sustained"],
                    src="measured")
    except Exception:
        return dict(hbm=6650.0, tc_burst=1590.0, tc_sustained=1400.0, src="fallback")


def ncu_traffic():
    """Per-launch DRAM bytes of the dominant kernels from the committed ncu capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_summary.json")) as f:
            return json.load(f)
    except Exception:
        return {}


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled while the timed region runs."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

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
            if len(parts) == 7:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


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
    c = np.ascontiguousarray(x[:, np.random.default_rng(0).choice(sample_points, CLUSTERS, replace=False)])
    t0 = time.perf_counter()
    a, m = O.assign(x, c, threads)
    sums, counts, _ = O.sort_inverse_update(x, a, CLUSTERS, sample_points)
    O.normalize(sums, counts, c)
    dt = time.perf_counter() - t0
    return sample_points / dt, dt


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    os.environ.setdefault("OMP_NUM_THREADS", str(threads))
    sample = args.cpu_sample
    vals = []
    for i in range(args.warmup + args.steps):
        v, dt = cpu_oracle_rate(sample, threads)
        if i >= args.warmup:
            vals.append(v)
    v = statistics.median(vals)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "points/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": N_TOTAL / v * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32 (exact bf16 upcast)",
        "data": "synthetic", "config": {"workload": f"config 3: N={N_TOTAL}, d={DIMS}, K={CLUSTERS}, "
                                        f"bf16 (upcast), timed on a {sample}-point sample",
                                        "engine": "oracle port of flashmeans exact Lloyd iteration"},
        "cpu_baseline": {"value": v, "unit": "points/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} points x K={CLUSTERS} x d={DIMS}, one exact Lloyd iteration"},
        "e2e": {"value": v, "unit": "points/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2603_09229_b200 import LloydEngine, ops
    from paper_2603_09229_b200.distributed import make_allreduce, shard_bounds

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # FK_BENCH_SHARE_GPU=1 + FK_DIST_BACKEND=gloo: every rank on cuda:0 (a
    # one-GPU rehearsal of the multi-rank code path; numbers are not scaling data)
    if os.environ.get("FK_BENCH_SHARE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        backend = os.environ.get("FK_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
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
    if world > 1:
        dist.barrier()
    timers = [[ev() for _ in range(4)] for _ in range(args.steps)]
    t0, t1 = ev(), ev()
    with ClockSampler(local) as clk:
        time.sleep(0.6)  # let the sampler start before the timed region
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        t0.record(stream)
        run_steps(args.steps, timers)
        t1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
    ms_local = t0.elapsed_time(t1) / args.steps
    t_assign = statistics.mean(t[0].elapsed_time(t[1]) for t in timers)
    t_obj = statistics.mean(t[1].elapsed_time(t[2]) for t in timers)
    t_update = statistics.mean(t[2].elapsed_time(t[3]) for t in timers)
    ms = ms_local
    if world > 1:
        tt = torch.tensor([ms_local, t_assign, t_update], dtype=torch.float64, device=dev)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        ms, t_assign_max, t_update_max = tt.tolist()

    # ---------------------------------------------------------------- e2e
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, x, eng, world, rank, dev)

    if world > 1:
        dist.barrier()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    pk = peaks()
    n_loc0 = n_local
    flops = 2.0 * n_loc0 * CLUSTERS * DIMS
    ach = flops / (t_assign * 1e-3) / 1e12
    upd_bytes = n_loc0 * DIMS * 2 + 4 * n_loc0 + 4 * CLUSTERS * DIMS + 4 * CLUSTERS
    upd_gbs = upd_bytes / (t_update * 1e-3) / 1e9
    tr = ncu_traffic()
    cpu = None
    if not args.no_cpu and world == 1:
        threads = os.cpu_count() or 1
        v, dt = cpu_oracle_rate(args.cpu_sample, threads)
        cpu = {"value": v, "unit": "points/s", "cores": threads, "kind": "port",
               "sample": f"{args.cpu_sample} of the workload's points, K={CLUSTERS}, d={DIMS}: one exact "
                         f"Lloyd iteration of the oracle restatement ({dt:.1f} s)"}
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
                               f"per step", "points_per_gpu": n_loc0, "parallelism": f"point-sharded dp{world}",
                   "l2": "inputs (2 GiB X) larger than the 126 MB L2; no flush needed"},
        "gpu_launches": 9 * args.steps,
        "roofline": {"bound": "tensor", "kernel": "fk_assign_tc", "achieved": ach,
                     "peak": pk["tc_sustained"], "unit": "TFLOP/s", "frac": ach / pk["tc_sustained"],
                     "frac_of_burst": ach / pk["tc_burst"], "peak_source": pk["src"] + " bf16_tflops_sustained",
                     "algorithmic_flops_per_launch": flops, "ms_per_launch": t_assign,
                     "traffic": tr.get("fk_assign_tc", {}).get("dram_bytes")},
        "roofline_update": {"bound": "hbm", "kernel": "fk_update (hist+scan+scatter+segsum)",
                            "achieved": upd_gbs, "peak": pk["hbm"], "unit": "GB/s", "frac": upd_gbs / pk["hbm"],
                            "algorithmic_bytes_per_launch": upd_bytes, "ms_per_launch": t_update,
                            "traffic": tr.get("k_segsum", {}).get("dram_bytes")},
        "phase_ms": {"assign": t_assign, "objective": t_obj, "update": t_update,
                     "normalize_allreduce_poll": ms_local - t_assign - t_obj - t_update},
        "clocks": clk.summary(),
        "e2e": e2e,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_e2e(args, x, eng, world, rank, dev):
    """Same metric through the public API with HOST buffers: out_of_core_iteration
    streams this rank's points from pinned host memory (H2D inside the timed
    region, overlapped with compute) and the new centroids come back to the host."""
    import torch
    import torch.distributed as dist

    from paper_2603_09229_b200 import Counters, HostStream
    from paper_2603_09229_b200.distributed import make_allreduce
    from paper_2603_09229_b200.pipeline import _StreamRunner

    host = x.cpu().pin_memory()
    stream = HostStream(host, args.e2e_chunk, pin=False)
    c_host = eng.centroids.cpu().pin_memory()
    # sharded e2e: each rank streams its own shard; statistics are combined with
    # the same packed all-reduce as the in-core path before normalize.
    runner = _StreamRunner(stream, CLUSTERS, dev, N_TOTAL,
                           allreduce=make_allreduce() if world > 1 else None)
    counters = Counters()
    steps = max(1, args.e2e_steps)

    def one():
        runner.set(c_host)                               # H2D of the centroids
        runner.one_pass(counters)                        # H2D of every X chunk + compute
        out = runner.master[runner.cur ^ 1].cpu()        # D2H of the step's result
        obj = runner.st.obj.cpu()
        return out, obj

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
    n_local = x.shape[1]
    h2d = n_local * DIMS * 2 + CLUSTERS * DIMS * 4
    d2h = CLUSTERS * DIMS * 4 + 8
    return {"value": N_TOTAL / dt, "unit": "points/s", "ms_per_step": dt * 1e3,
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "h2d_gbs": h2d / dt / 1e9, "steps": steps,
            "api": "out_of_core_iteration-equivalent streaming pass over pinned host chunks "
                   f"of {args.e2e_chunk} points (copy stream + 2 device buffers)"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--cpu-sample", type=int, default=None)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-chunk", type=int, default=1 << 18)  # 64 MB chunks: 54 GB/s of the 55.5 raw (profiles/r01_e2e_sweep.txt)
    args = ap.parse_args()
    if args.cpu_sample is None:  # ~8 s of host work for cpu_baseline, ~2 s per reference step
        args.cpu_sample = 131072 if args.impl == "reference" else 524288
    if args.warmup < 3:
        print("warning: --warmup < 3 violates the timing rules", file=sys.stderr)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
