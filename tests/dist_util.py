"""Multi-process harness for the sharded tests (TEST ONLY).

``spawn_world(world, fn, *args)`` starts ``world`` spawned processes, each of
which joins a process group on 127.0.0.1 (gloo by default) and calls
``fn(rank, world, *args)``; the per-rank return values come back in rank
order.  A rank that raises fails the test with its traceback.
"""

import os
import queue
import sys
import time
import traceback

import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _entry(rank, world, port, backend, fn, args, q, env):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ.update(env)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    try:
        if backend == "nccl":
            import torch

            dev = torch.device("cuda", rank % max(torch.cuda.device_count(), 1))
            torch.cuda.set_device(dev)
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
        else:
            dist.init_process_group(backend, rank=rank, world_size=world)
        try:
            q.put((rank, "ok", fn(rank, world, *args)))
        finally:
            dist.destroy_process_group()
    except BaseException:
        q.put((rank, "error", traceback.format_exc()))


def spawn_world(world, fn, *args, backend="gloo", timeout=300, env=None):
    port = 20000 + (os.getpid() * 7 + int(time.time() * 1000)) % 20000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_entry, args=(r, world, port, backend, fn, args, q, dict(env or {})))
             for r in range(world)]
    for p in procs:
        p.start()
    res, deadline = {}, time.time() + timeout
    try:
        while len(res) < world and time.time() < deadline:
            try:
                rank, status, val = q.get(timeout=2)
            except queue.Empty:
                if any(p.exitcode not in (None, 0) for p in procs):
                    break
                continue
            if status == "error":
                raise AssertionError(f"rank {rank} failed:\n{val}")
            res[rank] = val
    finally:
        for p in procs:
            if p.exitcode is None and len(res) < world:
                p.terminate()
        for p in procs:
            p.join(timeout=60)
    assert len(res) == world, f"only ranks {sorted(res)} of {world} reported"
    return [res[r] for r in range(world)]
