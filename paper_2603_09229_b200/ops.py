"""Device operators: thin torch wrappers over the C ABI.

Each function takes CUDA tensors, allocates the caller-owned outputs (the
reference's ownership rule: flash_assign.py:162-163, sort_inverse.py:125),
passes raw pointers plus torch's current stream to the library, and returns
tensors.  Nothing here computes on the host; nothing synchronizes.
"""

from __future__ import annotations

import ctypes
import os
import threading

import torch

from . import _native as N

_DT = {torch.float32: N.FK_F32, torch.bfloat16: N.FK_BF16, torch.float16: N.FK_F16,
       torch.float64: N.FK_F64}
LOWP = (torch.bfloat16, torch.float16)


def fk_dtype(t: torch.dtype) -> int:
    try:
        return _DT[t]
    except KeyError:
        raise ValueError(f"unsupported element type {t}; expected float32/float64/bfloat16/float16") from None


def _stream(device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


class _Workspace(threading.local):
    """Per-thread, per-(device, stream) scratch that only grows."""

    def __init__(self):
        self.bufs: dict = {}

    def get(self, device: torch.device, nbytes: int, tag: str = "") -> torch.Tensor | None:
        if nbytes <= 0:
            return None
        key = (device.index, torch.cuda.current_stream(device).cuda_stream, tag)
        buf = self.bufs.get(key)
        if buf is None or buf.numel() < nbytes:
            buf = torch.empty(max(nbytes, 1 << 20), dtype=torch.uint8, device=device)
            self.bufs[key] = buf
        return buf


_ws = _Workspace()


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("device operators take CUDA tensors")
    dev = ts[0].device
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    if idx not in _bound:
        if N.lib().fk_device_supported(idx) != 1:
            raise NotImplementedError("flash-kmeans kernels are compiled for sm_100a (B200) only")
        with torch.cuda.device(idx):  # load every kernel now: no lazy loading on a first shape
            N.check(N.lib().fk_preload(), "fk_preload")
        _bound.add(idx)
    return dev


_bound: set = set()


def assign_bias(c: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """The tensor-core bias operand of bf16/fp16 centroids (B,K,d): (B, kpad, 16)
    bf16 [hi, mid, lo] split of ||c||^2/2 (rows >= K: +inf).  ``assign`` takes
    it to skip its own pass over C; ``normalize(bias_out=)`` writes the next one."""
    dev = _require_cuda(c)
    c = c.contiguous()
    B, K, d = c.shape
    if out is None:
        out = torch.empty((B, N.lib().fk_assign_bias_rows(K), 16), dtype=torch.bfloat16, device=dev)
    N.check(N.lib().fk_assign_bias(fk_dtype(c.dtype), c.data_ptr(), B, K, d, out.data_ptr(), _stream(dev)),
            "fk_assign_bias")
    return out


def split_supported(x: torch.Tensor) -> bool:
    """f32/f64 data whose rows the certified tensor-core assign takes (d <= 128)."""
    B, n, d = x.shape
    return x.dtype in (torch.float32, torch.float64) and N.lib().fk_assign_xsplit_bytes(
        fk_dtype(x.dtype), B, n, d) > 0


def assign_xsplit(x: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """X's operand for the certified tensor-core assign of f32/f64 data (B,N,d),
    d <= 128: a uint8 device buffer holding the (B, N, 32*ceil(d/16)) bf16
    [hi | lo] rows (``xsplit_rows``) and the exact row norms.  Build once per
    data set and pass it to ``assign(xsplit=)`` while X is unchanged."""
    dev = _require_cuda(x)
    x = x.contiguous()
    B, n, d = x.shape
    if not split_supported(x):
        raise ValueError("the split operand needs float32/float64 data with d <= 128")
    nb = N.lib().fk_assign_xsplit_bytes(fk_dtype(x.dtype), B, n, d)
    if out is None:
        out = torch.empty((nb,), dtype=torch.uint8, device=dev)
    elif out.dtype != torch.uint8 or out.numel() < nb:
        raise ValueError("out must be a uint8 buffer of fk_assign_xsplit_bytes")
    N.check(N.lib().fk_assign_xsplit(fk_dtype(x.dtype), x.data_ptr(), B, n, d, out.data_ptr(),
                                     _stream(dev)), "fk_assign_xsplit")
    return out


def split_fallback_rows(x: torch.Tensor, clusters: int) -> list:
    """Diagnostic: rows per batch element that the last certified assign of
    this shape (on this thread and stream) sent to the exact fallback."""
    import ctypes

    dev = _require_cuda(x)
    B, n, d = x.shape
    ws = _ws.get(dev, 1, "assign")
    out = (ctypes.c_int32 * B)()
    N.check(N.lib().fk_assign_split_fallback_rows(fk_dtype(x.dtype), B, n, int(clusters), d, ws.data_ptr(),
                                                  ctypes.addressof(out), _stream(dev)),
            "fk_assign_split_fallback_rows")
    return list(out)


def xsplit_rows(xsplit: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
    """The (B, N, 32*ceil(d/16)) bf16 [hi | lo] rows inside ``assign_xsplit(x)``."""
    B, n, d = x.shape
    w = 32 * (-(-d // 16))
    return xsplit[: B * n * w * 2].view(torch.bfloat16).view(B, n, w)


_DOT = {"exact": 0, "fast": 1, "mirror": 2}
SPLIT_MIN_MACS = 6.7e7  # fk_api.cu split_auto: below this the exact mirror is faster


def split_auto(x: torch.Tensor, clusters: int) -> bool:
    """Whether ``assign`` on this data picks the certified tensor-core path by
    itself (same rule as the library: FK_ASSIGN_F32=mirror|split overrides)."""
    if not split_supported(x):
        return False
    env = os.environ.get("FK_ASSIGN_F32", "")
    if env[:1] in ("m", "s"):
        return env[0] == "s"
    B, n, d = x.shape
    return float(B) * n * clusters * d >= SPLIT_MIN_MACS


class HistFold:
    """An update workspace whose block histogram table the assign fills
    (fk_assign_hist -> fk_update_prehist): the update's first pass (k_hist)
    folded into the FlashAssign epilogue.  The table must be zero before an
    assign adds into it; fk_update_prehist leaves it zeroed again, so only a
    pair broken off after the assign (a speculative assign whose update never
    ran) needs ``clear()``."""

    def __init__(self, ws: torch.Tensor, table: int, inval: int, bpb: int, per: int, words: int):
        self.ws, self.table, self.inval, self.bpb, self.per = ws, table, inval, bpb, per
        off = table - ws.data_ptr()
        self._clear = ws[off:off + 4 * words]

    def clear(self) -> None:
        self._clear.zero_()


def hist_fold(x: torch.Tensor, clusters: int) -> HistFold | None:
    """A HistFold for (B,N,d) bf16/fp16 data and K clusters, or None where the
    fold is not offered (f32/f64 data, K > 16384, no tensor-core path)."""
    dev = _require_cuda(x)
    if x.dtype not in LOWP or x.dim() != 3:
        return None
    B, n, d = x.shape
    K = int(clusters)
    dt = fk_dtype(x.dtype)
    L = N.lib()
    ws = torch.zeros((int(L.fk_update_workspace(dt, B, n, K, d)),), dtype=torch.uint8, device=dev)
    tab, inv = ctypes.c_void_p(), ctypes.c_void_p()
    bpb, per, words = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    st = L.fk_update_hist_slots(dt, B, n, K, d, ws.data_ptr(), ctypes.byref(tab), ctypes.byref(inv),
                                ctypes.byref(bpb), ctypes.byref(per), ctypes.byref(words))
    if st == N.FK_EUNSUPPORTED:
        return None
    N.check(st, "fk_update_hist_slots")
    return HistFold(ws, tab.value, inv.value, bpb.value, per.value, words.value)


def assign_row_norms(x: torch.Tensor, clusters: int) -> torch.Tensor | None:
    """(B,N) fp32 ||x||^2 of bf16/fp16 data summed exactly as the tensor-core
    epilogue sums it for K = ``clusters`` (fk_assign_row_norms), or None where
    that path is not taken."""
    dev = _require_cuda(x)
    if x.dtype not in LOWP or x.dim() != 3:
        return None
    x = x.contiguous()
    B, n, d = x.shape
    out = torch.empty((B, n), dtype=torch.float32, device=dev)
    st = N.lib().fk_assign_row_norms(fk_dtype(x.dtype), x.data_ptr(), B, n, int(clusters), d,
                                     out.data_ptr(), _stream(dev))
    if st == N.FK_EUNSUPPORTED:
        return None
    N.check(st, "fk_assign_row_norms")
    return out


def assign(x: torch.Tensor, c: torch.Tensor, idx_prev: torch.Tensor | None = None,
           changed: torch.Tensor | None = None, idx_out: torch.Tensor | None = None,
           mind_out: torch.Tensor | None = None, bias: torch.Tensor | None = None,
           xsplit: torch.Tensor | None = None, dot_mode: str = "exact", path: str = "auto",
           hist: HistFold | None = None, xnorm: torch.Tensor | None = None):
    """Nearest centroid per point: (ids int32 (B,N), min_dists (B,N)).

    min_dists is in the data dtype for float32/float64 data and float32 for
    bfloat16/float16 data.  If ``idx_prev`` is given, ``changed`` (int32
    device scalar) is OR-ed with 1 when any id differs.  ``bias`` (bf16/fp16
    only): the precomputed ``assign_bias(c)``.

    float32/float64 data (the reference's dot modes, flash_assign.py:203-208):
    ``dot_mode="exact"`` is bitwise equal to the reference; for d <= 128 it
    runs the certified tensor-core path (``xsplit``: the cached
    ``assign_xsplit(x)``).  ``"fast"`` (the reference's relaxed mode) is
    served by the same certified path, so it returns the exact answer.  ``path``: "auto" | "split" | "mirror" (the exact
    CUDA-core kernel for every row) -- A/B and tests.
    ``hist`` (bf16/fp16): also add the ids into that HistFold's block table
    for a following ``update(..., hist=hist)``; ``xnorm`` (with ``hist``):
    ``assign_row_norms(x, K)`` of this data, min_dists unchanged bitwise.
    """
    dev = _require_cuda(x, c)
    if x.dim() != 3 or c.dim() != 3 or x.shape[0] != c.shape[0] or x.shape[2] != c.shape[2]:
        raise ValueError("x must be (B,N,d) and c (B,K,d) with matching B and d")
    if x.dtype != c.dtype:
        raise ValueError("data and centroids must share one precision")
    if dot_mode not in ("exact", "fast"):
        raise ValueError("dot_mode must be 'exact' or 'fast'")
    if path not in ("auto", "split", "mirror"):
        raise ValueError("path must be 'auto', 'split' or 'mirror'")
    x = x.contiguous()
    c = c.contiguous()
    B, n, d = x.shape
    K = c.shape[1]
    dt = fk_dtype(x.dtype)
    if idx_out is None:
        idx_out = torch.empty((B, n), dtype=torch.int32, device=dev)
    if mind_out is None:
        mdt = torch.float32 if x.dtype in LOWP else x.dtype
        mind_out = torch.empty((B, n), dtype=mdt, device=dev)
    L = N.lib()
    if x.dtype not in LOWP and (xsplit is not None or dot_mode == "fast" or path != "auto"):
        mode = "mirror" if path == "mirror" or not split_supported(x) else dot_mode
        if mode != "mirror" and xsplit is None:
            xsplit = assign_xsplit(x)
        if xsplit is not None and (xsplit.dtype != torch.uint8 or not xsplit.is_contiguous()
                                   or xsplit.numel() < L.fk_assign_xsplit_bytes(dt, B, n, d)):
            raise ValueError("xsplit must be assign_xsplit(x) of this data")
        need = L.fk_assign_split_workspace(dt, B, n, K, d)
        ws = _ws.get(dev, need, "assign")
        st = L.fk_assign_split(dt, x.data_ptr(), None if mode == "mirror" else xsplit.data_ptr(),
                               c.data_ptr(), B, n, K, d, _DOT[mode], idx_out.data_ptr(),
                               mind_out.data_ptr(), None if idx_prev is None else idx_prev.data_ptr(),
                               None if changed is None else changed.data_ptr(), ws.data_ptr(),
                               ws.numel(), _stream(dev))
        N.check(st, "fk_assign_split")
        return idx_out, mind_out
    need = L.fk_assign_workspace(dt, B, n, K, d)
    ws = _ws.get(dev, need, "assign")
    if hist is not None:
        st = L.fk_assign_hist(dt, x.data_ptr(), c.data_ptr(), None if bias is None else bias.data_ptr(),
                              B, n, K, d, idx_out.data_ptr(), mind_out.data_ptr(),
                              None if idx_prev is None else idx_prev.data_ptr(),
                              None if changed is None else changed.data_ptr(),
                              None if ws is None else ws.data_ptr(), 0 if ws is None else ws.numel(),
                              hist.table, hist.inval, hist.bpb, hist.per,
                              None if xnorm is None else xnorm.data_ptr(), _stream(dev))
        N.check(st, "fk_assign_hist")
        return idx_out, mind_out
    st = L.fk_assign(dt, x.data_ptr(), c.data_ptr(), None if bias is None else bias.data_ptr(),
                     B, n, K, d, idx_out.data_ptr(),
                     mind_out.data_ptr(), None if idx_prev is None else idx_prev.data_ptr(),
                     None if changed is None else changed.data_ptr(),
                     None if ws is None else ws.data_ptr(), 0 if ws is None else ws.numel(),
                     _stream(dev))
    N.check(st, "fk_assign")
    return idx_out, mind_out


def update(x: torch.Tensor, ids: torch.Tensor, clusters: int, chunk: int | None = None,
           accumulate: bool = False, sums: torch.Tensor | None = None,
           counts: torch.Tensor | None = None, merges: torch.Tensor | None = None,
           hist: HistFold | None = None):
    """Sort-inverse cluster statistics: (sums f64 (B,K,d), counts int64 (B,K)).

    ``merges`` (int64 device scalar, optional) is incremented by the segment
    count the reference's sort_inverse_update would record for ``chunk``.
    ``hist``: the HistFold the preceding ``assign(..., hist=)`` filled (no
    histogram pass here; the table is left zeroed).
    """
    dev = _require_cuda(x, ids)
    x = x.contiguous()
    ids = ids.contiguous()
    B, n, d = x.shape
    if ids.shape != (B, n) or ids.dtype != torch.int32:
        raise ValueError("ids must be int32 (B,N) matching x")
    K = int(clusters)
    dt = fk_dtype(x.dtype)
    if sums is None:
        sums = torch.empty((B, K, d), dtype=torch.float64, device=dev)
    if counts is None:
        counts = torch.empty((B, K), dtype=torch.int64, device=dev)
    L = N.lib()
    need = L.fk_update_workspace(dt, B, n, K, d)
    if hist is not None:
        st = L.fk_update_prehist(dt, x.data_ptr(), ids.data_ptr(), B, n, K, d, int(chunk or n),
                                 1 if accumulate else 0, sums.data_ptr(), counts.data_ptr(),
                                 None if merges is None else merges.data_ptr(), hist.ws.data_ptr(),
                                 hist.ws.numel(), _stream(dev))
        N.check(st, "fk_update_prehist")
        return sums, counts
    ws = _ws.get(dev, need, "update")
    st = L.fk_update(dt, x.data_ptr(), ids.data_ptr(), B, n, K, d, int(chunk or n),
                     1 if accumulate else 0, sums.data_ptr(), counts.data_ptr(),
                     None if merges is None else merges.data_ptr(), ws.data_ptr(), ws.numel(),
                     _stream(dev))
    N.check(st, "fk_update")
    return sums, counts


def argsort(ids: torch.Tensor, clusters: int):
    """Stable device counting sort of (B,N) int32 ids: (order int32 (B*N,) flat
    point indices grouped by key b*K + id, offsets int64 (B*K+1,))."""
    dev = _require_cuda(ids)
    ids = ids.contiguous()
    B, n = ids.shape
    K = int(clusters)
    order = torch.empty((B * n,), dtype=torch.int32, device=dev)
    offsets = torch.empty((B * K + 1,), dtype=torch.int64, device=dev)
    L = N.lib()
    need = L.fk_update_workspace(N.FK_F32, B, n, K, 1)
    ws = _ws.get(dev, need, "update")
    st = L.fk_argsort(ids.data_ptr(), B, n, K, order.data_ptr(), offsets.data_ptr(), ws.data_ptr(),
                      ws.numel(), _stream(dev))
    N.check(st, "fk_argsort")
    return order, offsets


def normalize(sums: torch.Tensor, counts: torch.Tensor, prev: torch.Tensor,
              out: torch.Tensor | None = None, operand_dtype: torch.dtype | None = None,
              operand_out: torch.Tensor | None = None, empty: torch.Tensor | None = None,
              shift2: torch.Tensor | None = None, bias_out: torch.Tensor | None = None):
    """c = sums/counts (empty clusters keep ``prev`` bitwise).

    ``prev``/``out`` are float32 or float64 masters; ``operand_out`` gets the
    rounded copy in ``operand_dtype`` (the next MMA operand).  ``shift2``
    (f64 device scalar, pre-zeroed) receives max_k ||out_k - prev_k||^2.
    Returns (out, operand_out, empty_mask uint8 (B,K)).
    """
    dev = _require_cuda(sums, counts, prev)
    B, K, d = prev.shape
    mdt = fk_dtype(prev.dtype)
    if prev.dtype not in (torch.float32, torch.float64):
        raise ValueError("centroid masters are float32 or float64")
    if out is None:
        out = torch.empty_like(prev)
    if operand_dtype is not None and operand_out is None:
        operand_out = torch.empty((B, K, d), dtype=operand_dtype, device=dev)
    if empty is None:
        empty = torch.empty((B, K), dtype=torch.uint8, device=dev)
    odt = fk_dtype(operand_out.dtype) if operand_out is not None else 0
    st = N.lib().fk_normalize(mdt, sums.data_ptr(), counts.data_ptr(), prev.data_ptr(),
                              out.data_ptr(), odt,
                              None if operand_out is None else operand_out.data_ptr(),
                              empty.data_ptr(), None if shift2 is None else shift2.data_ptr(),
                              B, K, d, None if bias_out is None else bias_out.data_ptr(), _stream(dev))
    N.check(st, "fk_normalize")
    return out, operand_out, empty


def objective(mind: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """Per-batch float64 sum of min_dists (pipeline._objective_row)."""
    dev = _require_cuda(mind)
    B, n = mind.shape
    if out is None:
        out = torch.empty((B,), dtype=torch.float64, device=dev)
    L = N.lib()
    need = L.fk_objective_workspace(B, n)
    ws = _ws.get(dev, need, "objective")
    st = L.fk_objective(fk_dtype(mind.dtype), mind.data_ptr(), B, n, out.data_ptr(),
                        ws.data_ptr(), ws.numel(), _stream(dev))
    N.check(st, "fk_objective")
    return out


OBJ_BLOCK = 8192  # elements per objective partial: numpy's reduction buffer (fk_objective_partials)


def objective_partials(mind: torch.Tensor, out: torch.Tensor) -> torch.Tensor:
    """Fixed-order f64 partial sums of (B,N) min_dists into out (B * ceil(N/8192),)."""
    dev = _require_cuda(mind, out)
    B, n = mind.shape
    N.check(N.lib().fk_objective_partials(fk_dtype(mind.dtype), mind.data_ptr(), B, n, out.data_ptr(),
                                          _stream(dev)), "fk_objective_partials")
    return out


def loop_tail(partials: torch.Tensor, B: int, n: int, obj: torch.Tensor, changed: torch.Tensor,
              shift2: torch.Tensor, merges: torch.Tensor, flags: torch.Tensor,
              history: torch.Tensor | None = None, history_row: torch.Tensor | None = None) -> None:
    """One launch at the end of an iteration: objective (+ history row), the
    [changed, shift^2, merges] flags, and the accumulators cleared."""
    dev = _require_cuda(partials, obj, changed, shift2, merges, flags)
    N.check(N.lib().fk_loop_tail(partials.data_ptr(), B, n, obj.data_ptr(),
                                 None if history is None else history.data_ptr(),
                                 None if history_row is None else history_row.data_ptr(),
                                 changed.data_ptr(), shift2.data_ptr(), merges.data_ptr(),
                                 flags.data_ptr(), _stream(dev)), "fk_loop_tail")


def normalize_loop_tail(sums, counts, prev, out, operand_out, empty, shift2, bias_out, mind, partials,
                        obj, changed, merges, flags, counter, history=None, history_row=None) -> None:
    """normalize + objective partials + loop tail in one launch (fk_normalize_loop_tail)."""
    dev = _require_cuda(sums, counts, prev, mind)
    B, K, d = prev.shape
    n = mind.shape[1]
    odt = fk_dtype(operand_out.dtype) if operand_out is not None else 0
    N.check(N.lib().fk_normalize_loop_tail(
        fk_dtype(prev.dtype), sums.data_ptr(), counts.data_ptr(), prev.data_ptr(), out.data_ptr(), odt,
        None if operand_out is None else operand_out.data_ptr(), empty.data_ptr(), shift2.data_ptr(),
        B, K, d, None if bias_out is None else bias_out.data_ptr(), fk_dtype(mind.dtype), mind.data_ptr(),
        n, partials.data_ptr(), obj.data_ptr(), None if history is None else history.data_ptr(),
        None if history_row is None else history_row.data_ptr(), changed.data_ptr(), merges.data_ptr(),
        flags.data_ptr(), counter.data_ptr(), _stream(dev)), "fk_normalize_loop_tail")


FARTHEST_EMAX = 8192


def farthest(mind: torch.Tensor, take: int) -> torch.Tensor:
    """The ``take`` points with the largest (B,N) min_dists, distance descending
    then index ascending (the reference's _farthest_order): (B, take) int64."""
    dev = _require_cuda(mind)
    mind = mind.contiguous()
    B, n = mind.shape
    take = int(take)
    if not 1 <= take <= n:
        raise ValueError("take must be in [1, N]")
    if mind.dtype not in (torch.float32, torch.float64):
        mind = mind.float()
    out = torch.empty((B, take), dtype=torch.int64, device=dev)
    L = N.lib()
    ws = _ws.get(dev, L.fk_farthest_workspace(B, take), "farthest")
    N.check(L.fk_farthest(fk_dtype(mind.dtype), mind.data_ptr(), B, n, take, out.data_ptr(), ws.data_ptr(),
                          ws.numel(), _stream(dev)), "fk_farthest")
    return out


def row_norms(m: torch.Tensor) -> torch.Tensor:
    """Exact row norms of a (rows, d) float32/float64 CUDA matrix (core.row_norms)."""
    dev = _require_cuda(m)
    m = m.contiguous()
    out = torch.empty((m.shape[0],), dtype=m.dtype, device=dev)
    st = N.lib().fk_row_norms(fk_dtype(m.dtype), m.data_ptr(), m.shape[0], m.shape[1],
                              out.data_ptr(), _stream(dev))
    N.check(st, "fk_row_norms")
    return out


def scatter(x: torch.Tensor, ids: torch.Tensor, clusters: int):
    """Contended atomic scatter (baseline.scatter_update foil, ncu comparisons only)."""
    dev = _require_cuda(x, ids)
    B, n, d = x.shape
    sums = torch.empty((B, clusters, d), dtype=torch.float64, device=dev)
    counts = torch.empty((B, clusters), dtype=torch.int64, device=dev)
    st = N.lib().fk_scatter(fk_dtype(x.dtype), x.contiguous().data_ptr(), ids.contiguous().data_ptr(),
                            B, n, clusters, d, sums.data_ptr(), counts.data_ptr(), _stream(dev))
    N.check(st, "fk_scatter")
    return sums, counts


def kmeanspp(x: torch.Tensor, clusters: int, first: torch.Tensor, u: torch.Tensor):
    """Device k-means++ D^2 seeding (core._kmeanspp_indices, core.py:342-357).

    ``first`` (B,) int64 holds each batch element's rng.integers(N) draw and
    ``u`` (B, K-1) float64 the rng.random() doubles of draws 1..K-1 (the RNG
    stays with the caller).  Returns (idx int64 (B,K), halted int32 (B,)):
    halted[b] < K marks the first draw whose total was 0 -- the reference
    switches to rng.integers(N) from there, which the caller replays.
    """
    dev = _require_cuda(x, first, u)
    x = x.contiguous()
    B, n, d = x.shape
    K = int(clusters)
    if first.shape != (B,) or u.shape != (B, max(K - 1, 0)) or u.dtype != torch.float64:
        raise ValueError("first must be (B,) and u float64 (B, K-1)")
    idx = torch.zeros((B, K), dtype=torch.int64, device=dev)
    idx[:, 0] = first.to(torch.int64)
    halted = torch.empty((B,), dtype=torch.int32, device=dev)
    m = torch.empty((B, n), dtype=torch.float64, device=dev)
    L = N.lib()
    need = L.fk_kmeanspp_workspace(B, n, K, d)
    ws = _ws.get(dev, need, "kmeanspp")
    u = u.contiguous()
    st = L.fk_kmeanspp(fk_dtype(x.dtype), x.data_ptr(), B, n, d, K, u.data_ptr() if K > 1 else None,
                       idx.data_ptr(), halted.data_ptr(), m.data_ptr(), ws.data_ptr(), ws.numel(),
                       _stream(dev))
    N.check(st, "fk_kmeanspp")
    return idx, halted


class KmeansppStream:
    """Streamed k-means++ pieces (pipeline._streaming_kmeanspp, pipeline.py:420-453):
    the (N,) f64 weight table lives on the device, chunks of rows are swept
    as they arrive, and ``select`` resolves one rng.choice draw."""

    def __init__(self, points: int, clusters: int, device):
        self.n, self.k, self.dev = int(points), int(clusters), torch.device(device)
        self.m = torch.empty((1, self.n), dtype=torch.float64, device=self.dev)
        self.idx = torch.zeros((1, self.k), dtype=torch.int64, device=self.dev)
        self.halted = torch.empty((1,), dtype=torch.int32, device=self.dev)
        self.u = torch.zeros((1, max(self.k - 1, 1)), dtype=torch.float64, device=self.dev)
        L = N.lib()
        need = L.fk_kmeanspp_workspace(1, self.n, 0, 0)
        self.ws = torch.empty(max(need, 256), dtype=torch.uint8, device=self.dev)
        N.check(L.fk_kmeanspp_init(self.halted.data_ptr(), 1, self.n, self.k, self.ws.data_ptr(),
                                   self.ws.numel(), _stream(self.dev)), "fk_kmeanspp_init")

    def sweep(self, rows: torch.Tensor, lo: int, center: torch.Tensor, first: bool, j: int) -> None:
        """min_d2[lo:lo+len(rows)] <- D^2 against ``center`` for draw j."""
        rows = rows.contiguous()
        n, d = rows.shape
        center = center.contiguous()
        st = N.lib().fk_kmeanspp_sweep(fk_dtype(rows.dtype), rows.data_ptr(), 1, n, d, n * d,
                                       center.data_ptr(), d, self.m[0, lo:].data_ptr(), self.n,
                                       1 if first else 0, self.halted.data_ptr(), int(j),
                                       _stream(self.dev))
        N.check(st, "fk_kmeanspp_sweep")

    def select(self, j: int, u: float) -> None:
        self.u[0, j - 1] = u
        st = N.lib().fk_kmeanspp_select(self.m.data_ptr(), 1, self.n, self.u.data_ptr(), self.k,
                                        int(j), self.idx.data_ptr(), self.halted.data_ptr(),
                                        self.ws.data_ptr(), self.ws.numel(), _stream(self.dev))
        N.check(st, "fk_kmeanspp_select")


def stats_pack(counts: torch.Tensor, obj: torch.Tensor, changed: torch.Tensor, red_tail: torch.Tensor,
               unpack: bool = False) -> None:
    """[counts | objective | changed] <-> the f64 tail of the all-reduce buffer (one launch)."""
    dev = _require_cuda(counts, obj, changed, red_tail)
    BK, B = counts.numel(), obj.numel()
    st = N.lib().fk_stats_pack(1 if unpack else 0, counts.data_ptr(), obj.data_ptr(), changed.data_ptr(),
                               red_tail.data_ptr(), BK, B, _stream(dev))
    N.check(st, "fk_stats_pack")


def merges_from_counts(counts: torch.Tensor, chunk: int, out: torch.Tensor, accumulate: bool = False) -> None:
    """The reference's synchronized_merges for one update, from GLOBAL (B,K) int64
    counts (sharded runs: evaluated after the all-reduce); ``out`` int64 scalar."""
    dev = _require_cuda(counts, out)
    B, K = counts.shape
    st = N.lib().fk_merges_from_counts(counts.data_ptr(), B, K, int(chunk), out.data_ptr(),
                                       1 if accumulate else 0, _stream(dev))
    N.check(st, "fk_merges_from_counts")
