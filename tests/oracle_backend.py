"""A CPU stand-in for paper_2603_09229_b200.ops built on the oracle (TEST ONLY).

It lets the device-agnostic orchestration (LloydEngine's ping-pong buffers,
changed flags, packed all-reduce, normalize-on-every-rank) run under gloo on
CPU tensors so the multi-rank path is covered without GPUs.  The product
never sees this module: LloydEngine defaults to the CUDA ops.
"""

import numpy as np
import torch

from oracle import oracle as O


def assign(x, c, idx_prev=None, changed=None, idx_out=None, mind_out=None):
    a, m = O.assign(x.numpy(), c.numpy())
    idx_out.copy_(torch.from_numpy(a))
    mind_out.copy_(torch.from_numpy(m))
    if idx_prev is not None and bool((idx_prev != idx_out).any()):
        changed.fill_(1)
    return idx_out, mind_out


def objective(mind, out):
    out.copy_(torch.from_numpy(O.objective_row(mind.numpy())))
    return out


def update(x, ids, clusters, chunk=None, accumulate=False, sums=None, counts=None, merges=None):
    s, c, mg = O.sort_inverse_update(x.numpy(), ids.numpy(), clusters, chunk or x.shape[1])
    if accumulate:
        sums += torch.from_numpy(s)
        counts += torch.from_numpy(c)
    else:
        sums.copy_(torch.from_numpy(s))
        counts.copy_(torch.from_numpy(c))
    if merges is not None:
        merges += mg
    return sums, counts


def normalize(sums, counts, prev, out=None, operand_out=None, empty=None, shift2=None):
    new, emp = O.normalize(sums.numpy(), counts.numpy(), prev.numpy())
    diff = new.astype(np.float64) - prev.numpy().astype(np.float64)
    if shift2 is not None:
        shift2.fill_(float(np.square(diff).sum(axis=2).max()))
    out.copy_(torch.from_numpy(new))
    if empty is not None:
        e = np.zeros(empty.shape, np.uint8)
        for b, lst in enumerate(emp):
            e[b, lst] = 1
        empty.copy_(torch.from_numpy(e))
    return out, operand_out, empty


class KmeansppStream:
    """CPU stand-in for ops.KmeansppStream (the (N,) weight table on the host)."""

    def __init__(self, points, clusters, device=None):
        self.n, self.k = int(points), int(clusters)
        self.m = torch.zeros((1, self.n), dtype=torch.float64)
        self.idx = torch.zeros((1, self.k), dtype=torch.int64)
        self.halted = torch.full((1,), self.k, dtype=torch.int32)

    def sweep(self, rows, lo, center, first, j):
        n = rows.shape[0]
        seg = np.ascontiguousarray(self.m[0, lo:lo + n].numpy())
        O.kmeanspp_sweep(rows.double().numpy(), center.double().numpy(), seg, first)
        self.m[0, lo:lo + n] = torch.from_numpy(seg)

    def select(self, j, u):
        m = self.m[0].numpy()
        total = O.pairwise_sum(m)
        if total > 0.0:
            self.idx[0, j] = O.choice_cdf(m, total, u)
        else:
            self.halted[0] = j


def merges_from_counts(counts, chunk, out, accumulate=False):
    """Restatement of k_merges_counts (sort_inverse.py:159-165 on global counts)."""
    c = counts.numpy().astype(np.int64)
    total = 0
    for row in c:
        s = np.concatenate([[0], np.cumsum(row)[:-1]])
        e = s + row
        nz = row > 0
        total += int(((e[nz] - 1) // chunk - s[nz] // chunk + 1).sum())
    if accumulate:
        out += total
    else:
        out.fill_(total)
