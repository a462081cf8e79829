"""Edge cases of the GPU path vs the oracle (run on a B200).

Covers the shapes the reference's own tests exercise (ragged tiles, K=1,
N < tile, d not a multiple of the vector width) plus the B200 buckets:
the tensor-core K-atom counts 1-4 (d up to 256), the CUDA-core fallbacks
(d > 256 or d % 8 != 0 for bf16/fp16), the global
histogram path (K beyond the shared-memory bins, BASELINE config 5's
K=65536), and the batched config-4 shape (B=64, d=64, K=256, fp16).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2603_09229_b200 import ops

    return ops


def blobs(B, N, K, d, seed, dtype):
    g = torch.Generator().manual_seed(seed)
    centers = torch.rand((B, max(1, K), d), generator=g) * 20 - 10
    lab = torch.randint(0, centers.shape[1], (B, N), generator=g)
    x = torch.gather(centers, 1, lab[..., None].expand(B, N, d)) + torch.randn((B, N, d), generator=g)
    x = x.to(dtype)
    idx = torch.stack([torch.randperm(N, generator=g)[:K] for _ in range(B)])
    c = torch.stack([x[b, idx[b]] for b in range(B)]).contiguous()
    return x.contiguous(), c


def check_assign(ops, oracle, x, c, exact):
    a, m = ops.assign(x.cuda(), c.cuda())
    torch.cuda.synchronize()
    xf = x.double().numpy() if x.dtype == torch.float64 else x.float().numpy()
    cf = c.double().numpy() if c.dtype == torch.float64 else c.float().numpy()
    a_ref, m_ref = oracle.assign(xf, cf)
    a_gpu = a.cpu().numpy()
    if exact:
        assert np.array_equal(a_gpu, a_ref)
        assert np.array_equal(m.cpu().numpy(), m_ref)
        return
    mism = a_gpu != a_ref
    if mism.any():
        for b in range(xf.shape[0]):
            mb = mism[b]
            if not mb.any():
                continue
            dg = ((xf[b][mb] - cf[b][a_gpu[b][mb]]) ** 2).astype(np.float64).sum(-1)
            dr = ((xf[b][mb] - cf[b][a_ref[b][mb]]) ** 2).astype(np.float64).sum(-1)
            assert np.all(np.abs(dg - dr) <= 1e-3 * dr + 1e-6)
    assert mism.mean() < 1e-3


@pytest.mark.parametrize("B,N,K,d,dtype", [
    (1, 1, 1, 8, torch.bfloat16),         # single point, single centroid
    (1, 5, 3, 16, torch.bfloat16),        # N < tile
    (2, 300, 1, 64, torch.float16),       # K = 1
    (3, 257, 255, 128, torch.bfloat16),   # ragged rows and columns
    (1, 1000, 513, 120, torch.bfloat16),  # d not a multiple of 64 (zero-filled K atom)
    (1, 700, 100, 200, torch.bfloat16),   # d = 200: 4 K atoms on the tensor cores (last one ragged)
    (2, 3000, 700, 256, torch.bfloat16),  # d = 256: widest tensor-core bucket
    (1, 2000, 300, 136, torch.float16),   # d = 136: 3 K atoms, fp16
    (1, 900, 64, 192, torch.float16),     # d = 192, single column tile (alternate-tile epilogue)
    (1, 700, 100, 264, torch.bfloat16),   # d > 256: CUDA-core fallback
    (1, 700, 50, 6, torch.float16),       # d % 8 != 0: CUDA-core fallback
    (64, 16384, 256, 64, torch.float16),  # BASELINE config 4 shape
    (1, 20000, 65536 // 8, 32, torch.bfloat16),
])
def test_assign_shapes(ops, oracle, B, N, K, d, dtype):
    x, c = blobs(B, N, K, d, B * 7 + N + K + d, dtype)
    check_assign(ops, oracle, x, c, exact=False)


@pytest.mark.parametrize("d", [1, 5, 16, 33])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float64])
def test_exact_mirror_ragged(ops, oracle, d, dtype):
    x, c = blobs(2, 333, 17, d, d, dtype)
    check_assign(ops, oracle, x, c, exact=True)


@pytest.mark.parametrize("B,N,K,d,dtype", [
    (1, 70000, 65536, 16, torch.bfloat16),  # global-histogram path (K > shared bins)
    (64, 16384, 256, 64, torch.float16),    # config 4
    (2, 999, 1, 24, torch.float32),         # single cluster
    (1, 1, 1, 8, torch.bfloat16),
    (3, 5000, 700, 36, torch.float16),      # 72-byte rows: generic (non-vector) segsum
])
def test_update_shapes(ops, oracle, B, N, K, d, dtype):
    g = torch.Generator().manual_seed(N + K)
    x = torch.randn((B, N, d), generator=g).to(dtype)
    ids = torch.randint(0, K, (B, N), generator=g, dtype=torch.int32)
    merges = torch.zeros((), dtype=torch.int64, device="cuda")
    sums, counts = ops.update(x.cuda(), ids.cuda(), K, 777, merges=merges)
    torch.cuda.synchronize()
    s_ref, c_ref, m_ref = oracle.sort_inverse_update(x.float().numpy() if dtype != torch.float64 else x.numpy(),
                                                     ids.numpy(), K, 777)
    assert np.array_equal(counts.cpu().numpy(), c_ref)
    assert int(merges.item()) == m_ref
    err = np.abs(sums.cpu().numpy() - s_ref).max()
    assert err <= 1e-6 * max(1.0, float(np.abs(s_ref).max())) * max(1, N // max(1, K)) ** 0.5 + 1e-9


def test_streaming_large_k(ops):
    """Streaming pass with many clusters: chunked == in-core statistics."""
    import paper_2603_09229_b200 as fk

    x, c = blobs(1, 50000, 4096, 32, 5, torch.bfloat16)
    cfg = fk.KMeansConfig(4096, max_iters=2, seed=1, precision="bf16",
                          tiling=fk.TilingConfig(64, 64, 50000))
    r_in = fk.lloyd_run(fk.DataMatrix(x.cuda()), cfg)
    r_st = fk.chunked_stream_run(fk.HostStream(x, 12345), cfg)
    assert r_st.iterations_run == r_in.iterations_run
    assert np.array_equal(r_st.assignments.numpy(), r_in.assignments.numpy())
    np.testing.assert_allclose(r_st.centroids.numpy(), r_in.centroids.numpy(), rtol=1e-5, atol=1e-5)


@pytest.mark.parametrize("d", [136, 200, 256])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_wide_rows_integer_grid_bitwise(ops, oracle, d, dtype):
    """Integer-grid data: every product and sum is exact, so the tensor-core
    result must equal the oracle bit for bit (ids, ties, min_dists) for 3-4
    K atoms as well."""
    g = torch.Generator().manual_seed(d)
    x = torch.randint(-4, 5, (2, 777, d), generator=g).to(dtype)
    c = torch.randint(-4, 5, (2, 300, d), generator=g).to(dtype)
    check_assign(ops, oracle, x, c, exact=True)


def test_config5_shape_fp16_k65536(ops, oracle):
    """BASELINE config 5's precision and shape per chunk (fp16, K=65536, d=128) at
    a reduced N: assign under the near-tie rule, then the update of the GPU's
    own ids -- bit-exact counts and merge count, sums within fp32-accumulation
    bounds -- through the large-K (global histogram) update path."""
    g = torch.Generator().manual_seed(5)
    K, N, d = 65536, 8192, 128
    centers = torch.rand((1, 4096, d), generator=g) * 20 - 10
    lab = torch.randint(0, 4096, (1, N), generator=g)
    x = (torch.gather(centers, 1, lab[..., None].expand(1, N, d)) + torch.randn((1, N, d), generator=g))
    x = x.to(torch.float16).contiguous()
    lab_c = torch.randint(0, 4096, (1, K), generator=g)
    c = (torch.gather(centers, 1, lab_c[..., None].expand(1, K, d))
         + torch.randn((1, K, d), generator=g)).to(torch.float16).contiguous()
    check_assign(ops, oracle, x, c, exact=False)
    ids, _ = ops.assign(x.cuda(), c.cuda())
    merges = torch.zeros((), dtype=torch.int64, device="cuda")
    sums, counts = ops.update(x.cuda(), ids, K, 1000, merges=merges)
    s_ref, c_ref, m_ref = oracle.sort_inverse_update(x.float().numpy(), ids.cpu().numpy(), K, 1000)
    assert np.array_equal(counts.cpu().numpy(), c_ref)
    assert int(merges.item()) == m_ref
    np.testing.assert_allclose(sums.cpu().numpy(), s_ref, rtol=1e-6, atol=1e-4)


_MC_SNIPPET = r"""
import sys, numpy as np, torch
sys.path.insert(0, '.')
from oracle import oracle as O
from paper_2603_09229_b200 import ops
shapes = [(1, 20000, 1000, 128, torch.bfloat16),   # quads only (few tile pairs)
          (1, 4096 * 9 + 300, 529, 64, torch.float16),  # odd tile count: one dummy tile
          (1, 90000 + 77, 300, 128, torch.bfloat16)]    # quads + pair kernel on the leftover SMs
for i, (B, N, K, d, dt) in enumerate(shapes):
    g = torch.Generator().manual_seed(100 + i)
    x = torch.randint(-4, 5, (B, N, d), generator=g).to(dt)
    c = torch.randint(-4, 5, (B, K, d), generator=g).to(dt)
    a, m = ops.assign(x.cuda(), c.cuda())
    a_ref, m_ref = O.assign(x.float().numpy(), c.float().numpy())
    assert np.array_equal(a.cpu().numpy(), a_ref), (N, K, d)
    assert np.array_equal(m.cpu().numpy(), m_ref), (N, K, d)
print('mc ok')
"""


def test_multicast_quads_integer_grid_bitwise():
    """The opt-in multicast-quad FlashAssign (FK_ASSIGN_MC=1: two CTA pairs
    sharing each C tile, plus the pair kernel on the SMs no 4-CTA cluster can
    use) equals the oracle bit for bit, ties included (the switch is read once
    per process, hence the subprocess)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, FK_ASSIGN_MC="1")
    r = subprocess.run([sys.executable, "-c", _MC_SNIPPET], cwd=root, env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "mc ok" in r.stdout, r.stderr[-2000:]
