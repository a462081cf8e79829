"""GPU parity of the C-ABI kernels against the CPU oracle (run on a B200).

Bars (BASELINE.json north_star):
  * assignments identical except documented near-ties: |d64(a_gpu) - d64(a_ref)|
    <= 1e-3 * d64(a_ref) for bf16/fp16, both recomputed in f64 from the exact
    fp32 upcast of the same inputs; bit-exact for f32/f64 and for integer-grid
    bf16 inputs (every product and sum is exact there);
  * counts bit-exact given identical assignments;
  * centroids <= 1e-3 relative (row-norm relative error).
"""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

NEAR_TIE_RTOL = 1e-3


@pytest.fixture(scope="module")
def ops():
    from paper_2603_09229_b200 import ops

    return ops


def d64(x, c, a):
    """Exact f64 squared distance of each point to centroid a (B,N)."""
    B, N, _ = x.shape
    out = np.empty((B, N))
    for b in range(B):
        diff = x[b].astype(np.float64) - c[b].astype(np.float64)[a[b]]
        out[b] = np.einsum("ij,ij->i", diff, diff)
    return out


def check_near_tie(x32, c32, a_gpu, a_ref, rtol=NEAR_TIE_RTOL):
    mism = a_gpu != a_ref
    if not mism.any():
        return 0
    dg = d64(x32, c32, a_gpu)[mism]
    dr = d64(x32, c32, a_ref)[mism]
    assert np.all(np.abs(dg - dr) <= rtol * np.maximum(dr, 1e-30) + 1e-30), (
        f"{mism.sum()} non-near-tie mismatches")
    return int(mism.sum())


def grid_case(golden, name, dtype):
    arr, _ = golden
    x = arr[name + "_x"].astype(np.float32)
    c = arr[name + "_c"].astype(np.float32)
    return x, c, arr[name + "_a"], arr[name + "_m"]


@pytest.mark.parametrize("name", ["grid_small", "grid_d64", "grid_d128"])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_tc_assign_integer_grid_bitwise(ops, golden, name, dtype):
    """Integer grid: tensor-core result must equal the reference bit for bit (ties included)."""
    x, c, a_ref, m_ref = grid_case(golden, name, dtype)
    xt = torch.from_numpy(x).to(dtype).cuda()
    ct = torch.from_numpy(c).to(dtype).cuda()
    a, m = ops.assign(xt, ct)
    torch.cuda.synchronize()
    assert np.array_equal(a.cpu().numpy(), a_ref)
    assert np.array_equal(m.cpu().numpy(), m_ref.astype(np.float32))


@pytest.mark.parametrize("B,N,K,d", [(1, 4096, 1024, 128), (1, 1000, 300, 128), (3, 777, 257, 64),
                                     (2, 513, 37, 32), (1, 300, 1, 16), (1, 128, 4096, 128),
                                     (1, 20000, 4096, 128)])
def test_tc_assign_random_near_tie(ops, oracle, B, N, K, d):
    g = torch.Generator().manual_seed(B * 1000003 + N * 7 + K * 13 + d)
    centers = torch.rand((B, max(1, K // 4), d), generator=g) * 20 - 10
    lab = torch.randint(0, centers.shape[1], (B, N), generator=g)
    x = torch.gather(centers, 1, lab[..., None].expand(B, N, d)) + torch.randn((B, N, d), generator=g)
    xb = x.to(torch.bfloat16)
    perm = torch.randperm(N, generator=g)[: min(K, N)]
    cb = xb[:, perm] if K <= N else torch.randn((B, K, d), generator=g).to(torch.bfloat16)
    a, m = ops.assign(xb.cuda(), cb.cuda())
    torch.cuda.synchronize()
    x32 = xb.float().numpy()
    c32 = cb.float().numpy()
    a_ref, m_ref = oracle.assign(x32, c32)
    a_gpu = a.cpu().numpy()
    check_near_tie(x32, c32, a_gpu, a_ref)
    # min_dists: tolerance relative to the distance scale
    dd = d64(x32, c32, a_gpu)
    np.testing.assert_allclose(m.cpu().numpy(), dd, rtol=1e-3, atol=1e-2 * max(1.0, dd.mean()) * 1e-2)


@pytest.mark.parametrize("prec,dt", [("single", np.float32), ("double", np.float64)])
def test_exact_mirror_bitwise(ops, golden, oracle, prec, dt):
    arr, meta = golden
    spec = meta["fixtures"][f"assign_{prec}"]
    x = oracle.generate_dataset(spec["batch"], spec["points"], spec["k_true"], spec["dims"],
                                spec["spread"], spec["seed"], dt)
    c = arr[f"assign_{prec}_c"]
    a, m = ops.assign(torch.from_numpy(x).cuda(), torch.from_numpy(c).cuda())
    torch.cuda.synchronize()
    assert np.array_equal(a.cpu().numpy(), arr[f"assign_{prec}_a"])
    assert np.array_equal(m.cpu().numpy(), arr[f"assign_{prec}_m"])


@pytest.mark.parametrize("prec,dt", [("single", np.float32), ("double", np.float64)])
def test_update_normalize_golden(ops, golden, oracle, prec, dt):
    arr, meta = golden
    spec = meta["fixtures"][f"update_{prec}"]
    x = torch.from_numpy(oracle.generate_dataset(2, 1000, 9, 6, 1.0, 7, dt)).cuda()
    ids = torch.from_numpy(arr[f"update_{prec}_ids"]).cuda()
    merges = torch.zeros((), dtype=torch.int64, device="cuda")
    sums, counts = ops.update(x, ids, spec["clusters"], spec["chunk"], merges=merges)
    prev = torch.from_numpy(arr[f"update_{prec}_prev"]).cuda()
    out, _, empty = ops.normalize(sums, counts, prev)
    torch.cuda.synchronize()
    assert np.array_equal(counts.cpu().numpy(), arr[f"update_{prec}_counts"])
    assert int(merges.item()) == spec["merges"]
    s_ref = arr[f"update_{prec}_sums"]
    if prec == "single":
        assert np.array_equal(sums.cpu().numpy(), s_ref)  # f64 sums of f32 addends are exact
        assert np.array_equal(out.cpu().numpy(), arr[f"update_{prec}_norm"])
    else:
        np.testing.assert_allclose(sums.cpu().numpy(), s_ref, rtol=1e-12, atol=1e-12)
        np.testing.assert_allclose(out.cpu().numpy(), arr[f"update_{prec}_norm"], rtol=1e-12)
    assert [list(np.flatnonzero(e)) for e in empty.cpu().numpy()] == spec["empty"]


@pytest.mark.parametrize("B,N,K,d,dtype", [(1, 200000, 1024, 128, torch.bfloat16),
                                           (2, 50000, 300, 64, torch.float16),
                                           (1, 10000, 8, 16, torch.float32),
                                           (4, 3000, 77, 24, torch.bfloat16),
                                           (1, 5000, 50, 6, torch.float32),
                                           (1, 4097, 4096, 128, torch.bfloat16)])
def test_update_vs_oracle(ops, oracle, B, N, K, d, dtype):
    g = torch.Generator().manual_seed(N + K + d)
    x = torch.randn((B, N, d), generator=g).to(dtype)
    ids = torch.randint(0, K, (B, N), generator=g, dtype=torch.int32)
    # Zipf-ish skew: a few giant clusters spanning many warp slices
    ids[:, : N // 3] = ids[:, : N // 3] % 3
    sums, counts = ops.update(x.cuda(), ids.cuda(), K, 4096)
    torch.cuda.synchronize()
    s_ref, c_ref, _ = oracle.sort_inverse_update(x.float().numpy(), ids.numpy(), K, 4096)
    assert np.array_equal(counts.cpu().numpy(), c_ref)
    s = sums.cpu().numpy()
    if dtype == torch.float32:
        assert np.array_equal(s, s_ref)
    else:
        # fp32 accumulation inside a warp slice: error bounded relative to sum |x|
        err = np.linalg.norm(s - s_ref, axis=-1)
        scale = (c_ref + 1) * np.sqrt(d)
        assert np.all(err <= 1e-6 * scale)


@pytest.mark.parametrize("B,N,K", [(1, 5_000_003, 4096), (2, 2_600_001, 3001)])
def test_update_staged_scatter_vs_oracle(ops, oracle, B, N, K):
    """Shapes whose per-block point ranges span more than one 16K-point sub-tile
    on a 148-SM B200 (the staged shared-memory counting sort of the scatter):
    counts, merges and f32 sums bit-exact against the reference restatement,
    with ragged sub-tiles and skewed keys."""
    d = 8
    g = torch.Generator().manual_seed(N + K)
    # small integers (as f32): every partial sum is exact in any order
    x = torch.randint(-8, 9, (B, N, d), generator=g).float()
    ids = torch.randint(0, K, (B, N), generator=g, dtype=torch.int32)
    ids[:, : N // 4] = ids[:, : N // 4] % 5
    merges = torch.zeros((), dtype=torch.int64, device="cuda")
    sums, counts = ops.update(x.cuda(), ids.cuda(), K, 65536, merges=merges)
    torch.cuda.synchronize()
    s_ref, c_ref, m_ref = oracle.sort_inverse_update(x.numpy(), ids.numpy(), K, 65536)
    assert np.array_equal(counts.cpu().numpy(), c_ref)
    assert np.array_equal(sums.cpu().numpy(), s_ref)
    assert int(merges.item()) == m_ref


def test_update_accumulate_and_merges(ops, oracle):
    x = torch.randn((1, 10000, 32)).float()
    ids = torch.randint(0, 40, (1, 10000), dtype=torch.int32)
    merges = torch.zeros((), dtype=torch.int64, device="cuda")
    s1, c1 = ops.update(x[:, :6000].contiguous().cuda(), ids[:, :6000].contiguous().cuda(), 40, 1000,
                        merges=merges)
    ops.update(x[:, 6000:].contiguous().cuda(), ids[:, 6000:].contiguous().cuda(), 40, 1000,
               accumulate=True, sums=s1, counts=c1, merges=merges)
    torch.cuda.synchronize()
    s_ref, c_ref, _ = oracle.sort_inverse_update(x.numpy(), ids.numpy(), 40, 1000)
    _, _, m1 = oracle.sort_inverse_update(x[:, :6000].numpy(), ids[:, :6000].numpy(), 40, 1000)
    _, _, m2 = oracle.sort_inverse_update(x[:, 6000:].numpy(), ids[:, 6000:].numpy(), 40, 1000)
    assert np.array_equal(c1.cpu().numpy(), c_ref)
    assert np.array_equal(s1.cpu().numpy(), s_ref)
    assert int(merges.item()) == m1 + m2


def test_changed_flag(ops):
    x = torch.randn((1, 5000, 64)).to(torch.bfloat16).cuda()
    c = x[:, :100].clone()
    a, _ = ops.assign(x, c)
    flag = torch.zeros((), dtype=torch.int32, device="cuda")
    ops.assign(x, c, idx_prev=a, changed=flag)
    assert int(flag.item()) == 0
    a2 = a.clone()
    a2[0, 4999] += 1
    ops.assign(x, c, idx_prev=a2, changed=flag)
    assert int(flag.item()) == 1


@pytest.mark.parametrize("N", [1, 7, 8, 129, 1000, 8191, 8192, 8193, 20000, 100000, 1 << 20])
def test_objective_f32_is_numpys_order(ops, N):
    """pipeline._objective_row on f32 min_dists: np.sum(m, dtype=float64) casts
    through numpy's 8192-element buffer and adds each buffer's pairwise sum in
    order -- reproduced addition for addition, on data whose f64 sums are NOT
    exact (magnitudes over many binades), through both the standalone objective
    and the engine's end-of-iteration launch (fused tail or the split path)."""
    rng = np.random.default_rng(N)
    m = (rng.random((3, N)) * np.exp(rng.uniform(-18, 10, (3, N)))).astype(np.float32)
    ref = np.array([np.sum(m[b], dtype=np.float64) for b in range(3)])
    out = ops.objective(torch.from_numpy(m).cuda()).cpu().numpy()
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))
    part = torch.empty((3 * -(-N // ops.OBJ_BLOCK),), dtype=torch.float64, device="cuda")
    ops.objective_partials(torch.from_numpy(m).cuda(), part)
    for b in range(3):
        acc = 0.0
        for v in part.view(3, -1)[b].cpu().numpy():
            acc = acc + v
        assert np.float64(acc).view(np.uint64) == ref[b].view(np.uint64)


@pytest.mark.parametrize("B,N,K", [(64, 16384, 256), (1, 100000, 1024), (3, 20000, 24)])
@pytest.mark.parametrize("tail", ["fused", "split"])
def test_loop_tail_objective_is_numpys_order(B, N, K, tail):
    """The engine's end-of-iteration launch(es) write numpy's objective too, for
    both forms (FK_TAIL=fused|split; run in a child so the switch is read fresh)."""
    import subprocess
    import sys

    code = f"""
import numpy as np, torch, sys
sys.path.insert(0, {repr(str(__import__('pathlib').Path(__file__).resolve().parents[1]))})
from paper_2603_09229_b200 import ops
B, N, K, d = {B}, {N}, {K}, 8
rng = np.random.default_rng(5)
m = torch.from_numpy((rng.random((B, N)) * np.exp(rng.uniform(-18, 10, (B, N)))).astype(np.float32)).cuda()
sums = torch.zeros((B, K, d), dtype=torch.float64, device="cuda")
counts = torch.ones((B, K), dtype=torch.int64, device="cuda")
prev = torch.zeros((B, K, d), dtype=torch.float32, device="cuda")
out = torch.empty_like(prev)
empty = torch.empty((B, K), dtype=torch.uint8, device="cuda")
shift2 = torch.zeros((), dtype=torch.float64, device="cuda")
nb = max(int(ops.N.lib().fk_objective_workspace(B, N)), B * -(-N // ops.OBJ_BLOCK) * 8)
part = torch.empty((-(-nb // 8),), dtype=torch.float64, device="cuda")
obj = torch.empty((B,), dtype=torch.float64, device="cuda")
changed = torch.zeros((), dtype=torch.int32, device="cuda")
merges = torch.zeros((), dtype=torch.int64, device="cuda")
flags = torch.zeros(3, dtype=torch.float64, device="cuda")
ctr = torch.zeros((1,), dtype=torch.int32, device="cuda")
for _ in range(2):
    ops.normalize_loop_tail(sums, counts, prev, out, None, empty, shift2, None, m, part, obj, changed, merges,
                            flags, ctr)
ref = np.array([np.sum(m[b].cpu().numpy(), dtype=np.float64) for b in range(B)])
assert np.array_equal(obj.cpu().numpy().view(np.uint64), ref.view(np.uint64)), (obj.cpu().numpy() - ref)
print("ok")
"""
    env = dict(__import__("os").environ, FK_TAIL=tail)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-2000:]


# ----------------------------------------------------------- stable sort / determinism
def test_device_argsort_hand_cases():
    """The reference's counting_sort known answers (test_sort_inverse.py:26-42)."""
    import paper_2603_09229_b200 as fk

    idx, a_sorted = fk.argsort_assignments(fk.Assignments(torch.tensor([[2, 0, 1, 0]], dtype=torch.int32).cuda()), 3)
    assert idx.order[0].tolist() == [1, 3, 2, 0]
    assert a_sorted[0].tolist() == [0, 0, 1, 2]
    idx, _ = fk.argsort_assignments(fk.Assignments(torch.tensor([[1, 1, 0, 1, 0]], dtype=torch.int32).cuda()), 2)
    assert idx.order[0].tolist() == [2, 4, 0, 1, 3]


@pytest.mark.parametrize("B,N,K,skew", [
    (1, 5_000_003, 4096, False),   # several sub-tiles per block, 2 radix passes
    (64, 16384, 256, False),       # config 4: one pass, many batch elements
    (2, 300_001, 1, False),        # K = 1
    (1, 200_000, 65536, False),    # global-row histograms, 2 passes
    (1, 400_000, 70000, True),     # 3 passes, skewed: one giant run + a long tail
    (3, 9000, 300, True),
])
def test_device_argsort_is_numpy_stable_argsort(ops, B, N, K, skew):
    g = torch.Generator().manual_seed(N + K)
    if skew:  # Zipf-like: most points in a few clusters
        ids = (torch.rand((B, N), generator=g) ** 6 * K).to(torch.int32).clamp_(max=K - 1)
    else:
        ids = torch.randint(0, K, (B, N), generator=g, dtype=torch.int32)
    order, off = ops.argsort(ids.cuda(), K)
    ref = np.concatenate([np.argsort(ids[b].numpy(), kind="stable") + b * N for b in range(B)])
    assert np.array_equal(order.cpu().numpy(), ref)
    cnt = np.stack([np.bincount(ids[b].numpy(), minlength=K) for b in range(B)]).reshape(-1)
    assert np.array_equal(off.cpu().numpy(), np.concatenate([[0], np.cumsum(cnt)]))


def test_device_argsort_skips_out_of_range_ids(ops):
    ids = torch.tensor([[3, -1, 0, 7, 1, 0, 2]], dtype=torch.int32)
    order, off = ops.argsort(ids.cuda(), 4)
    assert off.cpu().tolist() == [0, 2, 3, 4, 5]
    assert order.cpu().tolist()[:5] == [2, 5, 4, 6, 0]


@pytest.mark.parametrize("B,N,K,d,dtype", [
    (1, 4_000_000, 4096, 128, torch.bfloat16),
    (64, 16384, 256, 64, torch.float16),
    (1, 1 << 20, 1024, 128, torch.float64),
    (2, 700_001, 3001, 32, torch.float32),
    (1, 300_000, 20000, 16, torch.bfloat16),
])
def test_update_is_deterministic(ops, B, N, K, d, dtype):
    """Two updates of the same (X, ids) give the same bits -- sums included,
    for every dtype (stable order + slice-ordered boundary merges; no float
    atomics anywhere on the path)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    x = (torch.randn((B, N, d), device="cuda", generator=g) * 4 + 1).to(dtype)
    ids = torch.randint(0, K, (B, N), device="cuda", generator=g, dtype=torch.int32)
    s1, c1 = ops.update(x, ids, K, N)
    s1 = s1.clone()
    c1 = c1.clone()
    junk = torch.randint(0, K, (B, N), device="cuda", generator=g, dtype=torch.int32)
    ops.update(x, junk, K, N)  # reuse the workspace with other data in between
    s2, c2 = ops.update(x, ids, K, N)
    assert torch.equal(c1, c2)
    assert torch.equal(s1.view(torch.int64), s2.view(torch.int64))


@pytest.mark.parametrize("K", [1, 2, 3, 37, 4096])
def test_device_argsort_stable_under_heavy_collisions(ops, K):
    """Many lanes of a warp step share an id: the ranks must still follow the
    point index (the stable order), on every repetition."""
    g = torch.Generator().manual_seed(K)
    ids = torch.randint(0, K, (2, 600_000), generator=g, dtype=torch.int32)
    ids[:, 1000:40000] = 0  # long single-id stretches
    ref = np.concatenate([np.argsort(ids[b].numpy(), kind="stable") + b * ids.shape[1] for b in range(2)])
    idc = ids.cuda()
    for _ in range(10):
        order, _ = ops.argsort(idc, K)
        assert np.array_equal(order.cpu().numpy(), ref)


@pytest.mark.parametrize("dtype,K,d", [(torch.bfloat16, 300, 128), (torch.float16, 256, 64),
                                       (torch.bfloat16, 4096, 128), (torch.bfloat16, 77, 200)])
def test_normalize_bias_operand_is_assign_bias(ops, dtype, K, d):
    """normalize(bias_out=) writes, bit for bit, the bias operand fk_assign would
    compute from the rounded centroids, and assign gives the same ids with it."""
    g = torch.Generator(device="cuda").manual_seed(K + d)
    B = 2
    sums = torch.randn((B, K, d), device="cuda", generator=g, dtype=torch.float64) * 50
    counts = torch.randint(0, 9, (B, K), device="cuda", generator=g, dtype=torch.int64)
    prev = torch.randn((B, K, d), device="cuda", generator=g)
    kpad = ops.N.lib().fk_assign_bias_rows(K)
    bias = torch.zeros((B, kpad, 16), dtype=torch.bfloat16, device="cuda")
    ops.assign_bias(prev.to(dtype), out=bias)  # padding rows
    out, operand, _ = ops.normalize(sums, counts, prev, operand_dtype=dtype, bias_out=bias)
    ref = ops.assign_bias(operand)
    assert torch.equal(bias.view(torch.int16), ref.view(torch.int16))
    x = (torch.randn((B, 5000, d), device="cuda", generator=g) * 3).to(dtype)
    a0, m0 = ops.assign(x, operand)
    a1, m1 = ops.assign(x, operand, bias=bias)
    assert torch.equal(a0, a1) and torch.equal(m0, m1)


@pytest.mark.parametrize("n,E,dtype,ties", [(1000, 1, torch.float32, False), (5_000_000, 37, torch.float32, True),
                                             (300_001, 4096, torch.float64, True), (9, 9, torch.float32, True),
                                             (2_000_000, 8192, torch.float32, False)])
def test_device_farthest_is_reference_order(ops, n, E, dtype, ties):
    """fk_farthest == np.lexsort((arange, -mind))[:E] (pipeline.py:76-81), ties included."""
    g = torch.Generator().manual_seed(n + E)
    m = torch.rand((2, n), generator=g, dtype=torch.float64) * 100
    if ties:  # many exact duplicates, including among the winners
        m = torch.round(m * 4) / 4
    m = m.to(dtype)
    got = ops.farthest(m.cuda(), E).cpu().numpy()
    for b in range(2):
        v = m[b].double().numpy()
        ref = np.lexsort((np.arange(n), -v))[:E]
        assert np.array_equal(got[b], ref)


# ----------------------------------------------------------- histogram fold
@pytest.mark.parametrize("B,N,K,d,dtype", [
    (1, 100_000, 1024, 128, torch.bfloat16),   # bpb > 16: k_colscan reads the folded table
    (64, 16384, 256, 64, torch.float16),       # config 4's shape
    (3, 20_001, 37, 32, torch.bfloat16),       # ragged N, odd K
    (2, 50_000, 3000, 64, torch.float16),      # K beyond the shared-memory bins
    (1, 3000, 9000, 16, torch.bfloat16),       # more keys than points per block
])
def test_hist_fold_equals_assign_then_update(ops, B, N, K, d, dtype):
    """fk_assign_hist + fk_update_prehist == fk_assign + fk_update bit for bit
    (ids, min_dists, sums, counts, merges), and the table is left zeroed for
    the next assign (checked by running the pair twice)."""
    g = torch.Generator(device="cuda").manual_seed(N + K)
    x = (torch.randn((B, N, d), device="cuda", generator=g) * 3).to(dtype)
    c = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].contiguous()
    ids_r, m_r = ops.assign(x, c)
    mg_r = torch.zeros((), dtype=torch.int64, device="cuda")
    s_r, n_r = ops.update(x, ids_r, K, 4096, merges=mg_r)
    s_r, n_r = s_r.clone(), n_r.clone()
    fold = ops.hist_fold(x, K)
    assert fold is not None
    for rep in range(2):
        ids, m = ops.assign(x, c, hist=fold)
        mg = torch.zeros((), dtype=torch.int64, device="cuda")
        s, n = ops.update(x, ids, K, 4096, merges=mg, hist=fold)
        assert torch.equal(ids, ids_r) and torch.equal(m, m_r)
        assert torch.equal(n, n_r)
        assert torch.equal(s.view(torch.int64), s_r.view(torch.int64))
        assert int(mg) == int(mg_r)
        assert int(fold._clear.count_nonzero()) == 0


def test_hist_fold_offered_where_supported(ops):
    x = torch.zeros((1, 1000, 32), dtype=torch.bfloat16, device="cuda")
    assert ops.hist_fold(x, 16) is not None
    assert ops.hist_fold(x.float(), 16) is None       # f32 data: the certified path, no fold
    assert ops.hist_fold(x, 20_000) is None           # K beyond the warp-table scatter
    x20 = torch.zeros((1, 1000, 20), dtype=torch.bfloat16, device="cuda")
    assert ops.hist_fold(x20, 16) is None             # d = 20: the CUDA-core assign, nothing to fold into


def test_engine_without_tensor_core_path_runs(ops):
    """bf16 with d = 20 (rows not 16-byte multiples): no fold, no precomputed
    norms; the pipelined run still equals the stepwise loop."""
    from paper_2603_09229_b200 import LloydEngine

    g = torch.Generator(device="cuda").manual_seed(4)
    x = (torch.randn((2, 3000, 20), device="cuda", generator=g) * 3).to(torch.bfloat16)
    eng = LloydEngine(x, 12)
    assert eng._fold is None and eng._xn is None
    eng.set_centroids(x[:, :12].float())
    ref = LloydEngine(x, 12)
    ref.set_centroids(x[:, :12].float())
    its, slot, _ = eng.run(3, -1.0, stop_on_repeat=False)
    for _ in range(3):
        sb = ref.iterate()
        ref.poll()
        ref.commit()
    assert torch.equal(eng.centroids, ref.centroids) and torch.equal(eng.ids[slot], ref.ids[sb])


@pytest.mark.parametrize("B,N,K,d,dtype", [
    (2, 5000, 200, 64, torch.float16),     # one column tile: the alternating epilogue
    (3, 7001, 256, 96, torch.bfloat16),
    (1, 20000, 1024, 128, torch.bfloat16),  # column halves merged across warpgroups
    (2, 3000, 300, 200, torch.float16),     # 4 atoms, zero-filled tail
    (4, 999, 64, 8, torch.bfloat16),
])
def test_precomputed_row_norms_keep_min_dists_bitwise(ops, B, N, K, d, dtype):
    """fk_assign_row_norms sums ||x||^2 exactly as the tensor-core epilogue does
    from its swizzled shared tile, so fk_assign_hist with xnorm returns the same
    ids and min_dists bit for bit as the epilogue's own sum."""
    g = torch.Generator(device="cuda").manual_seed(N + d)
    x = (torch.randn((B, N, d), device="cuda", generator=g) * 2).to(dtype)
    c = x[:, torch.randperm(N, device="cuda", generator=g)[:K]].contiguous()
    ids_r, m_r = ops.assign(x, c)
    xn = ops.assign_row_norms(x, K)
    assert xn is not None and xn.shape == (B, N)
    fold = ops.hist_fold(x, K)
    ids, m = ops.assign(x, c, hist=fold, xnorm=xn)
    ops.update(x, ids, K, N, hist=fold)  # consume the table
    assert torch.equal(ids, ids_r)
    assert torch.equal(m.view(torch.int32), m_r.view(torch.int32))


def test_hist_fold_counts_invalid_rows(ops):
    """Rows whose scores are all NaN get id -1 from the tensor-core assign; the
    folded histogram counts them as invalid (hist_inval) exactly as k_hist
    does, so the update skips them identically (offsets, sums, counts)."""
    g = torch.Generator(device="cuda").manual_seed(3)
    B, N, K, d = 2, 40000, 300, 64
    x = torch.randn((B, N, d), device="cuda", generator=g).to(torch.bfloat16)
    c = x[:, :K].clone()
    x[0, 5:900:7] = float("nan")
    x[1, -300:] = float("nan")
    ids_r, m_r = ops.assign(x, c)
    assert int((ids_r < 0).sum()) > 0
    s_r, n_r = ops.update(x, ids_r, K, 4096)
    s_r, n_r = s_r.clone(), n_r.clone()
    fold = ops.hist_fold(x, K)
    ids, m = ops.assign(x, c, hist=fold)
    s, n = ops.update(x, ids, K, 4096, hist=fold)
    assert torch.equal(ids, ids_r)
    assert torch.equal(n, n_r)
    assert torch.equal(s.view(torch.int64), s_r.view(torch.int64))
    assert int(fold._clear.count_nonzero()) == 0


_PDL_SNIPPET = r"""
import hashlib, sys, torch
sys.path.insert(0, '.')
from paper_2603_09229_b200 import LloydEngine, ops
out = []
for (B, N, K, d, dt) in [(64, 16384, 256, 64, torch.float16), (1, 1 << 20, 1024, 128, torch.bfloat16)]:
    g = torch.Generator(device='cuda').manual_seed(5)
    x = (torch.randn((B, N, d), device='cuda', generator=g) * 4).to(dt)
    ids = torch.randint(0, K, (B, N), device='cuda', generator=g, dtype=torch.int32)
    s, c = ops.update(x, ids, K, N)
    eng = LloydEngine(x, K)
    eng.set_centroids(x[:, :K].float())
    h = torch.empty((8, B), dtype=torch.float64, device='cuda')
    eng.run(3, -1.0, h, stop_on_repeat=False)
    torch.cuda.synchronize()
    for t in (s.view(torch.int64), c, eng.master[eng.cur], h[:3]):
        out.append(hashlib.sha1(t.contiguous().cpu().numpy().tobytes()).hexdigest())
print(' '.join(out))
"""


def test_update_chain_pdl_matches_ordinary_launches():
    """Programmatic dependent launch along scatter -> segsum -> normalize/loop
    tail (the default) gives the same bits as ordinary launches (FK_PDL=0):
    update sums and counts, and three engine iterations (centroids and
    objective history). Each setting runs in its own process (the switch is
    read once)."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    res = []
    for v in ("1", "0"):
        r = subprocess.run([sys.executable, "-c", _PDL_SNIPPET], cwd=root, env=dict(os.environ, FK_PDL=v),
                           capture_output=True, text=True, timeout=600)
        assert r.returncode == 0, r.stderr[-2000:]
        res.append(r.stdout.strip().splitlines()[-1])
    assert res[0] == res[1]
