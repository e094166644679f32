"""Parity of the CUDA path (through the C ABI) with the reference.

Every test calls libsemidist_b200.so; the comparison target is the golden
vectors produced by the reference itself and, for sizes the fixtures do not
hold, the oracle (oracle/semidist_oracle.py, pinned bitwise to the reference
by tests/test_oracle_golden.py).  Tolerance rule: tests/parity.py.
"""

import numpy as np
import pytest

import paper_2104_06357_b200 as sd
from golden_cases import csr
from oracle import semidist_oracle as O
from parity import assert_knn_parity, assert_parity

pytestmark = pytest.mark.gpu

DTYPES = [np.float64, np.float32]


def _strategy(s):
    if isinstance(s, list):
        return sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=s[1], max_load_factor=s[2])
    return s


def _f32(m):
    return m.with_values(np.asarray(m.values, dtype=np.float32).astype(np.float64))


def _host(m):
    return sd.CsrMatrix(m.n_rows, m.n_cols, m.indptr, m.indices, m.values)


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    from paper_2104_06357_b200 import _lib
    _lib.load()


# ------------------------------------------------------------ golden vectors

@pytest.mark.parametrize("dtype", DTYPES)
def test_golden_pairwise_fused_and_engine(golden, dtype):
    """All 15 metrics x {auto (fused), dense, hash(8/16), naive} vs the reference's outputs."""
    cases, arrays = golden
    n = 0
    for c in cases:
        if c["kind"] != "pairwise":
            continue
        a, b = _host(csr(arrays, c["a"])), _host(csr(arrays, c["b"]))
        if dtype == np.float32 and not (np.asarray(a.values, np.float32) == a.values).all():
            a, b = _f32(a), _f32(b)
            ref = O.pairwise_distances(a, b, c["metric"], p=c["p"], strict=c["strict"])
        else:
            ref = arrays[c["id"] + ".out"]
        spec = sd.metric_registry(c["metric"], p=c["p"], strict=c["strict"])
        got, rep, _ = sd.pairwise_distances_detail(a, b, spec, _strategy(c["strategy"]), dtype=dtype)
        assert got.dtype == np.float64 and got.flags["C_CONTIGUOUS"]
        assert_parity(got, ref, a, b, c["metric"], dtype, p=c["p"], what=c["id"])
        assert [rep.peak_accumulator_entries, rep.workspace_elements, rep.chunks_executed] == c["report"], c["id"]
        n += 1
    assert n > 100


@pytest.mark.parametrize("strategy", [None, "dense", "hash", "naive"])
def test_golden_pairwise_all_strategies_fp64(golden, strategy):
    cases, arrays = golden
    for c in cases:
        if c["kind"] != "pairwise" or c["id"].startswith("zipf"):
            continue
        a, b = _host(csr(arrays, c["a"])), _host(csr(arrays, c["b"]))
        spec = sd.metric_registry(c["metric"], p=c["p"], strict=c["strict"])
        got = sd.pairwise_distances(a, b, spec, strategy)
        assert_parity(got, arrays[c["id"] + ".out"], a, b, c["metric"], np.float64, p=c["p"],
                      what=f"{c['id']}/{strategy}")


@pytest.mark.parametrize("dtype", DTYPES)
def test_golden_generalized(golden, dtype):
    cases, arrays = golden
    rings = {"dot": sd.dot_product(), "abs-diff": sd.absolute_difference(),
             "abs-diff-max": sd.max_absolute_difference(), "canberra-ratio": sd.canberra_ratio(),
             "mismatch": sd.mismatch_indicator(), "jensen-shannon-term": sd.jensen_shannon_term(),
             "min-plus": sd.tropical_min_plus(), "abs-diff-pow": sd.absolute_difference_power(1.5)}
    for c in cases:
        if c["kind"] != "generalized":
            continue
        a, b = _host(csr(arrays, c["a"])), _host(csr(arrays, c["b"]))
        ref = arrays[c["id"] + ".out"]
        if dtype == np.float32:
            a, b = _f32(a), _f32(b)
            ref = O.generalized(a, b, c["ring"], p=1.5 if c["ring"] == "abs-diff-pow" else None)
        for strat in (None, "naive", sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, 8)):
            got, _ = sd.pairwise_generalized(a, b, rings[c["ring"]], strat, dtype=dtype)
            if c["ring"] in ("min-plus", "abs-diff-max") and dtype == np.float64:
                np.testing.assert_array_equal(got, ref, err_msg=c["id"])   # exact semirings
            else:
                rtol = 1e-12 if dtype == np.float64 else 1e-5
                np.testing.assert_allclose(got, ref, rtol=rtol, atol=rtol * 30, err_msg=c["id"])


def test_appendix_golden_exact():
    a = sd.from_dense([[1.0, 0.0, 1.0]])
    b = sd.from_dense([[0.0, 1.0, 0.0]])
    spec = sd.metric_registry("manhattan")
    for strategy in (None, "dense", "naive"):
        assert sd.pairwise_distances(a, b, spec, strategy)[0, 0] == 3.0
    out = sd.allocate_output(a, b, spec.semiring)
    sd.pairwise_spmv_pass1(a, b, spec.semiring, sd.ExecutionStrategy(sd.StrategyKind.BALANCED_DENSE), out)
    assert out[0, 0] == 1.0
    sd.pairwise_spmv_pass2(a, b, spec.semiring, sd.ExecutionStrategy(sd.StrategyKind.BALANCED_DENSE), out)
    assert out[0, 0] == 3.0


@pytest.mark.parametrize("dtype", DTYPES)
def test_golden_knn(golden, dtype):
    cases, arrays = golden
    for c in cases:
        if c["kind"] != "knn":
            continue
        q, ix = _host(csr(arrays, c["a"])), _host(csr(arrays, c["b"]))
        spec = sd.metric_registry(c["metric"])
        res = sd.kneighbors(ix, q, c["k"], spec, dtype=dtype)
        full = O.pairwise_distances(q, ix, c["metric"])
        tol = 1e-12 if dtype == np.float64 else 1e-5
        assert_knn_parity(res.distances, res.indices, arrays[c["id"] + ".dist"], arrays[c["id"] + ".idx"],
                          full, tol=tol * 10)
        if dtype == np.float64:   # forced engine strategy + sd_topk_rows route
            res2 = sd.kneighbors(ix, q, c["k"], spec, strategy="dense", batch_rows=7)
            assert_knn_parity(res2.distances, res2.indices, arrays[c["id"] + ".dist"],
                              arrays[c["id"] + ".idx"], full, tol=tol * 10)


# ------------------------------------------------------------ reference test strategy, on GPU

def test_self_distance_exact_zero():
    """Norm and dot accumulate in the same order: euclidean/cosine self-distance is exactly 0
    (as in the reference, metrics.py:106-118)."""
    x = _host(sd.generate(sd.GenSpec(300, 5000, "zipf", zipf_s=1.3, zipf_max_degree=400, seed=4)))
    for dtype in DTYPES:
        for name in ("euclidean", "manhattan", "canberra", "hamming", "chebyshev", "jensenshannon"):
            d = sd.pairwise_distances(x, x, sd.metric_registry(name), dtype=dtype)
            if name in ("euclidean", "chebyshev", "hamming"):
                assert np.all(np.diag(d) == 0.0), (name, dtype)
            else:
                assert np.abs(np.diag(d)).max() <= (1e-9 if dtype == np.float64 else 1e-3), (name, dtype)


def test_kl_strict_and_permissive():
    a = sd.from_dense([[0.5, 0.5]])
    b = sd.from_dense([[1.0, 0.0]])
    with pytest.raises(sd.DomainError):
        sd.pairwise_distances(a, b, sd.metric_registry("kl"))
    assert sd.pairwise_distances(a, b, sd.metric_registry("kl", strict=False))[0, 0] == 1e308
    with pytest.raises(sd.DomainError):
        sd.pairwise_distances(a, b, sd.metric_registry("kl"), "dense")
    d32 = sd.pairwise_distances(a, b, sd.metric_registry("kl", strict=False), dtype=np.float32)
    assert np.isinf(d32[0, 0])


def test_domain_errors():
    neg = sd.from_dense([[-1.0, 0.5]])
    pos = sd.from_dense([[1.0, 0.5]])
    for name in ("kl", "jensenshannon", "hellinger"):
        with pytest.raises(sd.DomainError):
            sd.pairwise_distances(neg, pos, sd.metric_registry(name))
        with pytest.raises(sd.DomainError):
            sd.pairwise_distances(pos, neg, sd.metric_registry(name))
    with pytest.raises(sd.DimensionMismatch):
        sd.pairwise_distances(sd.from_dense([[1.0, 0.0]]), sd.from_dense([[1.0, 0, 0]]), sd.metric_registry("cosine"))


def test_expansion_apply_hand_cases():
    spec = sd.metric_registry("euclidean")
    na = [sd.NormVector(sd.NormKind.L2_SQUARED, np.array([2.0]))]
    nb = [sd.NormVector(sd.NormKind.L2_SQUARED, np.array([1.0]))]
    np.testing.assert_allclose(sd.expansion_apply(np.array([[1.0]]), na, nb, spec, n_cols=2), [[1.0]])
    norms = [sd.NormVector(sd.NormKind.L2_SQUARED, np.array([1.0]))]
    with pytest.raises(sd.DomainError):
        sd.expansion_apply(np.array([[10.0]]), norms, norms, spec, n_cols=2)
    np.testing.assert_array_equal(
        sd.expansion_apply(np.array([[1.0 + 2e-10]]), norms, norms, spec, n_cols=2), [[0.0]])
    jn = [sd.NormVector(sd.NormKind.L0, np.array([3.0]))]
    np.testing.assert_allclose(sd.expansion_apply(np.array([[3.0]]), jn, jn, sd.metric_registry("jaccard"),
                                                  n_cols=8), [[0.0]])


def test_determinism_bitwise():
    x = _host(sd.generate(sd.GenSpec(200, 3000, "zipf", zipf_s=1.3, zipf_max_degree=500, seed=9)))
    for name, strat in [("cosine", None), ("manhattan", None), ("canberra", "dense"), ("chebyshev", None),
                        ("manhattan", sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, 16))]:
        d1 = sd.pairwise_distances(x, x, sd.metric_registry(name), strat, dtype=np.float32)
        d2 = sd.pairwise_distances(x, x, sd.metric_registry(name), strat, dtype=np.float32)
        np.testing.assert_array_equal(d1, d2)


def test_knn_batching_invariance_and_ties():
    x = _host(sd.generate(sd.GenSpec(400, 300, "zipf", zipf_s=1.1, zipf_max_degree=150, seed=8)))
    spec = sd.metric_registry("cosine")
    base = sd.kneighbors(x, x, 10, spec, batch_rows=400)
    for rows in (1, 64, 117):
        r = sd.kneighbors(x, x, 10, spec, batch_rows=rows)
        np.testing.assert_array_equal(r.indices, base.indices)
        np.testing.assert_array_equal(r.distances, base.distances)
    ref_d, ref_i = O.kneighbors(x, x, 10, "cosine")
    full = O.pairwise_distances(x, x, "cosine")
    assert_knn_parity(base.distances, base.indices, ref_d, ref_i, full, tol=1e-11)
    with pytest.raises(sd.KTooLarge):
        sd.kneighbors(x, x, 401, spec)
    vals, idx = sd.select_topk([1.0, 1.0, 1.0], 2)
    assert idx.tolist() == [0, 1]
    vals, idx = sd.select_topk([3.0, 1.0, 2.0], 2)
    assert idx.tolist() == [1, 2] and vals.tolist() == [1.0, 2.0]


def test_knn_large_k_and_chebyshev_routes():
    x = _host(sd.generate(sd.GenSpec(300, 200, "zipf", zipf_s=1.3, zipf_max_degree=60, seed=18)))
    for name, k in (("cosine", 150), ("chebyshev", 12), ("manhattan", 64)):
        res = sd.kneighbors(x, sd.slice_rows(x, 0, 40), k, sd.metric_registry(name))
        ref_d, ref_i = O.kneighbors(x, O.Csr.of(x).slice(0, 40), k, name)
        full = O.pairwise_distances(O.Csr.of(x).slice(0, 40), x, name)
        assert_knn_parity(res.distances, res.indices, ref_d, ref_i, full, tol=1e-11)


def test_hash_chunking_forced_and_reported():
    """Degrees above 50% of a tiny capacity force column chunking (test_engine.py:294-303)."""
    rng = np.random.default_rng(12)
    a = sd.from_dense(np.where(rng.random((20, 60)) < 0.5, rng.uniform(0.1, 1, (20, 60)), 0.0))
    b = sd.from_dense(np.where(rng.random((10, 60)) < 0.3, rng.uniform(0.1, 1, (10, 60)), 0.0))
    strat = sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=16, max_load_factor=0.5)
    for ring in (sd.absolute_difference(), sd.max_absolute_difference(), sd.tropical_min_plus()):
        out, rep = sd.pairwise_generalized(a, b, ring, strat)
        assert rep.peak_accumulator_entries <= 8 and rep.chunks_executed > a.n_rows
        base = O.generalized(a, b, ring.name)
        np.testing.assert_allclose(out, base, rtol=1e-12, atol=1e-12)


def test_empty_and_degenerate_shapes():
    spec = sd.metric_registry("manhattan")
    z = sd.validate_and_canonicalize([0], [], [], n_cols=5)
    x = sd.from_dense([[0.0, 1.0, 0, 0, 2.0]])
    assert sd.pairwise_distances(z, x, spec).shape == (0, 1)
    assert sd.pairwise_distances(x, z, spec).shape == (1, 0)
    e = sd.validate_and_canonicalize([0, 0, 0], [], [], n_cols=5)
    for name in sd.METRIC_NAMES:
        p = 2.0 if name == "minkowski" else None
        d = sd.pairwise_distances(e, x, sd.metric_registry(name, p=p, strict=False))
        ref = O.pairwise_distances(e, x, name, p=p, strict=False)
        np.testing.assert_allclose(d, ref, rtol=1e-12, atol=1e-12, err_msg=name)


# ------------------------------------------------------------ full-size configs

@pytest.mark.parametrize("dtype", DTYPES)
def test_config1_full_vs_oracle(dtype):
    """BASELINE config 1 at full size (1k x 1k, 10k cols, 1% density), manhattan + cosine."""
    A = _f32(sd.generate(sd.GenSpec(1000, 10000, "uniform", degree=100, seed=1)))
    B = _f32(sd.generate(sd.GenSpec(1000, 10000, "uniform", degree=100, seed=2)))
    for name in ("manhattan", "cosine"):
        ref = O.pairwise_distances(A, B, name)
        for strategy in (None, "dense"):
            got = sd.pairwise_distances(A, B, sd.metric_registry(name), strategy, dtype=dtype)
            assert_parity(got, ref, A, B, name, dtype, what=f"C1/{name}/{strategy}")


def test_power_law_properties_at_scale():
    """MovieLens-shaped (config 2) index: size-independent properties on a full-size
    index — self-distance, symmetry of the self block, expanded vs two-pass euclidean,
    and oracle parity on a sampled block."""
    idx = _f32(sd.generate(sd.GenSpec(162541, 59047, "zipf", zipf_s=1.5, zipf_max_degree=32000, seed=25)))
    rng = np.random.default_rng(26)
    rows = np.sort(rng.choice(idx.n_rows, 64, replace=False))
    q = _gather_rows(idx, rows)
    d = sd.pairwise_distances(q, idx, sd.metric_registry("cosine"), dtype=np.float32)
    assert d.shape == (64, idx.n_rows)
    np.testing.assert_allclose(d[np.arange(64), rows], 0.0, atol=1e-5)  # fp32 parity tolerance
    cols = np.sort(rng.choice(idx.n_rows, 2000, replace=False))
    sub = _gather_rows(idx, cols)
    ref = O.pairwise_distances(q, sub, "cosine")
    assert_parity(d[:, cols], ref, q, sub, "cosine", np.float32, what="C2 sample")
    e = sd.pairwise_distances(q, sub, sd.metric_registry("euclidean"), dtype=np.float64)
    m2 = sd.pairwise_distances(q, sub, sd.metric_registry("minkowski", p=2.0), dtype=np.float64)
    np.testing.assert_allclose(e, m2, rtol=1e-9, atol=1e-9)


def _gather_rows(m, rows):
    ptr = np.asarray(m.indptr)
    parts_i, parts_v, newptr = [], [], [0]
    for r in rows:
        lo, hi = ptr[r], ptr[r + 1]
        parts_i.append(np.asarray(m.indices[lo:hi]))
        parts_v.append(np.asarray(m.values[lo:hi]))
        newptr.append(newptr[-1] + hi - lo)
    return sd.CsrMatrix(len(rows), m.n_cols, np.asarray(newptr, dtype=np.int64),
                        np.concatenate(parts_i), np.concatenate(parts_v))


def test_sharded_knn_emulated_on_one_gpu():
    """B sharded into 3 ranges processed one after another on the same GPU,
    merged with sd_topk_merge: equals the single-shard kNN (NCCL
    cannot place two ranks on one GPU, so shards are emulated)."""
    import torch
    from paper_2104_06357_b200.distributed import local_topk_padded, merge_candidates, shard_bounds
    x = _host(sd.generate(sd.GenSpec(500, 400, "zipf", zipf_s=1.2, zipf_max_degree=120, seed=31)))
    q = sd.slice_rows(x, 0, 60)
    spec = sd.metric_registry("cosine")
    for k in (7, 40):
        ds, is_ = [], []
        for lo, hi in shard_bounds(x.n_rows, 3):
            d, i = local_topk_padded(sd.slice_rows(x, lo, hi), q, k, spec, index_base=lo, dtype=np.float64)
            ds.append(d)
            is_.append(i)
        md, mi = merge_candidates(torch.stack(ds), torch.stack(is_), k)
        base = sd.kneighbors(x, q, k, spec)
        np.testing.assert_array_equal(mi.cpu().numpy(), base.indices)
        np.testing.assert_array_equal(md.cpu().numpy(), base.distances)


@pytest.mark.parametrize("dtype", DTYPES)
def test_fused_chebyshev_matches_engine_and_oracle(dtype):
    """Fused chebyshev (max over intersections + top-16 hit masks, exact merge
    when a row's top-16 all intersect) against the oracle, incl. rows dense
    enough to force the exact fallback."""
    rng = np.random.default_rng(41)
    for dens in (0.05, 0.3, 0.9):
        da = np.where(rng.random((40, 64)) < dens, rng.uniform(-1, 1, (40, 64)), 0.0)
        db = np.where(rng.random((70, 64)) < dens, rng.uniform(-1, 1, (70, 64)), 0.0)
        db[:5] = da[:5]                      # identical rows: every entry intersects
        a, b = _f32(sd.from_dense(da)), _f32(sd.from_dense(db))
        ref = O.pairwise_distances(a, b, "chebyshev")
        got = sd.pairwise_distances(a, b, sd.metric_registry("chebyshev"), dtype=dtype)
        if dtype == np.float64:
            np.testing.assert_array_equal(got, ref)
        else:
            np.testing.assert_allclose(got, ref, rtol=1e-6, atol=1e-7)
        eng = sd.pairwise_distances(a, b, sd.metric_registry("chebyshev"), "dense", dtype=dtype)
        np.testing.assert_array_equal(got, eng)
        res = sd.kneighbors(b, a, 5, sd.metric_registry("chebyshev"), dtype=dtype)
        ref_d, ref_i = O.kneighbors(b, a, 5, "chebyshev")
        assert_knn_parity(res.distances, res.indices, ref_d, ref_i, ref, tol=1e-6)


@pytest.mark.parametrize("dtype", DTYPES)
def test_tile_bands_partial_and_invariant(dtype):
    """Multi-tile index swept in bands of tiles (knob isect_band): a last, partial
    band (empty tile ranges for some items) and every band size give bitwise
    the same distances and neighbours, matching the oracle on a sample."""
    idx = _f32(sd.generate(sd.GenSpec(9500, 3000, "zipf", zipf_s=1.4, zipf_max_degree=900, seed=51)))
    q = _f32(sd.generate(sd.GenSpec(150, 3000, "zipf", zipf_s=1.4, zipf_max_degree=900, seed=52)))
    spec = sd.metric_registry("cosine")
    outs, knns = [], []
    from paper_2104_06357_b200 import _lib
    for band in (1, 2, 3, 1000):
        with _lib.tuned(isect_band=band):
            outs.append(sd.pairwise_distances(q, idx, spec, dtype=dtype))
            knns.append(sd.kneighbors(idx, q, 9, spec, dtype=dtype))
    for o, r in zip(outs[1:], knns[1:]):
        np.testing.assert_array_equal(o, outs[0])
        np.testing.assert_array_equal(r.indices, knns[0].indices)
        np.testing.assert_array_equal(r.distances, knns[0].distances)
    cols = np.arange(0, idx.n_rows, 7)
    sub = _gather_rows(idx, cols)
    ref = O.pairwise_distances(q, sub, "cosine")
    assert_parity(outs[0][:, cols], ref, q, sub, "cosine", dtype, what="bands sample")


DOT_FAMILY = ("cosine", "euclidean", "correlation", "dot", "dice", "jaccard", "hellinger", "russelrao")


@pytest.mark.parametrize("dtype", DTYPES)
def test_hybrid_heavy_rows_vs_oracle(dtype):
    """Hybrid path (hybrid.cu): query rows with >= max(64, n_cols/32) nonzeros are
    computed densely (GEMM against the index's heavy rows + gather over its
    light rows) and the sweep skips them.  Every dot-family metric against the
    oracle, and against the sweep-only path (knob hybrid=0) within rounding."""
    import torch
    from paper_2104_06357_b200 import _lib
    idx = _f32(sd.generate(sd.GenSpec(2600, 1600, "zipf", zipf_s=1.15, zipf_max_degree=900, seed=61)))
    deg = np.diff(np.asarray(idx.indptr))
    heavy = np.flatnonzero(deg >= max(64, -(-idx.n_cols // 32)))
    assert len(heavy) >= 64
    rows = np.sort(np.concatenate([heavy[:40], np.arange(0, idx.n_rows, 37)]))
    q = _gather_rows(idx, np.unique(rows))
    with _lib.tuned(hybrid=2, dense=0):   # (dense=0: this index is dense enough for the dense-index mode)
        hidx = _host(idx)
        ix = _lib.device_index(sd.to_device(hidx, dtype))
        assert ix.heavy_rows == 0   # the heavy block is built by the first dot-family call
        sd.pairwise_distances(_host(q), hidx, sd.metric_registry("cosine"), dtype=dtype)
        assert ix.heavy_rows == len(heavy)
        for name in DOT_FAMILY:
            a, b = (q, idx) if name not in ("dice", "jaccard", "russelrao") else (
                q.with_values(np.ones(q.nnz)), idx.with_values(np.ones(idx.nnz)))
            a, b = _host(a), _host(b)
            spec = sd.metric_registry(name)
            got = sd.pairwise_distances(a, b, spec, dtype=dtype)
            ref = O.pairwise_distances(a, b, name)
            assert_parity(got, ref, a, b, name, dtype, what=f"hybrid/{name}")
            with _lib.tuned(hybrid=0):
                sweep = sd.pairwise_distances(_host(a), _host(b), spec, dtype=dtype)
            assert_parity(got, sweep, a, b, name, dtype, what=f"hybrid vs sweep/{name}")
    torch.cuda.synchronize()


@pytest.mark.parametrize("n_heavy_q", [40, 300])
@pytest.mark.parametrize("dtype", DTYPES)
def test_hybrid_minsum_manhattan(dtype, n_heavy_q):
    """Manhattan's dense heavy block (hminsum.cu): with no negative index
    value, |a-b| - |a| - |b| = -2 min(max(a,0), b), so heavy query rows are
    summed densely (min-sum block over the index's heavy rows, min-gather over
    its light rows).  Against the oracle and the sweep-only path; queries with
    negative values take the max(a, 0) image; an index with a negative value
    keeps the sweep (no min-sum block)."""
    from paper_2104_06357_b200 import _lib
    idx = _f32(sd.generate(sd.GenSpec(2600, 1600, "zipf", zipf_s=1.15, zipf_max_degree=900, seed=61)))
    deg = np.diff(np.asarray(idx.indptr))
    heavy = np.flatnonzero(deg >= max(64, -(-idx.n_cols // 32)))
    assert len(heavy) >= 64
    rows = np.unique(np.concatenate([heavy[:n_heavy_q], np.arange(0, idx.n_rows, 37)]))
    q = _gather_rows(idx, rows)
    rng = np.random.default_rng(5)
    signed = q.with_values(np.asarray(q.values) * np.where(rng.random(q.nnz) < 0.3, -1.0, 1.0))
    spec = sd.metric_registry("manhattan")
    with _lib.tuned(hybrid=2):
        hidx = _host(idx)
        ix = _lib.device_index(sd.to_device(hidx, dtype))
        for a in (q, signed):
            a = _host(a)
            got = sd.pairwise_distances(a, hidx, spec, dtype=dtype)
            assert "minsum" in ix.hybrid_blocks
            ref = O.pairwise_distances(a, idx, "manhattan")
            assert_parity(got, ref, a, idx, "manhattan", dtype, what=f"minsum {n_heavy_q}")
            with _lib.tuned(hybrid=0):
                sweep = sd.pairwise_distances(_host(a), _host(idx), spec, dtype=dtype)
            assert_parity(got, sweep, a, idx, "manhattan", dtype, what="minsum vs sweep")
        # self-distances of the sampled rows: the reference gives exactly 0
        got = sd.pairwise_distances(_host(q), hidx, spec, dtype=dtype)
        assert np.all(np.abs(got[np.arange(len(rows)), rows]) <= (1e-12 if dtype == np.float64 else 1e-5) *
                      2 * np.add.reduceat(np.abs(np.asarray(q.values)), np.asarray(q.indptr)[:-1]))
        # an index with a negative value: no min-sum block, the sweep answers
        neg = _host(idx.with_values(np.asarray(idx.values) * np.where(np.arange(idx.nnz) == 7, -1.0, 1.0)))
        nix = _lib.device_index(sd.to_device(neg, dtype))
        got = sd.pairwise_distances(_host(q), neg, spec, dtype=dtype)
        assert "minsum" not in nix.hybrid_blocks
        assert_parity(got, O.pairwise_distances(q, neg, "manhattan"), q, neg, "manhattan", dtype, what="neg index")


@pytest.mark.parametrize("k", [7, 40])
def test_hybrid_knn_heavy_queries(k):
    """kNN with heavy query rows on the hybrid path: their dense rows (tcgen05
    GEMM + gather + heavy-row epilogue into a compact buffer) go through the
    chunked top-k and are scattered into the result; the light queries keep
    the fused sweep top-k.  Indices equal the oracle's up to ties, and equal
    the sweep-only path's."""
    from paper_2104_06357_b200 import _lib
    idx = _f32(sd.generate(sd.GenSpec(2600, 1600, "zipf", zipf_s=1.15, zipf_max_degree=900, seed=61)))
    deg = np.diff(np.asarray(idx.indptr))
    heavy = np.flatnonzero(deg >= max(64, -(-idx.n_cols // 32)))
    rows = np.unique(np.concatenate([heavy[:30], np.arange(0, idx.n_rows, 53)]))
    q = _gather_rows(idx, rows)
    spec = sd.metric_registry("cosine")
    ref_d, ref_i = O.kneighbors(idx, q, k, "cosine")
    with _lib.tuned(hybrid=2, dense=0):
        hidx = _host(idx)
        res = sd.kneighbors(hidx, _host(q), k, spec, dtype=np.float32)
        assert "dot" in _lib.device_index(sd.to_device(hidx, np.float32)).hybrid_blocks
    with _lib.tuned(hybrid=0, dense=0):
        sweep = sd.kneighbors(_host(idx), _host(q), k, spec, dtype=np.float32)
    for got in (res, sweep):
        np.testing.assert_allclose(got.distances, ref_d, rtol=1e-5, atol=1e-5)
        same = got.indices == ref_i
        ties = np.abs(got.distances - ref_d) <= 1e-5
        assert (same | ties).all()


@pytest.mark.parametrize("shape", [(300, 517, 700), (130, 129, 64)])
def test_dense_mode_vs_oracle(shape):
    """Dense-index mode (dense_tc.cu, knob dense=2 forces it on any index):
    the whole matrix as one tcgen05 bf16 GEMM with the metric in the
    epilogue; two bf16 planes (hi, lo) for general values, one for
    bf16-exact (binary) values.  Ragged tile edges (rows, queries and columns
    not multiples of 128 / 64).  Every dot-family metric against the oracle
    (fp32), and jaccard on binary data exactly equal to the sweep."""
    from paper_2104_06357_b200 import _lib
    n_idx, n_q, n_cols = shape
    idx = _f32(sd.generate(sd.GenSpec(n_idx, n_cols, "uniform", degree=max(3, n_cols // 12), seed=81)))
    q = _f32(sd.generate(sd.GenSpec(n_q, n_cols, "uniform", degree=max(3, n_cols // 10), seed=82)))
    for name in DOT_FAMILY:
        a, b = (q, idx) if name not in ("dice", "jaccard", "russelrao") else (
            q.with_values(np.ones(q.nnz)), idx.with_values(np.ones(idx.nnz)))
        a, b = _host(a), _host(b)
        spec = sd.metric_registry(name)
        with _lib.tuned(dense=2):
            got = sd.pairwise_distances(a, b, spec, dtype=np.float32)
        ref = O.pairwise_distances(a, b, name)
        assert_parity(got, ref, a, b, name, np.float32, what=f"dense/{name}")
        if name == "jaccard":
            with _lib.tuned(dense=0):
                sweep = sd.pairwise_distances(_host(a), _host(b), spec, dtype=np.float32)
            np.testing.assert_array_equal(got, sweep)


@pytest.mark.parametrize("n_heavy_q", [17, 300])
def test_hybrid_gemm_routes(n_heavy_q):
    """The heavy block's tcgen05 bf16 GEMM (dense_tc.cu, K split, hi/lo
    planes) with 128 queries per CTA (17 heavy queries) and 256 per CTA over
    two query tiles (300), against the oracle (fp32)."""
    idx = _f32(sd.generate(sd.GenSpec(2600, 1600, "zipf", zipf_s=1.15, zipf_max_degree=900, seed=61)))
    deg = np.diff(np.asarray(idx.indptr))
    heavy = np.flatnonzero(deg >= max(64, -(-idx.n_cols // 32)))
    q = _gather_rows(idx, np.sort(heavy[:n_heavy_q]))
    from paper_2104_06357_b200 import _lib
    for name in ("cosine", "euclidean"):
        a, b = _host(q), _host(idx)
        with _lib.tuned(hybrid=2, dense=0):
            got = sd.pairwise_distances(a, b, sd.metric_registry(name), dtype=np.float32)
        ref = O.pairwise_distances(a, b, name)
        assert_parity(got, ref, a, b, name, np.float32, what=f"hybrid gemm {n_heavy_q}/{name}")


# ------------------------------------------------------------ regressions

def test_knn_forced_strategy_ragged_index():
    """Forced-strategy kNN reads distance rows through their padded stride
    (index row count not a multiple of 4)."""
    x = _host(sd.generate(sd.GenSpec(301, 250, "zipf", zipf_s=1.3, zipf_max_degree=80, seed=71)))
    q = sd.slice_rows(x, 0, 23)
    spec = sd.metric_registry("manhattan")
    ref_d, ref_i = O.kneighbors(x, q, 6, "manhattan")
    full = O.pairwise_distances(q, x, "manhattan")
    for strategy, rows in (("dense", 7), ("hash", 5), ("naive", 23)):
        res = sd.kneighbors(x, q, 6, spec, strategy=strategy, batch_rows=rows)
        assert_knn_parity(res.distances, res.indices, ref_d, ref_i, full, tol=1e-11)


def test_hellinger_on_device_inputs():
    """DeviceCsr inputs (sd.upload) get the sqrt value transform exactly once."""
    rng = np.random.default_rng(72)
    a = sd.from_dense(np.where(rng.random((12, 40)) < 0.4, rng.uniform(0.1, 2, (12, 40)), 0.0))
    b = sd.from_dense(np.where(rng.random((30, 40)) < 0.4, rng.uniform(0.1, 2, (30, 40)), 0.0))
    ref = O.pairwise_distances(a, b, "hellinger")
    spec = sd.metric_registry("hellinger")
    da = sd.upload(a.n_rows, a.n_cols, a.indptr, a.indices, a.values)
    db = sd.upload(b.n_rows, b.n_cols, b.indptr, b.indices, b.values)
    for x, y in ((da, db), (da, b), (a, db)):
        for strategy in (None, "dense"):
            got = sd.pairwise_distances(x, y, spec, strategy)
            assert_parity(got, ref, a, b, "hellinger", np.float64, what=f"hellinger device/{strategy}")
    ref_d, ref_i = O.kneighbors(b, a, 4, "hellinger")
    for strategy in (None, "dense"):
        res = sd.kneighbors(db, da, 4, spec, strategy=strategy, batch_rows=5)
        assert_knn_parity(res.distances, res.indices, ref_d, ref_i, ref, tol=1e-11)
    # an fp32 device matrix used at the default float64 compute dtype is converted, not misread
    d32 = sd.upload(a.n_rows, a.n_cols, a.indptr, a.indices, np.asarray(a.values, np.float32))
    got = sd.pairwise_distances(d32, a, sd.metric_registry("cosine"))
    ref32 = O.pairwise_distances(a.with_values(np.asarray(a.values, np.float32).astype(np.float64)), a, "cosine")
    np.testing.assert_allclose(got, ref32, rtol=1e-6, atol=1e-6)


@pytest.mark.parametrize("dtype", DTYPES)
def test_forced_dense_wider_than_shared_memory(dtype):
    """strategy='dense' with n_cols beyond one shared-memory window (column
    windows of the staged row, engine.cu build_classes)."""
    a = _f32(sd.generate(sd.GenSpec(20, 70000, "uniform", degree=300, seed=73)))
    b = _f32(sd.generate(sd.GenSpec(45, 70000, "uniform", degree=300, seed=74)))
    for name in ("manhattan", "cosine"):
        ref = O.pairwise_distances(a, b, name)
        got = sd.pairwise_distances(a, b, sd.metric_registry(name), "dense", dtype=dtype)
        assert_parity(got, ref, a, b, name, dtype, what=f"wide dense {name}")


def test_timings_report_device_footprint():
    """pairwise_distances_detail's timings carry the device footprint beside
    the reference-shaped WorkspaceReport: the cached index and the output."""
    a = _host(sd.generate(sd.GenSpec(30, 200, "uniform", degree=10, seed=91)))
    b = _host(sd.generate(sd.GenSpec(50, 200, "uniform", degree=10, seed=92)))
    _, report, timings = sd.pairwise_distances_detail(a, b, sd.metric_registry("cosine"), dtype=np.float32)
    assert timings["device_index_bytes"] > 0
    assert timings["device_output_bytes"] >= 30 * 50 * 4
    assert report.peak_accumulator_entries >= 0


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_kl_coverage_rows_over_65536_columns(dtype):
    """The fused kernel keeps 16-bit KL coverage counts; query rows of >= 65,536
    columns are settled by the index row's degree, the count modulo 2^16 and a
    merge of the sorted rows (metrics.py:352-366 coverage, permissive KL)."""
    n = 140000
    rng = np.random.default_rng(65536)

    def rows(col_sets):
        d = np.zeros((len(col_sets), n))
        for r, cols in enumerate(col_sets):
            d[r, cols] = rng.uniform(0.1, 1.0, len(cols))
        return sd.from_dense(d)

    q = rows([np.arange(66000), np.arange(65536), np.arange(0, 40, 4)])
    b = rows([np.arange(70000),                       # covers all three queries
              np.arange(1, 66001),                    # misses column 0
              np.arange(70000, 136000),               # disjoint from query 1 (count 0 == 65536 mod 2^16)
              np.arange(0, 65999),                    # one column short of query 0
              np.arange(0, 40, 2)])                   # covers query 2 only
    got = sd.pairwise_distances(q, b, sd.metric_registry("kl", strict=False), dtype=dtype)
    ref = O.pairwise_distances_c(q, b, "kl", strict=False)
    covered = ref < 1e300
    assert covered.tolist() == [[True, False, False, False, False],
                                [True, False, False, True, False],
                                [True, False, False, True, True]]
    assert (np.isfinite(got) & (got < 1e300)).tolist() == covered.tolist()
    assert_parity(got, ref, q, b, "kl", dtype, what="kl rows over 65,536 columns")
