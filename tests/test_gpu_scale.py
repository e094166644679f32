"""Config-scale parity: the CUDA path vs the oracle at BASELINE.json's full
index sizes.

Query samples are small (16-64 rows) but every index is the FULL config
index, so the kernels run with the tile counts, L2 bands, hybrid heavy-row
blocks and posting-list lengths of the benchmark.  The checker is the C
restatement of the reference algorithm (oracle/semidist_oracle.c, pinned to
the reference's golden vectors by tests/test_oracle_golden.py); the rule is
tests/parity.py (BASELINE rtol 1e-5 fp32 / 1e-12 fp64 with conditioning-
based magnitudes, radicand comparison for root metrics).  Inputs are rounded
to fp32 once, so fp32 storage is not an error source and both dtypes are
checked against the same fp64 oracle.
"""

import numpy as np
import pytest

import paper_2104_06357_b200 as sd
from bench import WORKLOADS, binary, gather_rows
from oracle import semidist_oracle as O
from parity import assert_knn_parity, assert_parity

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

DTYPES = [np.float32, np.float64]


def _index(name):
    return sd.round_values_f32(sd.generate(sd.GenSpec(**WORKLOADS[name]["index"])))


def _sample(index, n_random, n_heavy=0, min_heavy=0, seed=26):
    """n_random rows drawn like the benchmark's queries plus n_heavy rows of
    degree >= min_heavy (the power-law tail the hybrid / long-row paths serve)."""
    rng = np.random.default_rng(seed)
    rows = set(rng.choice(index.n_rows, n_random, replace=False).tolist())
    if n_heavy:
        deg = np.diff(np.asarray(index.indptr))
        heavy = np.flatnonzero(deg >= min_heavy)
        assert heavy.size >= n_heavy, (heavy.size, n_heavy)
        rows |= set(rng.choice(heavy, n_heavy, replace=False).tolist())
    rows = np.array(sorted(rows))
    return rows, gather_rows(index, rows)


@pytest.fixture(scope="module")
def c2():
    index = _index("c2")
    theta = max(64, -(-index.n_cols // 32))   # hybrid heavy-row threshold (hybrid.cu)
    rows, q = _sample(index, 56, n_heavy=8, min_heavy=theta)
    return index, rows, q


@pytest.mark.parametrize("metric", ["cosine", "euclidean", "manhattan"])
def test_c2_full_index(c2, metric):
    """C2: 64 queries (8 of them heavy rows -> hybrid tensor-core path for the
    dot family) x the full 162,541 x 59,047 power-law index (zipf s = 1.544)."""
    index, rows, q = c2
    ref = O.pairwise_distances_c(q, index, metric)
    spec = sd.metric_registry(metric)
    for dtype in DTYPES:
        got = sd.pairwise_distances(q, index, spec, dtype=dtype)
        assert_parity(got, ref, q, index, metric, dtype, what=f"C2 {metric}")
    if metric != "cosine":   # self-distances (covered by the rule above) are exactly 0 in the reference
        assert np.all(ref[np.arange(len(rows)), rows] == 0.0)


@pytest.fixture(scope="module")
def c3():
    index = _index("c3")
    rows, q = _sample(index, 32)
    return index, rows, q


@pytest.mark.parametrize("metric", ["canberra", "chebyshev", "jensenshannon", "kl"])
def test_c3_full_index(c3, metric):
    """C3: 32 queries x the full 300,000 x 102,660 tf-idf index; the NAMM
    metrics (union decomposition over one-sided sums) and permissive KL."""
    index, rows, q = c3
    strict = metric != "kl"
    ref = O.pairwise_distances_c(q, index, metric, strict=strict)
    spec = sd.metric_registry(metric, strict=strict)
    for dtype in DTYPES:
        got = sd.pairwise_distances(q, index, spec, dtype=dtype)
        assert_parity(got, ref, q, index, metric, dtype, what=f"C3 {metric}")
    if metric == "kl":
        assert (ref >= 1e308).any() and (ref < 1e308).any()   # both classes exercised


@pytest.fixture(scope="module")
def c4():
    index = _index("c4")
    deg = np.diff(np.asarray(index.indptr))
    rows, q = _sample(index, 8, n_heavy=8, min_heavy=2048)   # rows of 2k-9.6k nonzeros
    assert deg[rows].max() > 4096
    return index, rows, q


@pytest.mark.parametrize("metric", ["hellinger", "jaccard"])
def test_c4_full_index(c4, metric):
    """C4: 16 queries (half of them 2k-9.6k nonzeros) x the full 65,000 x 26,000
    dense-ish index; jaccard on the binary pattern (BINARY_PREFERRED)."""
    index, rows, q = c4
    if metric == "jaccard":
        index, q = binary(index), binary(q)
    ref = O.pairwise_distances_c(q, index, metric)
    spec = sd.metric_registry(metric)
    for dtype in DTYPES:
        got = sd.pairwise_distances(q, index, spec, dtype=dtype)
        assert_parity(got, ref, q, index, metric, dtype, what=f"C4 {metric}")
        diag = got[np.arange(len(rows)), rows]
        if metric == "jaccard":     # counts are exact: self-distance exactly 0, as in the reference
            assert np.all(diag == 0.0) and np.all(ref[np.arange(len(rows)), rows] == 0.0)


@pytest.fixture(scope="module")
def c5():
    index = _index("c5")
    rows, q = _sample(index, 32)
    return index, rows, q


def test_c5_knn_full_index(c5):
    """C5: cosine k = 32 for 32 queries against the full 1,000,000-row index;
    indices bit-exact except inside tolerance tie groups (test_acceptance.py:203-233)."""
    index, rows, q = c5
    k = WORKLOADS["c5"]["k"]
    ref_d, ref_i, full = O.kneighbors_c(index, q, k, "cosine")
    spec = sd.metric_registry("cosine")
    for dtype, tol in ((np.float64, 1e-11), (np.float32, 1e-5)):
        res = sd.kneighbors(index, q, k, spec, dtype=dtype)
        assert_knn_parity(res.distances, res.indices, ref_d, ref_i, full, tol=tol)
