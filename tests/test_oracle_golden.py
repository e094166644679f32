"""Pin the oracle (oracle/semidist_oracle.py) to the reference's own outputs.

The golden vectors were produced by running /root/reference (semidist) on
seeded inputs (tests/golden/make_golden.py); the numpy restatement must
reproduce them BITWISE — it evaluates the same numpy operations in the same
order.  CPU only.
"""

import numpy as np
import pytest

from golden_cases import csr, strategy_arg
from oracle import semidist_oracle as O

_RINGS_P = {"abs-diff-pow": 1.5}


def test_golden_has_all_metrics(golden):
    cases, _ = golden
    metrics = {c["metric"] for c in cases if c["kind"] == "pairwise"}
    assert metrics == set(O.METRIC_NAMES)


def test_oracle_pairwise_bitwise(golden):
    cases, arrays = golden
    n = 0
    for c in cases:
        if c["kind"] != "pairwise":
            continue
        a, b = csr(arrays, c["a"]), csr(arrays, c["b"])
        got = O.pairwise_distances(a, b, c["metric"], p=c["p"], strict=c["strict"],
                                   strategy=strategy_arg(c["strategy"]))
        np.testing.assert_array_equal(got, arrays[c["id"] + ".out"], err_msg=c["id"])
        n += 1
    assert n > 100


def test_oracle_generalized_bitwise(golden):
    cases, arrays = golden
    for c in cases:
        if c["kind"] == "generalized":
            a, b = csr(arrays, c["a"]), csr(arrays, c["b"])
            got = O.generalized(a, b, c["ring"], p=_RINGS_P.get(c["ring"]))
            np.testing.assert_array_equal(got, arrays[c["id"] + ".out"], err_msg=c["id"])
        elif c["kind"] == "pass1":
            a, b = csr(arrays, c["a"]), csr(arrays, c["b"])
            ring = O.semiring(c["ring"])
            out = np.zeros((a.n_rows, b.n_rows))
            O.balanced_pass(a, b, ring, out, False)
            np.testing.assert_array_equal(out, arrays[c["id"] + ".out"])


def test_oracle_knn_bitwise(golden):
    cases, arrays = golden
    for c in cases:
        if c["kind"] != "knn":
            continue
        q, ix = csr(arrays, c["a"]), csr(arrays, c["b"])
        d, i = O.kneighbors(ix, q, c["k"], c["metric"])
        np.testing.assert_array_equal(i, arrays[c["id"] + ".idx"], err_msg=c["id"])
        np.testing.assert_array_equal(d, arrays[c["id"] + ".dist"], err_msg=c["id"])


def test_appendix_known_answers():
    """Manhattan appendix: 3 over both passes, 1 after pass 1."""
    a = O.csr_of_dense([[1.0, 0.0, 1.0]])
    b = O.csr_of_dense([[0.0, 1.0, 0.0]])
    assert O.pairwise_distances(a, b, "manhattan")[0, 0] == 3.0
    out = np.zeros((1, 1))
    O.balanced_pass(a, b, O.semiring("abs-diff"), out, False)
    assert out[0, 0] == 1.0


def test_oracle_matches_dense_arbiter():
    """Every metric vs the textbook dense formulas (oracle.py restated), rtol 1e-6/atol 1e-9
    as verification.py:12-13."""
    rng = np.random.default_rng(3)
    for name in O.METRIC_NAMES:
        for _ in range(3):
            m, n, k = rng.integers(1, 15), rng.integers(1, 15), rng.integers(1, 20)
            binary = name in ("dice", "jaccard", "russelrao", "hamming")
            ma, mb = rng.random((m, k)) < 0.4, rng.random((n, k)) < 0.4
            da = ma.astype(float) if binary else np.where(ma, rng.uniform(0.1, 1, (m, k)), 0)
            db = mb.astype(float) if binary else np.where(mb, rng.uniform(0.1, 1, (n, k)), 0)
            if name == "kl":
                db = rng.uniform(0.1, 1, (n, k))
            p = 2.5 if name == "minkowski" else None
            got = O.pairwise_distances(O.csr_of_dense(da), O.csr_of_dense(db), name, p=p)
            want = O.dense_pairwise(da, db, name, p=p)
            np.testing.assert_allclose(got, want, rtol=1e-6, atol=1e-9, err_msg=name)


def test_min_plus_exact():
    rng = np.random.default_rng(10)
    for _ in range(5):
        da = np.where(rng.random((8, 8)) < 0.4, rng.uniform(0.1, 1, (8, 8)), 0.0)
        db = np.where(rng.random((8, 8)) < 0.4, rng.uniform(0.1, 1, (8, 8)), 0.0)
        got = O.generalized(O.csr_of_dense(da), O.csr_of_dense(db), "min-plus")
        np.testing.assert_array_equal(got, O.min_plus_dense(da, db))


def test_oracle_vs_live_reference(reference_semidist):
    """Beyond the fixtures: a fresh random C1-style case against the live reference."""
    sd = reference_semidist
    A = sd.generate(sd.GenSpec(30, 2000, "uniform", degree=40, seed=11))
    B = sd.generate(sd.GenSpec(50, 2000, "zipf", zipf_s=1.4, zipf_max_degree=300, seed=12))
    for name in ("manhattan", "cosine", "jensenshannon", "chebyshev"):
        want = sd.pairwise_distances(A, B, sd.metric_registry(name))
        got = O.pairwise_distances(A, B, name)
        np.testing.assert_array_equal(got, want)


def test_c_oracle_pinned_to_golden(golden):
    """The C restatement (oracle/semidist_oracle.c, used for config-scale parity)
    equals every golden pairwise case to rounding — sequential instead of
    numpy's pairwise summation — and bit-for-bit where the sums are exact."""
    cases, arrays = golden
    n = 0
    for c in cases:
        if c["kind"] != "pairwise" or c["strategy"] not in (None, "auto"):
            continue
        a, b = csr(arrays, c["a"]), csr(arrays, c["b"])
        ref = arrays[c["id"] + ".out"]
        got = O.pairwise_distances_c(a, b, c["metric"], p=c["p"], strict=c["strict"], threads=4)
        sat = ref >= 1e308
        assert ((got >= 1e308) == sat).all(), c["id"]
        if c["metric"] in ("chebyshev", "hamming", "jaccard", "dice", "russelrao"):
            np.testing.assert_array_equal(got, ref, err_msg=c["id"])
        else:
            np.testing.assert_allclose(np.where(sat, 0, got), np.where(sat, 0, ref), rtol=1e-14, atol=1e-14,
                                       err_msg=c["id"])
        n += 1
    assert n >= 15


def test_c_oracle_vs_numpy_port_midsize():
    """C restatement vs the bitwise-pinned numpy port on a 40 x 3000 power-law case."""
    A = O.Csr.of(_zipf(40, 3000, 1.3, 700, 5))
    B = O.Csr.of(_zipf(300, 3000, 1.3, 700, 6))
    for name in O.METRIC_NAMES:
        p = 1.5 if name == "minkowski" else None
        want = O.pairwise_distances(A, B, name, p=p, strict=False)
        got = O.pairwise_distances_c(A, B, name, p=p, strict=False, threads=3)
        sat = want >= 1e308
        assert ((got >= 1e308) == sat).all(), name
        np.testing.assert_allclose(np.where(sat, 0, got), np.where(sat, 0, want), rtol=1e-12, atol=1e-12,
                                   err_msg=name)


def test_c_oracle_domain_errors():
    a = O.csr_of_dense([[0.5, 0.5]])
    b = O.csr_of_dense([[1.0, 0.0]])
    with pytest.raises(O.OracleDomainError):
        O.pairwise_distances_c(a, b, "kl")
    assert O.pairwise_distances_c(a, b, "kl", strict=False)[0, 0] == 1e308
    with pytest.raises(O.OracleDomainError):
        O.pairwise_distances_c(O.csr_of_dense([[-1.0, 0.5]]), b, "hellinger")


def _zipf(n, k, s, mx, seed):
    import paper_2104_06357_b200 as sd
    return sd.generate(sd.GenSpec(n, k, "zipf", zipf_s=s, zipf_max_degree=mx, seed=seed))
