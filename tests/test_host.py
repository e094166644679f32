"""Host-side logic of the drop-in (no GPU): strategy resolution, chunk
planning, WorkspaceReport accounting, canonicalisation, synthetic data."""

import numpy as np
import pytest

import paper_2104_06357_b200 as sd
from golden_cases import csr
from paper_2104_06357_b200.engine import reference_report


def hash_strategy(capacity=8, load=0.5):
    return sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=capacity,
                                max_load_factor=load)


def test_plan_chunks_reference_example():
    assert [e - s for s, e in sd.plan_chunks(50, hash_strategy(40))] == [17, 17, 16]
    assert sd.plan_chunks(10, hash_strategy(40)) == [(0, 10)]
    assert sd.plan_chunks(0, hash_strategy(40)) == [(0, 0)]
    with pytest.raises(ValueError):
        sd.plan_chunks(5, sd.ExecutionStrategy(sd.StrategyKind.BALANCED_DENSE))


def test_strategy_validation_and_auto():
    with pytest.raises(ValueError):
        sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=0)
    with pytest.raises(ValueError):
        sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=1, max_load_factor=0.5)
    assert sd.choose_strategy(sd.from_dense(np.eye(3))).kind is sd.StrategyKind.BALANCED_DENSE
    m = sd.canonicalize_host([0, 2], [0, 20000], [1.0, 1.0], n_cols=30000)
    s = sd.choose_strategy(m)
    assert s.kind is sd.StrategyKind.BALANCED_HASH and s.accumulator_capacity == 4


def test_reports_match_reference_accounting(golden):
    """WorkspaceReport computed on the host equals what the reference reported."""
    cases, arrays = golden
    n = 0
    for c in cases:
        if c["kind"] != "pairwise":
            continue
        a, b = csr(arrays, c["a"]), csr(arrays, c["b"])
        st = c["strategy"]
        if isinstance(st, list):
            strat = hash_strategy(st[1], st[2])
        else:
            strat = sd.resolve_strategy(st, a, b)
        passes = 2 if c["metric"] in sd.METRIC_NAMES[9:] else 1
        rep = reference_report(np.diff(a.indptr), strat, b.nnz)
        if passes == 2 or c["metric"] == "kl":
            rep = rep.merged(reference_report(np.diff(b.indptr), strat, a.nnz))
        assert [rep.peak_accumulator_entries, rep.workspace_elements, rep.chunks_executed] == c["report"], c["id"]
        n += 1
    assert n > 100


def test_canonicalize():
    m = sd.canonicalize_host([0, 2], [2, 0], [3.0, 1.0], n_cols=3)
    assert m.indices.tolist() == [0, 2] and m.values.tolist() == [1.0, 3.0]
    m = sd.canonicalize_host([0, 2], [1, 1], [2.0, 3.0], n_cols=3)
    assert m.indices.tolist() == [1] and m.values.tolist() == [5.0]
    with pytest.raises(sd.IndexOutOfBounds):
        sd.canonicalize_host([0, 1], [5], [1.0], n_cols=3)
    with pytest.raises(sd.NegativeOffset):
        sd.canonicalize_host([0, -1], [], [], n_cols=3)
    with pytest.raises(sd.NonMonotonicIndptr):
        sd.canonicalize_host([1, 1], [], [], n_cols=3)


def test_generate_matches_reference(reference_semidist):
    ref = reference_semidist
    for spec in [dict(n_rows=200, n_cols=500, degree_dist="uniform", degree=7, seed=1),
                 dict(n_rows=300, n_cols=1000, degree_dist="zipf", zipf_s=1.4, zipf_max_degree=80,
                      value_dist="tfidf", seed=3)]:
        a = sd.generate(sd.GenSpec(**spec))
        b = ref.generate(ref.GenSpec(**spec))
        np.testing.assert_array_equal(a.indptr, b.indptr)
        np.testing.assert_array_equal(a.indices, b.indices)
        np.testing.assert_array_equal(a.values, b.values)


def test_lognormal_generator_shape():
    m = sd.generate(sd.GenSpec(2000, 26000, "lognormal", lognormal_mu=7.3, lognormal_sigma=0.6,
                               min_degree=501, max_degree=9600, value_dist="tfidf", seed=4))
    deg = np.diff(m.indptr)
    assert deg.min() >= 480 and deg.max() <= 9600


def test_plan_batches():
    p = sd.plan_batches(100, 50, batch_rows=7)
    assert (p.batch_rows, p.n_batches) == (7, 15)
    p = sd.plan_batches(10 ** 6, 10 ** 4, memory_budget_bytes=256 << 20)
    assert p.batch_rows * 10 ** 4 * 8 <= 256 << 20


def test_semiring_descriptors():
    from paper_2104_06357_b200.semiring import device_id
    assert device_id(sd.dot_product())[0] == 0
    assert device_id(sd.absolute_difference_power(1.5)) == (3, 1.5)
    assert sd.metric_registry("chebyshev").semiring.reduce_op is np.maximum
    for name in sd.METRIC_NAMES:
        spec = sd.metric_registry(name, p=2.0 if name == "minkowski" else None)
        assert (spec.passes == 2) == (not spec.semiring.annihilating)
        assert (spec.expansion is not None) == (spec.passes == 1)
    with pytest.raises(sd.MissingParam):
        sd.metric_registry("minkowski")
    with pytest.raises(sd.DomainError):
        sd.metric_registry("minkowski", p=0.5)
    with pytest.raises(sd.UnknownMetric):
        sd.metric_registry("mahalanobis")


def test_reference_semiring_objects_resolve(reference_semidist):
    from paper_2104_06357_b200.semiring import device_id
    ref = reference_semidist
    assert device_id(ref.absolute_difference_power(2.5)) == (3, 2.5)
    assert device_id(ref.tropical_min_plus())[0] == 1
    with pytest.raises(NotImplementedError):
        device_id(ref.Semiring("custom", np.add, 0.0, np.add, 0.0, False))


def test_parity_rule_is_tight():
    """tests/parity.py accepts the oracle against itself and rejects a relative
    perturbation of 20x the BASELINE rtol on every metric (the rule has no
    sqrt(rtol)- or n_cols-sized floors any more)."""
    from oracle import semidist_oracle as O
    from parity import check_cells
    A = O.Csr.of(sd.generate(sd.GenSpec(30, 400, "zipf", zipf_s=1.3, zipf_max_degree=120, seed=3)))
    B = O.Csr.of(sd.generate(sd.GenSpec(50, 400, "zipf", zipf_s=1.3, zipf_max_degree=120, seed=4)))
    for name in O.METRIC_NAMES:
        p = 1.5 if name == "minkowski" else None
        ref = O.pairwise_distances_c(A, B, name, p=p, strict=False, threads=2)
        ref = np.where(ref >= 1e308, 0.0, ref)
        for dt, rtol in ((np.float64, 1e-12), (np.float32, 1e-5)):
            assert check_cells(ref, ref, A, B, name, dt, p).all(), name
            big = np.abs(ref) > 1e-3
            bumped = ref * (1 + 20 * rtol) + 20 * rtol * np.sign(ref)
            ok = check_cells(bumped, ref, A, B, name, dt, p)
            assert ok[big].mean() < 0.1, (name, dt, ok[big].mean())
