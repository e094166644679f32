"""Generate golden input/output vectors by running the REFERENCE itself.

Run here (the reference cannot travel to the GPU box):
    python tests/golden/make_golden.py
It imports semidist from /root/reference/pkg/src, evaluates it on seeded
inputs and writes tests/golden/golden.npz + golden.json.  Tests pin both the
oracle (tests/test_oracle_golden.py, CPU) and the CUDA path
(tests/test_gpu_parity.py) against these files.
"""

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)
import semidist as sd  # noqa: E402
from semidist.verification import random_instance  # noqa: E402

arrays = {}
cases = []


def put_csr(prefix, m):
    arrays[prefix + ".indptr"] = np.asarray(m.indptr, dtype=np.int64)
    arrays[prefix + ".indices"] = np.asarray(m.indices, dtype=np.int64)
    arrays[prefix + ".values"] = np.asarray(m.values, dtype=np.float64)
    return {"n_rows": int(m.n_rows), "n_cols": int(m.n_cols), "key": prefix}


def add_pairwise(cid, a, b, metric, p=None, strict=True, strategy=None, note=""):
    spec = sd.metric_registry(metric, p=p, strict=strict)
    strat = strategy
    if isinstance(strategy, tuple):
        strat = sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=strategy[1],
                                     max_load_factor=strategy[2])
    out, rep, _ = sd.pairwise_distances_detail(a, b, spec, strat)
    arrays[cid + ".out"] = out
    cases.append({"id": cid, "kind": "pairwise", "metric": metric, "p": p, "strict": strict,
                  "strategy": list(strategy) if isinstance(strategy, tuple) else strategy,
                  "a": put_csr(cid + ".a", a), "b": put_csr(cid + ".b", b),
                  "report": [rep.peak_accumulator_entries, rep.workspace_elements, rep.chunks_executed],
                  "note": note})


def add_generalized(cid, a, b, ring_name, ring, strategy=None):
    out, rep = sd.pairwise_generalized(a, b, ring, strategy)
    arrays[cid + ".out"] = out
    cases.append({"id": cid, "kind": "generalized", "ring": ring_name, "p": getattr(ring, "p", None),
                  "a": put_csr(cid + ".a", a), "b": put_csr(cid + ".b", b),
                  "report": [rep.peak_accumulator_entries, rep.workspace_elements, rep.chunks_executed]})


def add_knn(cid, index, queries, k, metric, batch_rows=None):
    spec = sd.metric_registry(metric)
    res = sd.kneighbors(index, queries, k, spec, batch_rows=batch_rows)
    arrays[cid + ".dist"] = res.distances
    arrays[cid + ".idx"] = res.indices
    cases.append({"id": cid, "kind": "knn", "metric": metric, "k": k,
                  "a": put_csr(cid + ".q", queries), "b": put_csr(cid + ".i", index)})


def main():
    # appendix vectors (test_acceptance.py:62-73)
    a = sd.from_dense([[1.0, 0.0, 1.0]])
    b = sd.from_dense([[0.0, 1.0, 0.0]])
    add_pairwise("appendix_manhattan", a, b, "manhattan")
    out = sd.allocate_output(a, b, sd.absolute_difference())
    sd.pairwise_spmv_pass1(a, b, sd.absolute_difference(), sd.ExecutionStrategy(sd.StrategyKind.BALANCED_DENSE), out)
    arrays["appendix_pass1.out"] = out
    cases.append({"id": "appendix_pass1", "kind": "pass1", "ring": "abs-diff", "p": None,
                  "a": put_csr("appendix_pass1.a", a), "b": put_csr("appendix_pass1.b", b)})

    # all 15 metrics on the reference's own verification instances (verification.py:28-51)
    rng = np.random.default_rng(20240417)
    for name in sd.METRIC_NAMES:
        for t in range(6):
            a, b = random_instance(rng, name, max_rows=24, max_cols=40)
            p = float(rng.choice([1.0, 1.5, 2.0, 3.0])) if name == "minkowski" else None
            strat = [None, "dense", ("hash", 8, 0.5), "naive", None, ("hash", 16, 0.5)][t]
            add_pairwise(f"metric_{name}_{t}", a, b, name, p=p, strategy=strat)

    # zero-norm / empty rows and degenerate shapes (test_metrics.py:164-184)
    e = sd.from_dense([[0.0, 0.0, 0.0], [1.0, 0.5, 0.0], [0.0, 0.0, 2.0]])
    for name in sd.METRIC_NAMES:
        p = 2.0 if name == "minkowski" else None
        add_pairwise(f"empty_rows_{name}", e, e, name, p=p, strict=False)
    # KL strict failure is an exception; permissive saturates (test_metrics.py:197-207)
    add_pairwise("kl_permissive", sd.from_dense([[0.5, 0.5], [0.2, 0.0]]),
                 sd.from_dense([[1.0, 0.0], [0.3, 0.7]]), "kl", strict=False)

    # semirings through pairwise_generalized incl. tropical (test_engine.py:200-238)
    rings = {"dot": sd.dot_product(), "abs-diff": sd.absolute_difference(),
             "abs-diff-max": sd.max_absolute_difference(), "canberra-ratio": sd.canberra_ratio(),
             "mismatch": sd.mismatch_indicator(), "jensen-shannon-term": sd.jensen_shannon_term(),
             "min-plus": sd.tropical_min_plus(), "abs-diff-pow": sd.absolute_difference_power(1.5)}
    rng = np.random.default_rng(5)
    for t in range(3):
        da = np.where(rng.random((12, 30)) < 0.35, rng.uniform(0.1, 1.0, (12, 30)), 0.0)
        db = np.where(rng.random((9, 30)) < 0.35, rng.uniform(0.1, 1.0, (9, 30)), 0.0)
        for rn, ring in rings.items():
            add_generalized(f"ring_{rn}_{t}", sd.from_dense(da), sd.from_dense(db), rn, ring)

    # C1-shaped slice (BASELINE config 1: 1% uniform density, 10k cols), fp32-representable values
    A = sd.generate(sd.GenSpec(64, 10000, "uniform", degree=100, seed=1))
    B = sd.generate(sd.GenSpec(200, 10000, "uniform", degree=100, seed=2))
    A = A.with_values(A.values.astype(np.float32).astype(np.float64))
    B = B.with_values(B.values.astype(np.float32).astype(np.float64))
    for name in ("manhattan", "cosine", "euclidean", "chebyshev", "jensenshannon", "canberra", "hellinger",
                 "correlation", "minkowski"):
        add_pairwise(f"c1slice_{name}", A, B, name, p=3.0 if name == "minkowski" else None)
    # high-dimensional power-law slice (hash path in the reference)
    Z = sd.generate(sd.GenSpec(400, 60000, "zipf", zipf_s=1.5, zipf_max_degree=3000, seed=25))
    Z = Z.with_values(Z.values.astype(np.float32).astype(np.float64))
    Q = sd.slice_rows(Z, 0, 40)
    for name in ("cosine", "euclidean", "manhattan", "kl"):
        add_pairwise(f"zipf_{name}", Q, Z, name, strict=False)

    # kNN (knn.py:50-94) incl. ties on binary data
    X = sd.generate(sd.GenSpec(300, 200, "zipf", zipf_s=1.3, zipf_max_degree=60, seed=8))
    add_knn("knn_cosine", X, sd.slice_rows(X, 0, 50), 10, "cosine", batch_rows=17)
    XB = X.with_values(np.ones_like(X.values))
    add_knn("knn_jaccard_ties", XB, sd.slice_rows(XB, 0, 50), 7, "jaccard")
    add_knn("knn_manhattan", X, sd.slice_rows(X, 100, 140), 5, "manhattan")

    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump({"generator": "tests/golden/make_golden.py", "reference": "semidist " + sd.__version__,
                   "numpy": np.__version__, "cases": cases}, f, indent=1)
    print(f"{len(cases)} cases, {sum(v.nbytes for v in arrays.values()) / 1e6:.1f} MB raw")


if __name__ == "__main__":
    main()
