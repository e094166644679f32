"""Small C1-size invocations of every hot kernel, for compute-sanitizer
(tools/sanitize.sh): the fused sweep (isect_kernel, dot family, NAMM,
chebyshev masks, KL counts, top-k), the engine (pass_kernel dense / hash,
naive_kernel), the hybrid heavy-row path (tcgen05 GEMM, gather, min-sum
block, heavy-row epilogue) and the dense-index tcgen05 GEMM.  Results are
checked loosely against the oracle so a silent corruption also fails.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import paper_2104_06357_b200 as sd
    from oracle import semidist_oracle as O
    from paper_2104_06357_b200 import _lib

    def f32(m):
        return m.with_values(np.asarray(m.values, dtype=np.float32).astype(np.float64))

    def check(got, ref, what, tol=1e-3):
        err = float(np.max(np.abs(got - ref) / (1.0 + np.abs(ref))))
        assert err < tol, (what, err)
        print(f"ok {what} {err:.2e}", flush=True)

    A = f32(sd.generate(sd.GenSpec(40, 300, "uniform", degree=12, seed=1)))
    B = f32(sd.generate(sd.GenSpec(70, 300, "uniform", degree=12, seed=2)))
    for name in ("cosine", "manhattan", "chebyshev", "kl", "jensenshannon"):
        spec = sd.metric_registry(name, strict=name != "kl")
        check(sd.pairwise_distances(A, B, spec), O.pairwise_distances(A, B, name, strict=name != "kl"), f"sweep {name}")
    for strat in ("dense", "hash", "naive"):
        spec = sd.metric_registry("manhattan")
        check(sd.pairwise_distances(A, B, spec, strategy=strat), O.pairwise_distances(A, B, "manhattan"),
              f"engine {strat}")
    res = sd.kneighbors(B, A, 5, sd.metric_registry("cosine"))
    _, ref_i = O.kneighbors(B, A, 5, "cosine")
    assert (res.indices[:, 0] == ref_i[:, 0]).mean() > 0.9
    print("ok knn", flush=True)
    X = f32(sd.generate(sd.GenSpec(600, 400, "zipf", zipf_s=1.15, zipf_max_degree=300, seed=61)))
    Q = sd.slice_rows(X, 0, 60)
    with _lib.tuned(hybrid=2, dense=0):
        for name in ("cosine", "manhattan"):
            check(sd.pairwise_distances(Q, X, sd.metric_registry(name), dtype=np.float32),
                  O.pairwise_distances(Q, X, name), f"hybrid {name}")
    with _lib.tuned(dense=2):
        check(sd.pairwise_distances(Q, X, sd.metric_registry("cosine"), dtype=np.float32),
              O.pairwise_distances(Q, X, "cosine"), "dense cosine")


if __name__ == "__main__":
    main()
