"""Parity rule between the CUDA path and the reference/oracle.

    |got - ref| <= rtol * |ref| + atol_ij

rtol is BASELINE.json's: 1e-12 for float64, 1e-5 for float32.  atol_ij is the
same rtol applied to the magnitude of the terms the metric sums for that pair
(the reference's own ATOL is 1e-9 absolute, verification.py:13); metrics that
end in a square root near zero use sqrt(rtol * magnitude), the rounding
amplification of sqrt at the origin.  Saturated KL cells (1e308 / +inf) are
compared as a mask.  kNN indices must match exactly except where the swapped
indices are ties within the same tolerance.
"""

import numpy as np

from oracle.semidist_oracle import Csr, _norm, segment_reduce

RTOL = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}


def one_sided(m, metric, p=None):
    m = Csr.of(m)
    v = np.abs(m.values)
    if metric in ("canberra", "hamming"):
        t = np.ones_like(v)
    elif metric == "minkowski":
        t = v ** p
    elif metric == "jensenshannon":
        t = v * np.log(2.0)
    else:
        t = v
    return segment_reduce(t, m.indptr, np.add, 0.0)


def atol_matrix(a, b, metric, rtol, p=None):
    a, b = Csr.of(a), Csr.of(b)
    m, n = a.n_rows, b.n_rows
    if metric in ("manhattan", "canberra", "hamming", "chebyshev"):
        s = one_sided(a, metric)[:, None] + one_sided(b, metric)[None, :]
        if metric == "hamming":
            s = s / max(1, a.n_cols)
        return rtol * s + 1e-300
    if metric == "minkowski":
        s = one_sided(a, metric, p)[:, None] + one_sided(b, metric, p)[None, :]
        return (rtol * s) ** (1.0 / p) + rtol * s ** (1.0 / p)
    if metric == "jensenshannon":
        s = one_sided(a, metric)[:, None] + one_sided(b, metric)[None, :]
        return np.sqrt(rtol * s) + 1e-300
    if metric == "euclidean":
        s = _norm(a, "l2sq")[:, None] + _norm(b, "l2sq")[None, :]
        return np.sqrt(rtol * s) + 1e-300
    if metric == "dot":
        return rtol * (_norm(a, "l2")[:, None] * _norm(b, "l2")[None, :]) + 1e-300
    if metric == "correlation":
        return np.full((m, n), rtol * max(1.0, a.n_cols))
    if metric == "hellinger":
        return np.full((m, n), np.sqrt(rtol))
    if metric == "kl":
        return np.full((m, n), rtol * 10.0)
    return np.full((m, n), rtol * 4.0)


def assert_parity(got, ref, a, b, metric, dtype, p=None, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} != {ref.shape}"
    if got.size == 0:
        return
    rtol = RTOL[np.dtype(dtype)]
    sat_ref = ref >= 1e308
    sat_got = got >= (1e308 if np.dtype(dtype) == np.float64 else np.inf)
    assert (sat_ref == sat_got).all(), f"{what}: KL saturation masks differ"
    ok = ~sat_ref
    atol = atol_matrix(a, b, metric, rtol, p)
    err = np.abs(got - ref)
    lim = rtol * np.abs(ref) + atol
    bad = ok & ~(err <= lim)
    if bad.any():
        i, j = np.argwhere(bad)[0]
        raise AssertionError(f"{what} [{metric}, {np.dtype(dtype).name}]: {int(bad.sum())} cells out of "
                             f"tolerance; first ({i},{j}) got {got[i, j]!r} ref {ref[i, j]!r} "
                             f"err {err[i, j]:.3e} lim {lim[i, j]:.3e}")


def assert_knn_parity(got_d, got_i, ref_d, ref_i, ref_full, tol):
    """Indices equal except at ties (|d_ref[q, got] - d_ref[q, ref]| <= tol)."""
    got_d, ref_d = np.asarray(got_d, dtype=np.float64), np.asarray(ref_d, dtype=np.float64)
    assert got_i.shape == ref_i.shape
    assert np.all(np.abs(got_d - ref_d) <= tol + 1e-300 + tol * np.abs(ref_d)), "kNN distances differ"
    diff = got_i != ref_i
    for q, t in np.argwhere(diff):
        alt = ref_full[q, got_i[q, t]]
        assert abs(alt - ref_d[q, t]) <= tol * (1 + abs(ref_d[q, t])), \
            f"query {q} slot {t}: index {got_i[q, t]} (d={alt}) vs {ref_i[q, t]} (d={ref_d[q, t]}) not a tie"
    for q in range(got_i.shape[0]):
        assert len(set(got_i[q].tolist())) == got_i.shape[1], "duplicate neighbour ids"
