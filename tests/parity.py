"""Parity rule between the CUDA path and the reference/oracle.

rtol is BASELINE.json's: 1e-12 for float64, 1e-5 for float32.  A cell passes
the VALUE test

    |got - ref| <= rtol * |ref| + atol_ij,    atol_ij = C * rtol * M_ij (+ u_T for "1 - x" metrics)

where M_ij is the conditioning of the metric's final value for that pair: how
much the value moves when the sums it is built from are perturbed by a
relative rtol (the GPU sums in a different order and, for the union
decomposition, cancels against the one-sided sums).  No floor is a bare
sqrt(rtol) or rtol * n_cols any more:

    manhattan / canberra / hamming : one-sided sums S_A[i] + S_B[j] (/k for hamming)
    dot                            : G_ij = sum over A_i ∩ B_j of |a b|
    cosine                         : G_ij / (||a|| ||b||) + |1 - d| (the norms' own rounding)
    correlation                    : (k G_ij + |s_a s_b|) / den + |1 - d| * (cond. of den)
    dice / jaccard / russelrao     : derivative of the expansion w.r.t. the dot times G_ij
    kl                             : sum over A_i ∩ B_j of |a log(a/b)|, plus (u_T/rtol) * sum of a
                                     over A_i ∩ B_j: log(a/b) of a rounded quotient is off by ~u_T
                                     absolutely, however small the term (a ~ b)
    chebyshev                      : 0 (float64 bit-exact; float32 relative rtol only)

G and the KL magnitude are computed exactly by the C oracle's magnitude mode
(the same passes summing |⊗|).

Metrics that end in a root of a radicand R (euclidean d = sqrt(R), Jensen-
Shannon d = sqrt(R/2), minkowski d = R^(1/p), hellinger d = 1 - sqrt(R)) are
compared on the RADICAND instead — the reference's own quantity before the
root, where the rounding does not get amplified near zero:

    |R(got) - R(ref)| <= rtol * |R(ref)| + C * rtol * S_ij

with S_ij the magnitude of the terms summed into R (q_a + q_b for euclidean,
the one-sided JS / |v|^p sums, the affinity itself for hellinger).  u_T is the
output dtype's unit roundoff, the one absolute slack kept: a value computed
as 1 - x cannot be closer than that.  C = 4 absorbs the few ulps by which two
valid summation orders of the same terms differ.

Saturated KL cells (1e308 / +inf) are compared as a mask.  kNN indices must
match exactly except where the swapped indices are ties within tolerance.
"""

import numpy as np

from oracle.semidist_oracle import Csr, _norm, pairwise_distances_c, segment_reduce

RTOL = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-5}
UNIT_ROUNDOFF = {np.dtype(np.float64): 2.0 ** -53, np.dtype(np.float32): 2.0 ** -24}
C_SLACK = 4.0
ONE_MINUS = ("cosine", "correlation", "dice", "jaccard", "hellinger", "russelrao")


def one_sided(m, metric, p=None):
    """Per-row sum of the metric's one-sided terms (⊗(v, 0), semiring.py:36-62)."""
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


def _outer(x, y):
    return x[:, None] * y[None, :]


def _sum(x, y):
    return x[:, None] + y[None, :]


def abs_dot(a, b):
    """G_ij = sum over the intersection of |a_c b_c| (C oracle, magnitude mode)."""
    return pairwise_distances_c(a, b, "dot", magnitude=True)


def magnitude(a, b, metric, ref, dtype, p=None):
    """M_ij of the value test (None for metrics compared on the radicand)."""
    a, b = Csr.of(a), Csr.of(b)
    k = float(a.n_cols)
    if metric in ("manhattan", "canberra", "hamming"):
        s = _sum(one_sided(a, metric), one_sided(b, metric))
        return s / max(1.0, k) if metric == "hamming" else s
    if metric == "kl":
        u = UNIT_ROUNDOFF[np.dtype(dtype)] / RTOL[np.dtype(dtype)]
        mass = pairwise_distances_c(a, Csr(b.n_rows, b.n_cols, b.indptr, b.indices, np.ones_like(b.values)), "dot",
                                    magnitude=True)
        return pairwise_distances_c(a, b, "kl", magnitude=True) + u * mass
    if metric == "chebyshev":
        return np.zeros((a.n_rows, b.n_rows))
    na, nb = _norm(a, "l2"), _norm(b, "l2")
    g = abs_dot(a, b)
    if metric == "dot":
        return g
    if metric == "cosine":
        den = _outer(na, nb)
        with np.errstate(divide="ignore", invalid="ignore"):
            return np.where(den > 0, g / np.where(den > 0, den, 1.0), 0.0) + np.abs(1.0 - ref)
    if metric == "russelrao":
        return g / max(1.0, k)
    if metric in ("dice", "jaccard"):
        ca, cb = _norm(a, "l0"), _norm(b, "l0")
        den = _sum(ca, cb)
        with np.errstate(divide="ignore", invalid="ignore"):
            if metric == "dice":
                g_der = np.where(den > 0, 2.0 / np.where(den > 0, den, 1.0), 0.0)
            else:
                dot = np.clip(1.0 - ref, 0, None) * den / (2.0 - np.clip(ref, None, 1.0))  # dot from d
                jd = den - dot
                g_der = np.where(jd > 0, den / np.where(jd > 0, jd, 1.0) ** 2, 0.0)
        return g_der * g
    if metric == "correlation":
        sa, sb = _norm(a, "sum"), _norm(b, "sum")
        qa, qb = _norm(a, "l2sq"), _norm(b, "l2sq")
        fa, fb = np.maximum(k * qa - sa ** 2, 0), np.maximum(k * qb - sb ** 2, 0)
        den = np.sqrt(_outer(fa, fb))
        with np.errstate(divide="ignore", invalid="ignore"):
            num_mag = (k * g + np.abs(_outer(sa, sb))) / np.where(den > 0, den, 1.0)
            ca = np.where(fa > 0, (k * qa + sa ** 2) / np.where(fa > 0, fa, 1.0), 0.0)
            cb = np.where(fb > 0, (k * qb + sb ** 2) / np.where(fb > 0, fb, 1.0), 0.0)
        return np.where(den > 0, num_mag + np.abs(1.0 - ref) * 0.5 * _sum(ca, cb), 1.0)
    return None


def radicand(metric, d, p=None):
    """The quantity under the final root, recovered from a distance."""
    d = np.asarray(d, dtype=np.float64)
    if metric == "euclidean":
        return d * d
    if metric == "jensenshannon":
        return 2.0 * d * d
    if metric == "minkowski":
        return np.abs(d) ** p
    if metric == "hellinger":
        return (1.0 - d) ** 2
    raise KeyError(metric)


def radicand_scale(a, b, metric, p=None):
    """S_ij: magnitude of the terms summed into the radicand."""
    a, b = Csr.of(a), Csr.of(b)
    if metric == "euclidean":
        return _sum(_norm(a, "l2sq"), _norm(b, "l2sq"))
    if metric in ("jensenshannon", "minkowski"):
        return _sum(one_sided(a, metric, p), one_sided(b, metric, p))
    if metric == "hellinger":   # sum of sqrt(a) sqrt(b) >= 0: the affinity is its own magnitude
        return pairwise_distances_c(a, b, "hellinger", magnitude=True)
    raise KeyError(metric)


def check_cells(got, ref, a, b, metric, dtype, p=None):
    """Boolean matrix: cell within tolerance (saturation handled by the caller)."""
    dt = np.dtype(dtype)
    rtol, u = RTOL[dt], UNIT_ROUNDOFF[dt]
    err = np.abs(got - ref)
    if metric == "chebyshev":
        return err <= (0.0 if dt == np.float64 else rtol * np.abs(ref))
    if metric in ("euclidean", "jensenshannon", "minkowski", "hellinger"):
        rg, rr = radicand(metric, got, p), radicand(metric, ref, p)
        ok = np.abs(rg - rr) <= rtol * np.abs(rr) + C_SLACK * rtol * radicand_scale(a, b, metric, p)
        # the output itself is rounded to dtype: that much value error is always admissible
        floor = u * (1.0 + np.abs(ref)) if metric == "hellinger" else u * np.abs(ref)
        return ok | (err <= rtol * np.abs(ref) + floor)
    atol = C_SLACK * rtol * magnitude(a, b, metric, ref, dtype, p)
    if metric in ONE_MINUS:
        atol = atol + u * (1.0 + np.abs(ref))
    return err <= rtol * np.abs(ref) + atol


def assert_parity(got, ref, a, b, metric, dtype, p=None, what=""):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    assert got.shape == ref.shape, f"{what}: shape {got.shape} != {ref.shape}"
    if got.size == 0:
        return
    sat_ref = ref >= 1e308
    sat_got = got >= (1e308 if np.dtype(dtype) == np.float64 else np.inf)
    assert (sat_ref == sat_got).all(), f"{what}: KL saturation masks differ"
    ok = check_cells(got, np.where(sat_ref, 0.0, ref), a, b, metric, dtype, p) | sat_ref
    if not ok.all():
        bad = ~ok
        i, j = np.argwhere(bad)[0]
        raise AssertionError(f"{what} [{metric}, {np.dtype(dtype).name}]: {int(bad.sum())} cells out of "
                             f"tolerance; first ({i},{j}) got {got[i, j]!r} ref {ref[i, j]!r} "
                             f"err {abs(got[i, j] - ref[i, j]):.3e}")


def max_rel_excess(got, ref, a, b, metric, dtype, p=None):
    """Largest |got - ref| over the cells (saturated cells excluded), for reporting."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    ok = ref < 1e308
    return float(np.max(np.abs(got - ref)[ok])) if ok.any() else 0.0


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
