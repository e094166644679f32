"""The drop-in surface beyond the distance kernels, on the GPU: the reference's
own unit tests for segment_reduce, the hash accumulator, mix32, semiring
products, metric epilogues, Matrix Market I/O, canonicalisation and the CLI
(/root/reference/pkg/tests/test_sparse.py, test_hashtable.py, test_semiring.py,
test_mmio.py, test_cli.py) re-pointed at paper_2104_06357_b200, plus reference
objects passed straight into the drop-in and the INTEGRATION.md binding."""

import json
import os
import re
import subprocess
import sys

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

import paper_2104_06357_b200 as sd
from oracle import semidist_oracle as O
from parity import assert_parity

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _random_dense(rng, m, k, density, low=0.05, high=1.0, binary=False):
    mask = rng.random((m, k)) < density
    return mask.astype(np.float64) if binary else np.where(mask, rng.uniform(low, high, (m, k)), 0.0)


def _densify(m):
    out = np.zeros((m.n_rows, m.n_cols))
    out[np.repeat(np.arange(m.n_rows), np.diff(m.indptr)), np.asarray(m.indices)] = m.values
    return out


# ------------------------------------------------------------ segment_reduce (sparse.py:31-53)

def test_segment_reduce_reference_cases():
    np.testing.assert_array_equal(sd.segment_reduce(np.array([1.0, 2.0, 3.0]), [0, 0, 2, 2, 3], np.add, 0.0),
                                  [0.0, 3.0, 0.0, 3.0])
    np.testing.assert_array_equal(sd.segment_reduce(np.array([1.0, 5.0, 2.0]), [0, 2, 3], np.maximum, 0.0),
                                  [5.0, 2.0])
    np.testing.assert_array_equal(sd.segment_reduce(np.array([3.0, 1.0]), [0, 0, 2], np.minimum, np.inf),
                                  [np.inf, 1.0])
    with pytest.raises(ValueError):
        sd.segment_reduce(np.array([1.0, 2.0]), [0, 1], np.add, 0.0)
    with pytest.raises(NotImplementedError):
        sd.segment_reduce(np.array([1.0, 2.0]), [0, 2], np.subtract, 0.0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_segment_reduce_bitwise_reduceat(dtype):
    """numpy's reduceat association (v[0] + pairwise sum of the rest) reproduced
    bit for bit, for every segment length class (< 8, <= 128, recursive halves)."""
    rng = np.random.default_rng(5)
    lengths = list(range(0, 140)) + [255, 256, 257, 1000, 4097, 25000]
    bounds = np.concatenate(([0], np.cumsum(lengths)))
    v = (rng.standard_normal(bounds[-1]) * rng.uniform(0, 1e3, bounds[-1])).astype(dtype)
    got = sd.segment_reduce(v, bounds, np.add, 0.0)
    starts = bounds[:-1]
    ne = starts < bounds[1:]
    want = np.zeros(len(lengths))
    want[ne] = np.add.reduceat(v, starts[ne])
    np.testing.assert_array_equal(got, want)
    for uf, ident in ((np.maximum, 0.0), (np.minimum, np.inf), (np.multiply, 1.0)):
        w = np.full(len(lengths), ident)
        vv = v if uf is not np.multiply else (1 + 1e-3 * v).astype(dtype)
        w[ne] = uf.reduceat(vv, starts[ne])
        np.testing.assert_array_equal(sd.segment_reduce(vv, bounds, uf, ident), w)


# ------------------------------------------------------------ hash accumulator (hashtable.py)

def test_hash_build_probe_and_rebuild():
    t = sd.HashAccumulator(8)
    t.build(np.array([3, 7]), np.array([1.5, 2.0]))
    assert t.probe(7) == 2.0 and t.probe(3) == 1.5 and t.probe(11) is None
    t2 = sd.HashAccumulator(16)
    t2.build(np.array([2, 9, 11]), np.array([0.5, 1.0, 2.5]))
    vals, found = t2.probe_many(np.array([9, 4, 11, 2, 100]))
    np.testing.assert_array_equal(vals, [1.0, 0.0, 2.5, 0.5, 0.0])
    np.testing.assert_array_equal(found, [True, False, True, True, False])
    e = sd.HashAccumulator(4)
    e.build(np.array([], dtype=np.int64), np.array([]))
    assert not e.probe_many(np.array([1, 2, 3]))[1].any() and e.probe(1) is None
    t.build(np.array([5]), np.array([9.0]))
    assert t.probe(3) is None and t.probe(5) == 9.0
    with pytest.raises(ValueError):
        sd.HashAccumulator(4).build(np.arange(4), np.ones(4))
    with pytest.raises(ValueError):
        sd.HashAccumulator(0)
    assert sd.EMPTY_SLOT == np.iinfo(np.int64).max
    t37 = sd.HashAccumulator(37)
    assert t37._keys.size == 37 and t37._values.size == 37


def test_hash_adversarial_collisions_at_half_load():
    """Keys that all hash to shared slots (multiples of the capacity), 50% load
    (test_hashtable.py:45-59)."""
    cap = 64
    t = sd.HashAccumulator(cap)
    keys = np.arange(0, 32, dtype=np.int64) * cap
    vals = np.arange(32, dtype=np.float64) + 1.0
    t.build(keys, vals)
    ref = dict(zip(keys.tolist(), vals.tolist()))
    probe = np.concatenate([keys, keys + 1, np.array([cap * 100])])
    v, f = t.probe_many(probe)
    for key, vv, ff in zip(probe.tolist(), v, f):
        assert (ff and vv == ref[key]) if key in ref else (not ff and vv == 0.0)


def _layout(keys, vals, cap):
    """The reference's sequential insertion (hashtable.py:43-63), for the slot layout."""
    tk = np.full(cap, sd.EMPTY_SLOT, dtype=np.int64)
    tv = np.zeros(cap)
    for k, v in zip(keys.tolist(), vals.tolist()):
        h = int(_mix32_np(np.array([k]))[0] % np.uint64(cap))
        while tk[h] != sd.EMPTY_SLOT:
            h = (h + 1) % cap
        tk[h], tv[h] = k, v
    return tk, tv


def _mix32_np(keys):
    h = np.asarray(keys).astype(np.uint64) & np.uint64(0xFFFFFFFF)
    h ^= h >> np.uint64(16)
    h = (h * np.uint64(0x85EBCA6B)) & np.uint64(0xFFFFFFFF)
    h ^= h >> np.uint64(13)
    h = (h * np.uint64(0xC2B2AE35)) & np.uint64(0xFFFFFFFF)
    return h ^ (h >> np.uint64(16))


@settings(max_examples=40, deadline=None)
@given(st.integers(0, 10 ** 6))
def test_hash_matches_dict_and_reference_layout(seed):
    rng = np.random.default_rng(seed)
    cap = int(rng.integers(2, 65))
    n = int(rng.integers(0, cap // 2 + 1))
    keys = rng.choice(10 * cap, size=n, replace=False).astype(np.int64)
    vals = rng.random(n)
    t = sd.HashAccumulator(cap)
    t.build(keys, vals)
    tk, tv = _layout(keys, vals, cap)
    np.testing.assert_array_equal(t._keys, tk)
    ref = dict(zip(keys.tolist(), vals.tolist()))
    q = rng.integers(0, 10 * cap, size=40).astype(np.int64)
    v, f = t.probe_many(q)
    for key, vv, ff in zip(q.tolist(), v, f):
        assert ff == (key in ref) and vv == ref.get(key, 0.0)
        assert t.probe(key) == ref.get(key, None)


def test_mix32_matches_reference_formula():
    keys = np.concatenate([np.arange(1000), np.array([2 ** 31, 2 ** 33 + 5, -7, np.iinfo(np.int64).max])])
    got = sd.mix32(keys)
    assert got.dtype == np.uint64
    np.testing.assert_array_equal(got, _mix32_np(keys))
    assert np.unique(np.diff(got[:1000].astype(np.int64))).size > 10


# ------------------------------------------------------------ semiring products (semiring.py)

def test_semiring_products_on_device():
    assert float(sd.metric_registry("manhattan").semiring.product_op(3.0, 1.0)) == 2.0
    ring = sd.absolute_difference()
    assert [float(ring.product_op(x, y)) for x, y in ((1, 0), (0, 1), (0, 0), (1, 1))] == [1.0, 1.0, 0.0, 0.0]
    assert float(sd.canberra_ratio().product_op(0.0, 0.0)) == 0.0
    js = sd.jensen_shannon_term()
    np.testing.assert_allclose(float(js.product_op(0.7, 0.0)), 0.7 * np.log(2.0), rtol=1e-15)
    np.testing.assert_allclose(float(js.product_op(0.0, 0.7)), 0.7 * np.log(2.0), rtol=1e-15)
    trop = sd.tropical_min_plus()
    assert float(trop.product_op(2.0, 4.0)) == 6.0 and float(trop.reduce_op(3.0, 5.0)) == 3.0
    for v in (0.0, 1.5, 1e6):
        for r in (sd.absolute_difference(), sd.canberra_ratio(), sd.mismatch_indicator(),
                  sd.jensen_shannon_term(), sd.max_absolute_difference(), sd.absolute_difference_power(1.5)):
            assert np.isfinite(float(r.product_op(v, 0.0))) and np.isfinite(float(r.product_op(0.0, v)))
        assert float(sd.dot_product().product_op(v, 0.0)) == 0.0
    # broadcasting, as criterion 4's dense evaluation uses it
    rng = np.random.default_rng(1)
    da, db = rng.uniform(0.1, 1, (5, 7)), rng.uniform(0.1, 1, (4, 7))
    prods = sd.absolute_difference_power(2.5).product_op(da[:, None, :], db[None, :, :])
    np.testing.assert_allclose(prods, np.abs(da[:, None, :] - db[None, :, :]) ** 2.5, rtol=1e-14)
    with pytest.raises(TypeError):
        sd.Semiring("bad", np.add, 0.0, lambda x, y: x + y, 0.0, False)


def test_metric_epilogue_callables():
    """MetricSpec.expansion / post_scale are callables with the reference's
    signatures, evaluated on device (metrics.py:40-52, 102-180)."""
    rng = np.random.default_rng(3)
    a = sd.from_dense(_random_dense(rng, 6, 9, 0.5))
    b = sd.from_dense(_random_dense(rng, 5, 9, 0.5))
    for name in sd.METRIC_NAMES:
        p = 1.5 if name == "minkowski" else None
        spec = sd.metric_registry(name, p=p, strict=False)
        raw = O.generalized(a if name != "hellinger" else O.Csr.of(a).with_values(np.sqrt(a.values)),
                            b if name != "hellinger" else O.Csr.of(b).with_values(np.sqrt(b.values)),
                            O._RING.get(name, "dot"), p=p)
        norms_a = [sd.row_norms(a, k) for k in spec.norms_needed]
        norms_b = [sd.row_norms(b, k) for k in spec.norms_needed]
        sa = sd.SideStats.from_norms(norms_a, signed_sum=sd.row_signed_sums(a))
        sb = sd.SideStats.from_norms(norms_b, signed_sum=sd.row_signed_sums(b))
        out = spec.expansion(raw, sa, sb, a.n_cols) if spec.expansion else raw
        if spec.post_scale is not None:
            out = spec.post_scale(out, a.n_cols)
        want = O.expand(name, raw, O.Csr.of(a), O.Csr.of(b), a.n_cols, p)
        np.testing.assert_allclose(out, want, rtol=1e-13, atol=1e-13, err_msg=name)
    euc = sd.metric_registry("euclidean")
    radic = euc.expansion(np.array([[1.0]]), sd.SideStats(l2sq=np.array([2.0])), sd.SideStats(l2sq=np.array([1.0])), 2)
    assert radic[0, 0] == 1.0 and euc.post_scale(np.array([[4.0]]), 2)[0, 0] == 2.0


# ------------------------------------------------------------ canonicalisation + Matrix Market

def test_canonicalize_device_matches_host():
    """sd_canonicalize vs the numpy restatement: unsorted rows, duplicates
    (summed in input order, bitwise), explicit and cancelling zeros, empty rows."""
    rng = np.random.default_rng(9)
    for trial in range(20):
        n_rows, n_cols = int(rng.integers(0, 40)), int(rng.integers(1, 30))
        deg = rng.integers(0, 12, n_rows)
        ptr = np.concatenate(([0], np.cumsum(deg))).astype(np.int64)
        idx = rng.integers(0, n_cols, ptr[-1])
        val = rng.choice([0.0, 1.0, -1.0, 0.1, 2.5, 1e-17, 3.0], ptr[-1]) * rng.uniform(0.5, 2, ptr[-1])
        if trial % 3 == 0 and ptr[-1] > 1:
            val[1] = -val[0]
            idx[1] = idx[0]
        got = sd.validate_and_canonicalize(ptr, idx, val, n_cols=n_cols)
        want = sd.canonicalize_host(ptr, idx, val, n_cols=n_cols)
        assert got.n_rows == want.n_rows
        np.testing.assert_array_equal(got.indptr, want.indptr)
        np.testing.assert_array_equal(got.indices, want.indices)
        np.testing.assert_array_equal(got.values, want.values)


def test_canonicalize_errors_name_the_row():
    with pytest.raises(sd.IndexOutOfBounds) as e:
        sd.validate_and_canonicalize([0, 1, 3], [0, 1, 9], [1.0, 1.0, 1.0], n_cols=3)
    assert (e.value.row, e.value.column, e.value.n_cols) == (1, 9, 3)
    with pytest.raises(sd.NegativeOffset) as e:
        sd.validate_and_canonicalize([0, -1, 1], [0], [1.0], n_cols=3)
    assert e.value.row == 1 and e.value.offset == -1
    with pytest.raises(sd.NonMonotonicIndptr) as e:
        sd.validate_and_canonicalize([0, 2, 1, 3], [0, 1, 1], [1.0, 1.0, 1.0], n_cols=3)
    assert e.value.row == 1
    with pytest.raises(sd.NonMonotonicIndptr):
        sd.validate_and_canonicalize([1, 1], [], [], n_cols=3)
    with pytest.raises(ValueError):
        sd.validate_and_canonicalize([0, 2], [0], [1.0], n_cols=3)
    m = sd.validate_and_canonicalize([0, 2], [1, 1], [2.0, 3.0], n_cols=3)
    assert m.indices.tolist() == [1] and m.values.tolist() == [5.0]


def _write(tmp_path, text, name="m.mtx"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_matrix_market_reader(tmp_path):
    m = sd.read_matrix_market(_write(tmp_path, "%%MatrixMarket matrix coordinate real general\n2 3 1\n1 3 2.5\n"))
    assert (m.n_rows, m.n_cols, m.nnz) == (2, 3, 1) and _densify(m)[0, 2] == 2.5
    m = sd.read_matrix_market(_write(tmp_path, "%%MatrixMarket matrix coordinate pattern general\n2 2 1\n2 1\n"))
    np.testing.assert_array_equal(_densify(m), [[0, 0], [1.0, 0]])
    m = sd.read_matrix_market(_write(tmp_path, "%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n"
                                               "2 1 4.0\n3 3 1.0\n"))
    d = _densify(m)
    assert (d == d.T).all() and d[1, 0] == 4.0 and d[2, 2] == 1.0
    m = sd.read_matrix_market(_write(tmp_path, "%%MatrixMarket matrix coordinate real general\n% c\n\n"
                                               "1 1 1\n1 1 7.0\n"))
    assert m.values[0] == 7.0
    m = sd.read_matrix_market(_write(tmp_path, "%%MatrixMarket matrix coordinate integer general\n1 1 1\n1 1 3\n"))
    assert m.values[0] == 3.0
    m = sd.read_matrix_market(_write(tmp_path, "%%MatrixMarket matrix coordinate real general\n2 2 3\n"
                                               "2 2 1.0\n1 2 0.5\n2 2 -1.0\n"))
    assert m.nnz == 1 and m.values[0] == 0.5   # duplicates summed, the cancelled entry dropped
    cases = [("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n2 2\n", sd.ParseError, 4),
             ("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n", sd.ParseError, None),
             ("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n", sd.ParseError, 3),
             ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 1.0\n", sd.ParseError, 4),
             ("%%MatrixMarket matrix coordinate real general\n2 2 1\n1 x 1.0\n", sd.ParseError, 3),
             ("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1.0 0.0\n", sd.UnsupportedField, None),
             ("%%MatrixMarket matrix array real general\n1 1\n1.0\n", sd.UnsupportedField, None),
             ("1 1 1\n1 1 1.0\n", sd.ParseError, 1)]
    for text, exc, line in cases:
        with pytest.raises(exc) as e:
            sd.read_matrix_market(_write(tmp_path, text))
        if line is not None:
            assert e.value.line_no == line, text


def test_matrix_market_round_trip_and_writers(tmp_path):
    rng = np.random.default_rng(0)
    for _ in range(10):
        m = sd.from_dense(_random_dense(rng, int(rng.integers(0, 12)), int(rng.integers(1, 10)), 0.4, -2.0, 2.0))
        path = str(tmp_path / "rt.mtx")
        sd.write_matrix_market(m, path)
        back = sd.read_matrix_market(path)
        np.testing.assert_array_equal(back.indptr, m.indptr)
        np.testing.assert_array_equal(back.indices, m.indices)
        np.testing.assert_array_equal(back.values, m.values)
    p = tmp_path / "d.csv"
    sd.write_output(np.array([[3.0, 1.5]]), str(p), "csv", header=True)
    assert p.read_text().splitlines() == ["j0,j1", "3,1.5"]
    mat = rng.random((3, 4))
    sd.write_output(mat, str(p), "csv")
    np.testing.assert_array_equal(np.array([[float(t) for t in l.split(",")] for l in p.read_text().splitlines()]),
                                  mat)
    sd.write_output(mat, str(tmp_path / "d.json"), "json")
    np.testing.assert_array_equal(np.array(json.loads((tmp_path / "d.json").read_text())["distances"]), mat)
    res = sd.NeighborResult(np.array([[0.5, 1.0]]), np.array([[2, 0]]))
    sd.write_output(res, str(tmp_path / "k.csv"), "csv", header=True)
    assert (tmp_path / "k.csv").read_text().splitlines() == ["query_id,neighbor_id,distance", "0,2,0.5", "0,0,1"]
    sd.write_output(sd.NeighborResult(np.array([[0.5], [0.25]]), np.array([[1], [0]])), str(tmp_path / "k.json"),
                    "json")
    assert json.loads((tmp_path / "k.json").read_text())[0] == {"query_id": 0, "neighbor_id": 1, "distance": 0.5}
    with pytest.raises(ValueError):
        sd.write_output(np.zeros((1, 1)), str(tmp_path / "x"), "yaml")


# ------------------------------------------------------------ CLI (cli.py, exit codes 0/1/2/3)

@pytest.fixture()
def small_mtx(tmp_path):
    rng = np.random.default_rng(11)
    path = tmp_path / "X.mtx"
    sd.write_matrix_market(sd.from_dense(_random_dense(rng, 40, 30, 0.25, 0.1, 1.0)), str(path))
    return str(path)


def test_cli_dist_knn_gen(tmp_path, small_mtx, capsys):
    from paper_2104_06357_b200.cli import main
    a, b = tmp_path / "a.mtx", tmp_path / "b.mtx"
    sd.write_matrix_market(sd.from_dense([[1, 0, 1]]), str(a))
    sd.write_matrix_market(sd.from_dense([[0, 1, 0]]), str(b))
    out = tmp_path / "d.csv"
    assert main(["dist", "--metric", "manhattan", "--input", str(a), "--input-b", str(b), "--out", str(out)]) == 0
    assert out.read_text() == "3\n"
    outs = []
    for strat in ("naive", "dense", "hash"):
        o = tmp_path / f"{strat}.csv"
        assert main(["dist", "--metric", "manhattan", "--input", small_mtx, "--strategy", strat, "--out", str(o)]) == 0
        outs.append(np.array([[float(t) for t in l.split(",")] for l in o.read_text().splitlines()]))
    np.testing.assert_allclose(outs[0], outs[1], atol=1e-10)
    np.testing.assert_allclose(outs[1], outs[2], atol=1e-10)
    assert main(["dist", "--metric", "minkowski", "--input", small_mtx]) == 2
    assert main(["dist", "--metric", "manhattan", "--input", "/nonexistent.mtx"]) == 2
    assert main(["dist", "--metric", "manhattan"]) == 1
    assert main(["dist", "--metric", "nosuch", "--input", "x"]) == 1
    assert main(["nosuchcommand"]) == 1
    k = tmp_path / "k.json"
    assert main(["knn", "--metric", "euclidean", "--k", "1", "--input", small_mtx, "--out", str(k),
                 "--format", "json"]) == 0
    assert all(r["query_id"] == r["neighbor_id"] for r in json.loads(k.read_text()))
    g1, g2 = tmp_path / "g1.mtx", tmp_path / "g2.mtx"
    args = ["gen", "--rows", "80", "--cols", "60", "--degree-dist", "zipf:1.2:30", "--seed", "9"]
    assert main(args + ["--out", str(g1)]) == 0 and main(args + ["--out", str(g2)]) == 0
    assert g1.read_text() == g2.read_text()
    capsys.readouterr()


def test_cli_bench_checksums_and_verify(small_mtx, capsys, monkeypatch):
    from paper_2104_06357_b200 import cli, harness
    sums = []
    for strat in ("naive", "dense", "hash"):
        assert cli.main(["bench", "--metric", "manhattan", "--input", small_mtx, "--k", "3", "--strategy", strat,
                         "--json"]) == 0
        rep = json.loads(capsys.readouterr().out)
        for phase in ("load", "norms", "pass1", "pass2", "expansion", "topk"):
            assert phase in rep["timings"]
        sums.append(rep["checksum"])
    assert len(set(sums)) == 1
    assert cli.main(["bench", "--metric", "dot", "--input", small_mtx, "--json"]) == 0
    assert json.loads(capsys.readouterr().out)["timings"]["pass2"] == 0.0
    assert cli.main(["verify", "--metric", "all", "--trials", "4"]) == 0
    assert capsys.readouterr().out.strip().endswith("PASS")
    monkeypatch.setattr(cli, "verify_metric", lambda name, **kw: harness.VerifyResult(name, 1, 1, 1.0))
    assert cli.main(["verify", "--metric", "manhattan", "--trials", "1"]) == 3
    proc = subprocess.run([sys.executable, "-m", "paper_2104_06357_b200", "--help"], capture_output=True, text=True,
                          cwd=ROOT)
    assert proc.returncode == 0 and "verify" in proc.stdout


def test_checksum_agrees_with_cpu_reference():
    """run_bench's quantized checksum of GPU kNN distances equals the one of
    the oracle's (bench.py:18-23: reduction-order noise below 1e-8 vanishes)."""
    from paper_2104_06357_b200.harness import quantized_checksum, run_bench
    A = sd.round_values_f32(sd.generate(sd.GenSpec(1000, 10000, "uniform", degree=100, seed=1)))
    B = sd.round_values_f32(sd.generate(sd.GenSpec(1000, 10000, "uniform", degree=100, seed=2)))
    for name in ("manhattan", "cosine"):
        rep = run_bench(B, A, sd.metric_registry(name), k=10)
        d, _ = O.kneighbors(B, A, 10, name)
        assert rep["checksum"] == quantized_checksum(d), name


def test_verify_dense_arbiter_errors():
    from paper_2104_06357_b200.harness import dense_pairwise, verify_metric
    with pytest.raises(sd.DomainError):
        dense_pairwise(np.array([[-1.0, 1.0]]), np.array([[1.0, 1.0]]), "hellinger")
    with pytest.raises(sd.DomainError):
        dense_pairwise(np.array([[0.5, 0.5]]), np.array([[1.0, 0.0]]), "kl")
    assert dense_pairwise(np.array([[0.5, 0.5]]), np.array([[1.0, 0.0]]), "kl", strict=False)[0, 0] == 1e308
    for name in sd.METRIC_NAMES:
        assert verify_metric(name, trials=10, seed=1234).passed, name


# ------------------------------------------------------------ acceptance criteria (test_acceptance.py)

NAIVE = sd.ExecutionStrategy(sd.StrategyKind.NAIVE_MERGE)
DENSE = sd.ExecutionStrategy(sd.StrategyKind.BALANCED_DENSE)


def _metric_instance(rng, name, m, n, k, density):
    binary = name in sd.BINARY_PREFERRED
    da = _random_dense(rng, m, k, density, low=0.1, binary=binary)
    db = rng.uniform(0.1, 1.0, (n, k)) if name == "kl" else _random_dense(rng, n, k, density, low=0.1, binary=binary)
    return sd.from_dense(da), sd.from_dense(db)


def test_criterion_01_02_golden_appendix_and_oracle_suite():
    a, b = sd.from_dense([[1.0, 0.0, 1.0]]), sd.from_dense([[0.0, 1.0, 0.0]])
    spec = sd.metric_registry("manhattan")
    assert sd.pairwise_distances(a, b, spec)[0, 0] == 3.0
    out = sd.allocate_output(a, b, spec.semiring)
    sd.pairwise_spmv_pass1(a, b, spec.semiring, DENSE, out)
    assert out[0, 0] == 1.0
    from paper_2104_06357_b200.harness import verify_metric
    for name in sd.METRIC_NAMES:   # 15 metrics x 50 instances vs the dense arbiter, rtol 1e-6 / atol 1e-9
        res = verify_metric(name, trials=50, max_rows=40, max_cols=32, seed=1234, rtol=1e-6, atol=1e-9)
        assert res.passed, (name, res.failures, res.max_abs_err)


def test_criterion_03_strategy_cross_equivalence():
    rng = np.random.default_rng(99)
    hash8 = sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=8)
    chunked = 0
    for name in sd.METRIC_NAMES:
        spec = sd.metric_registry(name, p=1.5 if name == "minkowski" else None)
        for t in range(20):
            m, n = int(rng.integers(2, 26)), int(rng.integers(2, 26))
            k, dens = (int(rng.integers(16, 33)), 0.5) if t % 2 else (int(rng.integers(4, 33)),
                                                                       float(rng.uniform(0.05, 0.5)))
            a, b = _metric_instance(rng, name, m, n, k, dens)
            chunked += max(int(np.diff(a.indptr).max()), int(np.diff(b.indptr).max())) > 4
            d_naive = sd.pairwise_distances(a, b, spec, NAIVE)
            np.testing.assert_allclose(sd.pairwise_distances(a, b, spec, DENSE), d_naive, atol=1e-10)
            np.testing.assert_allclose(sd.pairwise_distances(a, b, spec, hash8), d_naive, atol=1e-10)
            np.testing.assert_allclose(sd.pairwise_distances(a, b, spec), d_naive, atol=1e-10)
    assert chunked > 50


def test_criterion_04_union_decomposition_exhaustive():
    rng = np.random.default_rng(7)
    two_pass = [sd.metric_registry(n, p=1.5 if n == "minkowski" else None) for n in sd.METRIC_NAMES]
    two_pass = [s for s in two_pass if s.passes == 2]
    assert len(two_pass) == 6

    def dense_eval(da, db, ring):
        return ring.reduce_op.reduce(np.asarray(ring.product_op(da[:, None, :], db[None, :, :])), axis=2)

    for k in (2, 4, 6):
        pat = (np.arange(2 ** k)[:, None] >> np.arange(k)[None, :]) & 1
        da, db = pat * rng.uniform(0.1, 1.0, pat.shape), pat * rng.uniform(0.1, 1.0, pat.shape)
        for spec in two_pass:
            got, _ = sd.pairwise_generalized(sd.from_dense(da), sd.from_dense(db), spec.semiring)
            np.testing.assert_allclose(got, dense_eval(da, db, spec.semiring), atol=1e-12)


def test_criterion_05_06_expanded_route_and_axioms():
    rng = np.random.default_rng(55)
    for _ in range(50):
        m, n, k = int(rng.integers(1, 31)), int(rng.integers(1, 31)), int(rng.integers(1, 25))
        a = sd.from_dense(_random_dense(rng, m, k, float(rng.uniform(0.1, 0.6)), low=0.05))
        b = sd.from_dense(_random_dense(rng, n, k, float(rng.uniform(0.1, 0.6)), low=0.05))
        np.testing.assert_allclose(sd.pairwise_distances(a, b, sd.metric_registry("euclidean")),
                                   sd.pairwise_distances(a, b, sd.metric_registry("minkowski", p=2.0)),
                                   rtol=1e-6, atol=1e-9)
    rng = np.random.default_rng(66)
    x = sd.from_dense(_random_dense(rng, 60, 20, 0.5, low=0.1))
    tri = rng.integers(0, 60, size=(1000, 3))
    for name, p in [("euclidean", None), ("manhattan", None), ("minkowski", 1.0), ("minkowski", 1.5),
                    ("minkowski", 2.0), ("minkowski", 3.0), ("chebyshev", None), ("canberra", None)]:
        for dtype, tol in ((np.float64, 1e-9), (np.float32, 1e-4)):
            d = sd.pairwise_distances(x, x, sd.metric_registry(name, p=p), dtype=dtype)
            assert np.abs(np.diag(d)).max() <= tol and np.abs(d - d.T).max() <= tol, (name, p, dtype)
            assert (d[tri[:, 0], tri[:, 2]] <= d[tri[:, 0], tri[:, 1]] + d[tri[:, 1], tri[:, 2]] + tol).all()


def test_criterion_07_workspace_accounting():
    x = sd.generate(sd.GenSpec(10000, 10000, "uniform", degree=50, seed=42))
    spec = sd.metric_registry("manhattan")
    _, rep, _, _ = sd.kneighbors_detail(x, sd.slice_rows(x, 0, 256), 10, spec, DENSE, batch_rows=256)
    assert rep.workspace_elements == x.nnz
    h = sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=64, max_load_factor=0.5)
    _, rep, _, _ = sd.kneighbors_detail(x, sd.slice_rows(x, 0, 32), 10, spec, h, batch_rows=32)
    assert rep.workspace_elements <= x.nnz and rep.peak_accumulator_entries <= 32 and rep.chunks_executed > x.n_rows


def test_criterion_08_knn_end_to_end():
    x = sd.generate(sd.GenSpec(2000, 1000, "zipf", zipf_s=1.1, zipf_max_degree=500, seed=8))
    spec = sd.metric_registry("cosine")
    res = {r: sd.kneighbors(x, x, 10, spec, batch_rows=r) for r in (64, 500, 2000)}
    for r in (64, 500):
        np.testing.assert_array_equal(res[r].indices, res[2000].indices)
        np.testing.assert_array_equal(res[r].distances, res[2000].distances)
    base = res[2000]
    dense = _densify(x)
    norms = np.sqrt((dense ** 2).sum(axis=1))
    outer = norms[:, None] * norms[None, :]
    ref = np.where(outer > 0, 1.0 - (dense @ dense.T) / np.where(outer > 0, outer, 1.0), 1.0)
    np.fill_diagonal(ref, np.where(norms > 0, np.diag(ref), 0.0))
    assert np.abs(np.take_along_axis(ref, base.indices, axis=1) - base.distances).max() <= 1e-9
    for q in range(2000):
        order = np.lexsort((np.arange(2000), np.round(ref[q], 9)))[:10]
        got = base.indices[q][np.lexsort((base.indices[q], np.round(base.distances[q], 9)))]
        np.testing.assert_array_equal(got, order)


def test_criterion_10_tropical_exact():
    rng = np.random.default_rng(10)
    ring = sd.tropical_min_plus()
    for _ in range(20):
        da, db = _random_dense(rng, 10, 10, 0.4, low=0.1), _random_dense(rng, 10, 10, 0.4, low=0.1)
        for strat in (NAIVE, DENSE, sd.ExecutionStrategy(sd.StrategyKind.BALANCED_HASH, accumulator_capacity=16)):
            got, _ = sd.pairwise_generalized(sd.from_dense(da), sd.from_dense(db), ring, strat)
            np.testing.assert_array_equal(got, O.min_plus_dense(da, db))


# ------------------------------------------------------------ reference objects into the drop-in

class _Kind:
    def __init__(self, value):
        self.value = value


class RefStrategy:
    """Field layout of semidist.ExecutionStrategy (engine.py:59-77)."""

    def __init__(self, kind, accumulator_capacity=0, max_load_factor=0.5):
        self.kind = _Kind(kind)
        self.accumulator_capacity = accumulator_capacity
        self.max_load_factor = max_load_factor


class RefCsr:
    """Field layout of semidist.CsrMatrix (sparse.py:56-94)."""

    def __init__(self, m):
        self.n_rows, self.n_cols = m.n_rows, m.n_cols
        self.indptr, self.indices, self.values = np.array(m.indptr), np.array(m.indices), np.array(m.values)

    @property
    def nnz(self):
        return int(self.indptr[-1])


def _ref_abs_diff_pow(p):
    """A semidist.Semiring-like object whose p lives only in the product closure (semiring.py:90-97)."""
    class Ring:
        pass
    r = Ring()
    r.name = f"abs-diff-pow-{p:g}"
    r.product_op = lambda x, y: np.abs(np.subtract(x, y)) ** p
    r.reduce_op, r.reduce_identity, r.annihilating = np.add, 0.0, False
    return r


def test_reference_shaped_objects_accepted():
    """Objects with the reference classes' field layout (no import of semidist
    on the GPU box) flow through the drop-in: CsrMatrix, MetricSpec (name +
    params), ExecutionStrategy (kind.value) and a Semiring whose p is only in
    the closure of its product."""
    rng = np.random.default_rng(21)
    a = RefCsr(sd.from_dense(_random_dense(rng, 9, 14, 0.4, low=0.1)))
    b = RefCsr(sd.from_dense(_random_dense(rng, 11, 14, 0.4, low=0.1)))

    class RefSpec:
        name, params, passes = "minkowski", {"p": 2.5}, 2

    got = sd.pairwise_distances(a, b, RefSpec(), RefStrategy("hash", 8, 0.5))
    np.testing.assert_allclose(got, O.pairwise_distances(a, b, "minkowski", p=2.5), rtol=1e-12)
    out, _ = sd.pairwise_generalized(a, b, _ref_abs_diff_pow(1.75), RefStrategy("dense"))
    np.testing.assert_allclose(out, O.generalized(a, b, "abs-diff-pow", p=1.75), rtol=1e-12)
    res = sd.kneighbors(b, a, 3, RefSpec(), RefStrategy("naive"))
    ref_d, ref_i = O.kneighbors(b, a, 3, "minkowski", p=2.5)
    np.testing.assert_array_equal(res.indices, ref_i)


def test_real_reference_objects(reference_semidist):
    """With the reference importable (build container): its own objects in, same numbers out."""
    ref = reference_semidist
    A = ref.generate(ref.GenSpec(20, 300, "zipf", zipf_s=1.3, zipf_max_degree=60, seed=3))
    B = ref.generate(ref.GenSpec(30, 300, "zipf", zipf_s=1.3, zipf_max_degree=60, seed=4))
    for name in ("cosine", "manhattan", "jensenshannon"):
        spec = ref.metric_registry(name)
        np.testing.assert_allclose(sd.pairwise_distances(A, B, spec, ref.ExecutionStrategy(ref.StrategyKind.BALANCED_HASH,
                                                                                           accumulator_capacity=16)),
                                   ref.pairwise_distances(A, B, spec), rtol=1e-12, atol=1e-12)
    out, _ = sd.pairwise_generalized(A, B, ref.absolute_difference_power(3.0))
    np.testing.assert_allclose(out, ref.pairwise_generalized(A, B, ref.absolute_difference_power(3.0))[0], rtol=1e-12)


def test_integration_md_binding():
    """The reference-side ctypes binding printed in INTEGRATION.md §2 runs as
    written and agrees with the oracle."""
    text = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = re.search(r"## 2\..*?```python\n(.*?)```", text, re.S).group(1)
    from paper_2104_06357_b200 import _lib
    os.environ["SEMIDIST_B200_LIB"] = _lib.LIB_PATH
    ns = {"DimensionMismatch": sd.DimensionMismatch, "DomainError": sd.DomainError}
    exec(compile(code, "INTEGRATION.md", "exec"), ns)
    rng = np.random.default_rng(4)
    a = sd.from_dense(_random_dense(rng, 7, 20, 0.3))
    b = sd.from_dense(_random_dense(rng, 9, 20, 0.3))
    for name in ("cosine", "manhattan", "chebyshev"):
        got = ns["pairwise_distances_gpu"](a, b, sd.metric_registry(name))
        assert_parity(got, O.pairwise_distances(a, b, name), a, b, name, np.float64, what="INTEGRATION")
    with pytest.raises(sd.DimensionMismatch):
        ns["pairwise_distances_gpu"](a, sd.from_dense(np.ones((2, 3))), sd.metric_registry("cosine"))


# ------------------------------------------------------------ CSR -> COO on device (sparse.py:220-225)

@pytest.mark.parametrize("shape", [(0, 5, 0.0), (7, 9, 0.0), (64, 300, 0.05), (513, 2000, 0.02)])
def test_csr_to_coo_device_matches_host(shape):
    """sd_csr_to_coo (coo_rows_kernel) against the reference's row expansion
    (np.repeat over the row degrees), empty rows and empty matrices included."""
    from paper_2104_06357_b200 import _lib
    m, k, dens = shape
    rng = np.random.default_rng(m + k)
    a = sd.from_dense(_random_dense(rng, m, k, dens)) if m else sd.from_dense(np.zeros((0, k)))
    d = sd.to_device(a, "float32")
    got = _lib.coo_rows(d).cpu().numpy()
    np.testing.assert_array_equal(got, np.asarray(a.coo_row_ids))
    np.testing.assert_array_equal(np.asarray(sd.csr_to_coo(a).rows), got)
