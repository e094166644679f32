"""Multi-process (world_size 2, gloo, CPU) coverage of the sharded paths'
host logic: shard planning, the candidate all-gather and the merge order.
The per-rank compute here is the oracle (no GPU in this container); on a GPU
box the same functions run the fused kernels and NCCL (tests/test_gpu_parity)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import semidist_oracle as O
from paper_2104_06357_b200.distributed import gather_candidates, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _merge_cpu(cd, ci, k):
    """Reference merge: lexicographic (distance, index), NaN last — what sd_topk_merge computes."""
    lists, m, _ = cd.shape
    out_d = np.empty((m, k))
    out_i = np.empty((m, k), dtype=np.int64)
    for q in range(m):
        d = cd[:, q, :].reshape(-1)
        i = ci[:, q, :].reshape(-1)
        order = np.lexsort((i, np.where(np.isnan(d), np.inf, d), np.isnan(d)))[:k]
        out_d[q], out_i[q] = d[order], i[order]
    return out_d, out_i


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(7)
        dense = np.where(rng.random((90, 40)) < 0.2, rng.uniform(0.1, 1.0, (90, 40)), 0.0)
        index = O.csr_of_dense(dense)
        queries = O.csr_of_dense(dense[:17])
        k = 6
        lo, hi = shard_bounds(index.n_rows, world)[rank]
        shard = index.slice(lo, hi)
        full = O.pairwise_distances(queries, shard, "manhattan")
        order = np.argsort(full, axis=1, kind="stable")[:, :k]
        ld = torch.from_numpy(np.take_along_axis(full, order, 1).copy())
        li = torch.from_numpy((order + lo).astype(np.int64))
        cd, ci = gather_candidates(ld, li)
        md, mi = _merge_cpu(cd.numpy(), ci.numpy(), k)
        # pairwise: query-row shards, no collective; gather only for the check
        plo, phi = shard_bounds(queries.n_rows, world)[rank]
        block = torch.from_numpy(O.pairwise_distances(queries.slice(plo, phi), index, "cosine"))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([block.shape[0]]))
        rows = max(int(s.item()) for s in sizes)   # gloo gathers equal shapes: pad, then trim
        padded = torch.zeros((rows, index.n_rows), dtype=block.dtype)
        padded[:block.shape[0]] = block
        blocks = [torch.zeros_like(padded) for _ in range(world)]
        dist.all_gather(blocks, padded)
        full = torch.cat([b[:int(s.item())] for b, s in zip(blocks, sizes)])
        if rank == 0:
            q.put((md, mi, full.numpy()))
    finally:
        dist.destroy_process_group()


def test_knn_shard_gather_merge_equals_global():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    md, mi, pw = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    rng = np.random.default_rng(7)
    dense = np.where(rng.random((90, 40)) < 0.2, rng.uniform(0.1, 1.0, (90, 40)), 0.0)
    index = O.csr_of_dense(dense)
    queries = O.csr_of_dense(dense[:17])
    ref_d, ref_i = O.kneighbors(index, queries, 6, "manhattan")
    np.testing.assert_array_equal(mi, ref_i)
    np.testing.assert_array_equal(md, ref_d)
    np.testing.assert_array_equal(pw, O.pairwise_distances(queries, index, "cosine"))


def test_shard_bounds_cover_and_balance():
    for n, w in [(0, 2), (1, 4), (10, 3), (1000, 8)]:
        b = shard_bounds(n, w)
        assert b[0][0] == 0 and b[-1][1] == n
        assert all(b[r][1] == b[r + 1][0] for r in range(w - 1))
    weights = np.array([100.0] + [1.0] * 99)
    b = shard_bounds(100, 2, weights)
    assert b[0] == (0, 1) or b[0][1] <= 2   # the heavy row gets (nearly) its own shard
    with pytest.raises(ValueError):
        shard_bounds(5, 0)
