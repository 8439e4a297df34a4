"""N > 1 orchestration on CPU: world_size-2 gloo process groups run the
sharded kNN flow (shard ranges, global index bases, all_gather, merge with
ties -> lower global index).  The local shard kernel and the merge are the
oracle here (injected through local_fn / merge_fn), so this exercises the
host-side logic only; the CUDA kernels are covered by tests/test_knn_gpu.py."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import knn as oknn
from paper_2206_14148_b200 import distributed


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _oracle_local(x, q, k, base):
    d, i = oknn.exact(x.numpy(), q.numpy(), min(k, x.shape[0]))
    return torch.from_numpy(d), torch.from_numpy(i + base)


def _oracle_merge(dl, il):
    L, m, k = dl.shape
    d = dl.permute(1, 0, 2).reshape(m, L * k).numpy()
    i = il.permute(1, 0, 2).reshape(m, L * k).numpy()
    od = np.empty((m, k))
    oi = np.empty((m, k), np.int64)
    for r in range(m):
        order = np.lexsort((i[r], d[r]))[:k]
        od[r], oi[r] = d[r, order], i[r, order]
    return torch.from_numpy(od), torch.from_numpy(oi)


def _worker(rank, world, port, x, q, k, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, e = distributed.shard_range(x.shape[0], rank, world)
        d, i = distributed.knn_sharded(torch.from_numpy(x[s:e]), torch.from_numpy(q), k,
                                       index_base=s, local_fn=_oracle_local,
                                       merge_fn=_oracle_merge)
        results[rank] = (d.numpy(), i.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_knn_matches_single(world):
    rng = np.random.default_rng(0)
    x = rng.standard_normal((1001, 6))
    x[500:520] = x[0:20]                       # duplicates straddling shard edges
    q = rng.standard_normal((25, 6))
    q[:5] = x[:5]
    ref_d, ref_i = oknn.exact(x, q, 7)
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, x, q, 7, results))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(world):
        d, i = results[r]
        assert np.array_equal(i, ref_i)
        assert np.allclose(d, ref_d, rtol=1e-12, atol=1e-12)


def test_shard_range_partitions():
    for n in (1, 7, 1000, 1_000_000):
        for w in (1, 2, 3, 8):
            if n < w:
                continue
            spans = [distributed.shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [e - s for s, e in spans]
            assert max(sizes) - min(sizes) <= 1


def _sgpr_worker(rank, world, port, X, y, Z, packed, results):
    """One rank of the SGPR N-split: this rank's rows -> local statistics
    (the fp64 oracle stands in for tb_sgpr_stats_run), then the product's
    allreduce_statistics, then the tail (oracle) on the reduced sums."""
    from oracle import sgpr as osgpr
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        s, e = distributed.shard_range(X.shape[0], rank, world)
        S, v, yy = osgpr.sufficient_stats(X[s:e], y[s:e], Z, "rbf", 1.3, 0.8)
        St = torch.from_numpy(S.reshape(-1).copy() if packed else S.copy())
        vt = torch.from_numpy(v.copy())
        yt = torch.tensor([yy], dtype=torch.float64)
        St, vt, yy_tot, n_tot = distributed.allreduce_statistics(St, vt, yt, e - s)
        S_tot = St.numpy().reshape(S.shape)
        bound, w = osgpr.elbo_from_stats(S_tot, vt.numpy(), yy_tot, n_tot,
                                         osgpr.kuu(Z, "rbf", 1.3, 0.8), 0.02, 1.3)
        results[rank] = (S_tot, vt.numpy().copy(), yy_tot, n_tot, bound, w)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,packed", [(2, False), (3, True)])
def test_sharded_sgpr_statistics_allreduce(world, packed):
    """SGPR at N > 1 (north star: per-rank partial M x M / M x 1 sums, one
    all_reduce, the tail on every rank): gloo world 2/3 through the same
    distributed.allreduce_statistics that SGPR(group=...) calls; every rank
    ends with the single-process statistics and ELBO.  ``packed`` reduces a
    flat buffer (the packed-tile layout is an elementwise sum too)."""
    from oracle import sgpr as osgpr
    from paper_2206_14148_b200 import synthetic
    X, y, Z, _ = synthetic.sgpr_data(1003, 3, 40, seed=21, dtype=np.float64)
    S_ref, v_ref, yy_ref = osgpr.sufficient_stats(X, y, Z, "rbf", 1.3, 0.8)
    e_ref, w_ref = osgpr.elbo(X, y, Z, "rbf", 1.3, 0.8, 0.02)
    ctx = mp.get_context("spawn")
    manager = ctx.Manager()
    results = manager.dict()
    port = _free_port()
    procs = [ctx.Process(target=_sgpr_worker, args=(r, world, port, X, y, Z, packed, results))
             for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    for r in range(world):
        S, v, yy, n, bound, w = results[r]
        assert n == X.shape[0]
        assert np.allclose(S, S_ref, rtol=1e-12, atol=1e-12 * np.abs(S_ref).max())
        assert np.allclose(v, v_ref, rtol=1e-12, atol=1e-12 * np.abs(v_ref).max())
        assert abs(yy - yy_ref) <= 1e-12 * yy_ref
        assert abs(bound - e_ref) <= 1e-9 * abs(e_ref)
        assert np.allclose(w, w_ref, rtol=1e-8, atol=1e-8 * np.abs(w_ref).max())
    # every rank holds bit-identical sums (the tail is redundant per rank)
    assert all(np.array_equal(results[0][0], results[r][0]) for r in range(world))
