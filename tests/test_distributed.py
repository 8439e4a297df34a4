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
