"""Multi-GPU partitioner: one process per GPU, N sharded across ranks.

The reference has no distributed execution.  The north star
shards the data axis N over one 8xB200 box:

* kNN  — rank g owns database rows [start_g, stop_g) (``shard_range``) and
  reports global indices via ``index_base = start_g``.  Each rank returns its
  exact fp64 top-k; one NCCL ``all_gather`` over NVLink exchanges the
  [m, k] lists (m*k*16 B per rank: 1.6 MB at m=1e4, k=10) and
  ``tb_topk_merge`` merges them with ties -> lower global index.  Because
  every shard's list is exact, the merge is exact and independent of the
  shard count.
* SGPR — rank g owns N/G training rows; Sigma, v, yy are summed with one
  ``all_reduce`` (see ``sgpr.sgpr_elbo(group=...)``).

``local_fn`` / ``merge_fn`` hooks exist so the orchestration can be tested
with the gloo backend on CPU (tests/test_distributed.py); the product path
uses the CUDA library for both.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib


def _torch():
    import torch
    return torch


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """np.array_split boundaries: the first n % world shards get one extra row."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def merge_topk(dist_lists, idx_lists, stream=None):
    """[L, m, k] per-shard ascending lists -> global [m, k] (CUDA tensors)."""
    torch = _torch()
    L, m, k = (int(v) for v in dist_lists.shape)
    dl = dist_lists.contiguous()
    il = idx_lists.to(torch.int64).contiguous()
    od = torch.empty((m, k), dtype=dl.dtype, device=dl.device)
    oi = torch.empty((m, k), dtype=torch.int64, device=dl.device)
    st = stream if stream is not None else torch.cuda.current_stream(dl.device)
    dt = _lib.TB_F32 if dl.dtype == torch.float32 else _lib.TB_F64
    rc = _lib.load().tb_topk_merge(dl.data_ptr(), il.data_ptr(), L, m, k, dt,
                                   od.data_ptr(), oi.data_ptr(), st.cuda_stream)
    _lib.check(rc, "topk_merge")
    return od, oi


def knn_sharded(x_shard, q, k: int, *, index_base: int, group=None, operator=None,
                memory_limit=None, engine: str = "auto", local_fn=None, merge_fn=None,
                out_dtype=None, events=None):
    """Global kNN over a database sharded across the ranks of ``group``.

    Every rank passes its own shard and the full query set; every rank
    receives the global (dist[m,k], idx[m,k]).  Shards must hold >= k rows.
    ``events`` (optional torch.cuda.Event pairs) time this rank's candidate
    engine launches, as in ``KnnOperator.run``.
    """
    torch = _torch()
    import torch.distributed as dist

    if local_fn is None:
        if operator is None:
            from .neighbors import KnnOperator
            operator = KnnOperator(int(x_shard.shape[0]), int(q.shape[0]),
                                   int(q.shape[1]), k, dtype=_np_dtype(x_shard),
                                   out_dtype=np.float64, engine=engine,
                                   memory_limit=memory_limit)
        d, i = operator.run(x_shard, q, index_base=index_base, events=events)
    else:
        d, i = local_fn(x_shard, q, k, index_base)
    world = dist.get_world_size(group)
    if world == 1:
        dl, il = d.unsqueeze(0), i.unsqueeze(0)
    else:
        dl = torch.empty((world,) + tuple(d.shape), dtype=d.dtype, device=d.device)
        il = torch.empty((world,) + tuple(i.shape), dtype=i.dtype, device=i.device)
        dist.all_gather(list(dl.unbind(0)), d.contiguous(), group=group)
        dist.all_gather(list(il.unbind(0)), i.contiguous(), group=group)
    od, oi = (merge_fn or merge_topk)(dl, il)
    if out_dtype is not None:
        od = od.to(_torch_dtype(out_dtype))
    return od, oi


def knn_sharded_host(xh_shard, qh, k: int, *, index_base: int, operator, group=None,
                     staging=None, out_host=None):
    """knn_sharded from HOST buffers: this rank's database shard and the
    queries are copied in through ``operator.run_host`` (tb_knn_run_host,
    chunk copies overlapped with compute), the per-shard lists are exchanged
    on the device (all_gather + tb_topk_merge) and the global (dist, idx)
    is copied back into pinned host tensors.  ``operator`` must be planned
    for this shard with fp64 output (exact ties across shards)."""
    torch = _torch()
    if staging is None:
        p = operator.plan
        td = torch.float32 if operator.dtype == np.float32 else torch.float64
        staging = (torch.empty((int(p.n), int(p.d)), dtype=td, device=operator.device),
                   torch.empty((int(p.m), int(p.d)), dtype=td, device=operator.device),
                   *operator.alloc_outputs())
    dd, idd = staging[2], staging[3]
    # the per-shard host copy of tb_knn_run_host is not used (the lists meet
    # on the device); its pinned buffers are made once per operator, not per
    # call (a pinned allocation costs far more than the copy)
    cached = getattr(operator, "_shard_host_out", None)
    if cached is None or tuple(cached[0].shape) != tuple(dd.shape) or cached[0].dtype != dd.dtype:
        cached = (torch.empty(tuple(dd.shape), dtype=dd.dtype).pin_memory(),
                  torch.empty(tuple(idd.shape), dtype=torch.int64).pin_memory())
        operator._shard_host_out = cached
    dh_local, ih_local = cached

    def local(_x, _q, _k, base):
        operator.run_host(xh_shard, qh, (dh_local, ih_local), index_base=base,
                          staging=staging, synchronize=False)
        return dd, idd

    od, oi = knn_sharded(None, None, k, index_base=index_base, group=group, local_fn=local)
    if out_host is None:
        out_host = (torch.empty(tuple(od.shape), dtype=od.dtype).pin_memory(),
                    torch.empty(tuple(oi.shape), dtype=torch.int64).pin_memory())
    out_host[0].copy_(od, non_blocking=True)
    out_host[1].copy_(oi, non_blocking=True)
    torch.cuda.current_stream(od.device).synchronize()
    return out_host


def allreduce_statistics(Sigma, v, yy, n_local: int, group=None):
    """Sum per-rank SGPR sufficient statistics over ``group`` (the north
    star's N-split: each rank streams its own training rows).  ``Sigma`` is
    reduced in place in whatever layout the rank's plan produced (full
    [M, M] or packed lower tiles: an elementwise sum either way, and every
    rank's plan has the same layout because M and the engine are shared);
    v, yy and the row count travel together in one small fp64 buffer.
    Returns (Sigma, v, yy: float, N_total: int).  The fixed order of a ring
    or tree sum is deterministic for a given world size and backend."""
    torch = _torch()
    import torch.distributed as dist

    small = torch.empty(v.numel() + 2, dtype=torch.float64, device=v.device)
    small[:v.numel()].copy_(v.reshape(-1))
    small[v.numel()] = yy if not torch.is_tensor(yy) else yy.reshape(-1)[0]
    small[v.numel() + 1] = float(n_local)
    dist.all_reduce(Sigma, group=group)
    dist.all_reduce(small, group=group)
    v.reshape(-1).copy_(small[:v.numel()])
    return Sigma, v, float(small[v.numel()].item()), int(round(float(small[-1].item())))


def _np_dtype(t):
    torch = _torch()
    return np.float32 if t.dtype == torch.float32 else np.float64


def _torch_dtype(dt):
    torch = _torch()
    return torch.float32 if np.dtype(dt) == np.float32 else torch.float64
