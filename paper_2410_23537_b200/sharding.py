"""Multi-GPU partitioning of the hot path (one process per GPU, torch.distributed).

* KV swap: jobs are independent units.  ``lpt_assign`` places them on GPUs by
  longest-processing-time first on fp16 bytes; there is no collective on the data
  path.
* Predictor: the query DB is row-sharded by insert sequence, ``seq % G == rank``.
  With a global capacity ``G * local_capacity`` each shard's FIFO ring evicts exactly
  the rows the single global ring (predictor.py:138) would.  A batched search has two
  exchange steps over NCCL (NVLink): after the per-shard coarse scan, a max
  all-reduce of the per-query exact-score lower bounds (B floats) lets every shard
  rescore only rows that can still enter the global top-k; then the per-shard (sim,
  seq, len, count) records are all-gathered and merged by (-sim, seq).
"""
from __future__ import annotations

import numpy as np


def lpt_assign(weights, n_bins: int) -> list:
    """Longest-processing-time-first: jobs sorted by weight (desc, then index) go to the
    least-loaded bin (lowest index on ties).  Returns per-bin sorted job indices."""
    order = sorted(range(len(weights)), key=lambda i: (-weights[i], i))
    loads = [0] * n_bins
    bins = [[] for _ in range(n_bins)]
    for i in order:
        b = min(range(n_bins), key=lambda j: (loads[j], j))
        bins[b].append(i)
        loads[b] += weights[i]
    return [sorted(b) for b in bins]


def shard_rows(seqs, rank: int, world: int):
    """Mask of the rows (by global insert sequence) owned by `rank`."""
    return (np.asarray(seqs) % world) == rank


def merge_topk_host(sims, seqs, lens, counts, k: int):
    """Reference merge of G per-shard sorted lists ([G,B,k] arrays) by (-sim, seq).
    Host restatement of the k_topk_merge kernel, used by the CPU multi-process tests."""
    sims, seqs, lens, counts = map(np.asarray, (sims, seqs, lens, counts))
    G, B, _ = sims.shape
    o_sim = np.zeros((B, k))
    o_seq = np.zeros((B, k), np.int64)
    o_len = np.zeros((B, k), np.int32)
    o_cnt = np.zeros(B, np.int32)
    for q in range(B):
        items = [(-sims[g, q, i], seqs[g, q, i], lens[g, q, i]) for g in range(G) for i in range(counts[g, q])]
        items.sort(key=lambda t: (t[0], t[1]))
        items = items[:k]
        o_cnt[q] = len(items)
        for i, (ns, sq, ln) in enumerate(items):
            o_sim[q, i], o_seq[q, i], o_len[q, i] = -ns, sq, ln
    return o_sim, o_seq, o_len, o_cnt


def all_gather_records(local, group=None):
    """All-gather a tuple of equally shaped per-rank tensors; returns [G, ...] stacks."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    nccl = dist.get_backend(group) == "nccl"
    out = []
    for t in local:
        t = t.contiguous()
        buf = torch.empty((world,) + tuple(t.shape), dtype=t.dtype, device=t.device)
        if nccl:
            dist.all_gather_into_tensor(buf, t, group=group)
        else:  # gloo (multi-process tests; CUDA tensors are staged through the host)
            tc = t.cpu()
            parts = [torch.empty_like(tc) for _ in range(world)]
            dist.all_gather(parts, tc, group=group)
            buf.copy_(torch.stack(parts))
        out.append(buf)
    return out


def all_reduce_max(t, group=None):
    """In-place max all-reduce of a CUDA tensor (NCCL; gloo stages through the host)."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    else:
        tc = t.cpu()
        dist.all_reduce(tc, op=dist.ReduceOp.MAX, group=group)
        t.copy_(tc)
    return t


class ShardedVectorStore:
    """A VectorStore sharded over the ranks of a process group (one GPU each).

    ``add_batch`` takes the full batch of new records on every rank (as the serving
    frontend broadcasts them) and keeps this rank's residue class.  ``search_batch``
    returns the global exact top-k on every rank.
    """

    def __init__(self, dimension: int, capacity: int, group=None):
        import torch.distributed as dist

        from . import _lib
        from .predictor import VectorStore
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        if capacity % self.world:
            raise ValueError("capacity must be a multiple of the shard count for exact FIFO semantics")
        self.dimension = dimension
        self.capacity = capacity
        self.local = VectorStore(dimension, capacity // self.world)
        _lib.call("alise_db_set_seq_stride", self.local._h, self.world)
        self.next_seq = 0

    @property
    def size(self) -> int:
        return min(self.next_seq, self.capacity)

    def __len__(self):
        return self.size

    def add_batch(self, vectors, lens):
        import torch

        from . import _lib
        vectors = np.asarray(vectors) if not isinstance(vectors, torch.Tensor) else vectors
        n = len(lens)
        seqs = np.arange(self.next_seq, self.next_seq + n, dtype=np.int64)
        mine = np.flatnonzero(shard_rows(seqs, self.rank, self.world))
        loc = self.local
        if len(mine):
            dev = loc._dev()
            v = torch.as_tensor(vectors[mine] if not isinstance(vectors, torch.Tensor)
                                else vectors[torch.as_tensor(mine)])
            v = v.to(dev, torch.float32).contiguous()
            ln = torch.as_tensor(np.asarray(lens)[mine]).to(dev, torch.int32).contiguous()
            sq = torch.as_tensor(seqs[mine]).to(dev)
            cap = loc.capacity
            for c0 in range(0, len(mine), cap):
                c1 = min(len(mine), c0 + cap)
                _lib.call("alise_db_append", loc._h, _lib.ptr(v[c0:c1]), _lib.ptr(ln[c0:c1]),
                          _lib.ptr(sq[c0:c1]), c1 - c0, _lib.stream_ptr())
            loc.next_seq += len(mine)
            loc.size = min(cap, loc.size + len(mine))
        self.next_seq += n

    def search_batch(self, queries, k: int):
        """Global exact top-k: local tcgen05 scan + exact rescoring, NCCL all-gather of
        the per-shard records, (-sim, seq) merge.  Returns CUDA tensors."""
        import torch

        from . import _lib
        dev = self.local._dev()
        q = torch.as_tensor(queries if isinstance(queries, torch.Tensor) else np.asarray(queries))
        q = q.to(dev, torch.float32).reshape(-1, self.dimension).contiguous()
        B = q.shape[0]
        # scan, all-reduce (max) of the per-query coarse k-th lower bounds, then exact
        # rescoring of only the rows that can still enter the global top-k
        sims = torch.zeros((B, k), dtype=torch.float64, device=dev)
        seqs = torch.zeros((B, k), dtype=torch.int64, device=dev)
        lens = torch.zeros((B, k), dtype=torch.int32, device=dev)
        cnt = torch.zeros(B, dtype=torch.int32, device=dev)
        bound = torch.empty(B, dtype=torch.float32, device=dev)
        h = self.local._h
        _lib.call("alise_db_topk_scan", h, _lib.ptr(q), B, k, _lib.ptr(bound), _lib.stream_ptr())
        all_reduce_max(bound, self.group)
        _lib.call("alise_db_topk_rescore", h, _lib.ptr(q), B, k, _lib.ptr(bound), _lib.ptr(sims), _lib.ptr(seqs),
                  _lib.ptr(lens), _lib.ptr(cnt), _lib.stream_ptr())
        g_sims, g_seqs, g_lens, g_cnt = all_gather_records((sims, seqs, lens, cnt), self.group)
        o_sim = torch.empty((B, k), dtype=torch.float64, device=dev)
        o_seq = torch.empty((B, k), dtype=torch.int64, device=dev)
        o_len = torch.empty((B, k), dtype=torch.int32, device=dev)
        o_cnt = torch.empty(B, dtype=torch.int32, device=dev)
        _lib.call("alise_topk_merge", self.world, B, k, _lib.ptr(g_sims), _lib.ptr(g_seqs), _lib.ptr(g_lens),
                  _lib.ptr(g_cnt), _lib.ptr(o_sim), _lib.ptr(o_seq), _lib.ptr(o_len), _lib.ptr(o_cnt),
                  _lib.stream_ptr())
        return o_sim, o_seq, o_len, o_cnt, q
