"""Multi-GPU partitioning of the hot path (one process per GPU, torch.distributed).

* KV swap: jobs are independent units.  ``lpt_assign`` places them on GPUs by
  longest-processing-time first on fp16 bytes; there is no collective on the data
  path.
* Predictor, ``layout="rows"``: the query DB is row-sharded by insert sequence,
  ``seq % G == rank``.  With a global capacity ``G * local_capacity`` each shard's FIFO
  ring evicts exactly the rows the single global ring (predictor.py:138) would.  A
  batched search has two exchange steps over NCCL (NVLink): after the per-shard coarse
  scan, a max all-reduce of the per-query exact-score lower bounds (B floats) lets
  every shard rescore only rows that can still enter the global top-k; then the
  per-shard (sim, seq, len, count) records are all-gathered and merged by (-sim, seq).
* Predictor, ``layout="queries"``: every rank holds the whole DB (C4's 1M x 768 is
  4.6 GB of a 180 GB GPU) and searches a contiguous slice of the batch's queries; the
  data path has no collective (``search_batch_local``), the drop-in ``search_batch``
  all-gathers the slices' records.  Per-rank work is the full DB against B/G queries.
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


def _gather_objects(obj, group=None):
    """All-gather of small host objects (snapshots, refit data; not the hot path)."""
    import torch.distributed as dist
    out = [None] * dist.get_world_size(group)
    dist.all_gather_object(out, obj, group=group)
    return out


class ShardedVectorStore:
    """A VectorStore sharded over the ranks of a process group (one GPU each); a drop-in
    for ``VectorStore`` (predictor.py:120-189) on every rank.

    Every rank calls every method with the same arguments (the serving front-end
    broadcasts new records and query batches): ``add`` / ``add_batch`` keep this
    rank's residue class ``seq % G``; ``search`` / ``search_batch`` return the global
    exact top-k on every rank; ``newest`` / ``export`` / ``save`` gather the shards;
    ``save_binary`` / ``load_binary`` snapshot each shard on its own rank and restore
    the global FIFO (same sequence numbers, slots and next_seq).
    """

    LAYOUTS = ("rows", "queries")

    def __init__(self, dimension: int, capacity: int, group=None, dtype=np.float64, order: str = "exact",
                 blas_threads: int | None = None, layout: str = "rows"):
        import torch.distributed as dist

        from . import _lib
        from .predictor import VectorStore
        if layout not in self.LAYOUTS:
            raise ValueError(f"layout must be one of {self.LAYOUTS}")
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.layout = layout
        self.replicated = layout == "queries"
        if not self.replicated and capacity % self.world:
            raise ValueError("capacity must be a multiple of the shard count for exact FIFO semantics")
        self.dimension = dimension
        self.capacity = capacity
        self.dtype = np.dtype(dtype)
        local_cap = capacity if self.replicated else capacity // self.world
        self.local = VectorStore(dimension, local_cap, dtype=dtype, order=order, blas_threads=blas_threads)
        if not self.replicated:
            _lib.call("alise_db_set_seq_stride", self.local._h, self.world)
        self.order = order
        self.next_seq = 0

    @property
    def size(self) -> int:
        return min(self.next_seq, self.capacity)

    def __len__(self):
        return self.size

    def add(self, vector, observed_len: int) -> int:
        """VectorStore.add (predictor.py:135-152): the owner rank appends the record."""
        from .predictor import PredictorError
        if observed_len < 1:
            raise PredictorError("observed_len must be >= 1")
        if self.replicated:  # every rank appends (pinned staging ring, no host sync)
            self.next_seq = self.local.add(vector, observed_len) + 1
            return self.next_seq - 1
        seq = self.next_seq
        self.add_batch(np.asarray(vector, dtype=np.float64)[None, :], [int(observed_len)])
        return seq

    def add_batch(self, vectors, lens, stream=None, seqs=None):
        """Append a batch in insert order; this rank keeps its residue class.  ``seqs``
        (host, increasing) restores records under their original sequence numbers."""
        import torch

        from .predictor import PredictorError, _host_lens
        hl = _host_lens(lens)
        if hl is None:
            hl = lens.cpu().numpy().astype(np.int64).reshape(-1)
        n = len(hl)
        if n and hl.min() < 1:
            raise PredictorError("observed_len must be >= 1")
        if self.replicated:
            self.local.add_batch(vectors, hl if hl is not None else lens, stream=stream, seqs=seqs)
            self.next_seq = self.local.next_seq
            return self.next_seq - 1
        if seqs is None:
            seqs = np.arange(self.next_seq, self.next_seq + n, dtype=np.int64)
        else:
            seqs = np.asarray(seqs, dtype=np.int64).reshape(-1)
        mine = np.flatnonzero(shard_rows(seqs, self.rank, self.world))
        if len(mine):
            if isinstance(vectors, torch.Tensor):
                v = vectors[torch.as_tensor(mine, device=vectors.device)]
            else:
                v = np.asarray(vectors)[mine]
            self.local.add_batch(v, hl[mine], stream=stream, seqs=seqs[mine])
        if n:
            self.next_seq = int(seqs[-1]) + 1
        return self.next_seq - 1

    def query_slice(self, B: int):
        """This rank's rows [lo, hi) of a B-query batch (layout "queries": equal slices of
        ceil(B / G), the last ones shorter or empty)."""
        per = -(-B // self.world)
        lo = min(B, self.rank * per)
        return lo, min(B, lo + per)

    def search_batch_local(self, queries, k: int, stream=None):
        """Layout "queries": the exact top-k of this rank's query slice over the whole
        (replicated) DB -- no collective.  Returns (lo, hi, VectorStore.search_batch of
        rows lo..hi)."""
        if not self.replicated:
            raise ValueError('search_batch_local needs layout="queries"')
        q = self.local._as_rows(queries)
        lo, hi = self.query_slice(q.shape[0])
        return lo, hi, self.local.search_batch(q[lo:hi], k, stream=stream)

    def search_batch(self, queries, k: int, stream=None):
        """Global exact top-k.  Layout "rows": local tcgen05 scan, NCCL max all-reduce of
        the per-query exact-score lower bounds, exact rescoring of the rows that can still
        enter the global top-k, NCCL all-gather of the per-shard records, (-sim, seq)
        merge.  Layout "queries": each rank searches its query slice over the whole DB
        and the slices' records are all-gathered.  Returns CUDA tensors like
        VectorStore.search_batch."""
        import torch

        from . import _lib
        from .predictor import MAX_K, PredictorError
        if k < 1 or k > MAX_K:
            raise PredictorError(f"k must be in [1, {MAX_K}]")
        dev = self.local._dev()
        q = self.local._as_rows(queries)
        B = q.shape[0]
        if self.replicated:
            per = -(-B // self.world)
            lo, hi = self.query_slice(B)
            cur = torch.cuda.current_stream(dev) if stream is None else stream
            with torch.cuda.stream(cur):
                part = [torch.zeros((per, k), dtype=torch.float64, device=dev),
                        torch.zeros((per, k), dtype=torch.int64, device=dev),
                        torch.zeros((per, k), dtype=torch.int32, device=dev),
                        torch.zeros(per, dtype=torch.int32, device=dev)]
                if hi > lo:
                    r = self.local.search_batch(q[lo:hi], k, stream=stream)
                    for dst, src in zip(part, r[:4]):
                        dst[: hi - lo].copy_(src)
                g = all_gather_records(part, self.group)
            return tuple(t.reshape((self.world * per,) + tuple(t.shape[2:]))[:B] for t in g) + (q,)
        sp = _lib.stream_ptr(stream)
        sims = torch.zeros((B, k), dtype=torch.float64, device=dev)
        seqs = torch.zeros((B, k), dtype=torch.int64, device=dev)
        lens = torch.zeros((B, k), dtype=torch.int32, device=dev)
        cnt = torch.zeros(B, dtype=torch.int32, device=dev)
        bound = torch.empty(B, dtype=torch.float32, device=dev)
        h = self.local._h
        if self.order == "blas":  # rows are numbered by the global ring (predictor.py:138)
            self.local.set_order("blas", self.local.blas_threads, self.capacity, self.size)
        cur = torch.cuda.current_stream(dev) if stream is None else stream
        with torch.cuda.stream(cur):
            _lib.call("alise_db_topk_scan", h, _lib.ptr(q), B, k, _lib.ptr(bound), sp)
            all_reduce_max(bound, self.group)
            _lib.call("alise_db_topk_rescore", h, _lib.ptr(q), B, k, _lib.ptr(bound), _lib.ptr(sims),
                      _lib.ptr(seqs), _lib.ptr(lens), _lib.ptr(cnt), sp)
            g_sims, g_seqs, g_lens, g_cnt = all_gather_records((sims, seqs, lens, cnt), self.group)
            o_sim = torch.empty((B, k), dtype=torch.float64, device=dev)
            o_seq = torch.empty((B, k), dtype=torch.int64, device=dev)
            o_len = torch.empty((B, k), dtype=torch.int32, device=dev)
            o_cnt = torch.empty(B, dtype=torch.int32, device=dev)
            _lib.call("alise_topk_merge", self.world, B, k, _lib.ptr(g_sims), _lib.ptr(g_seqs), _lib.ptr(g_lens),
                      _lib.ptr(g_cnt), _lib.ptr(o_sim), _lib.ptr(o_seq), _lib.ptr(o_len), _lib.ptr(o_cnt), sp)
        return o_sim, o_seq, o_len, o_cnt, q

    def search(self, vector, k: int):
        """VectorStore.search (predictor.py:154-163) over all shards."""
        if self.size == 0:
            return np.array([]), np.array([], dtype=np.int64), np.array([], dtype=np.int64)
        k = min(k, self.size)
        sims, seqs, lens, cnt, _ = self.search_batch(np.asarray(vector, dtype=np.float64)[None, :], k)
        c = int(cnt[0].item())
        return (sims[0, :c].cpu().numpy(), lens[0, :c].cpu().numpy().astype(np.int64),
                seqs[0, :c].cpu().numpy())

    def export(self):
        """All live records of all shards on every rank: (vectors f64, lens, seqs) in
        insert order."""
        if self.replicated:
            vecs, lens, seqs = self.local.export()
            order = np.argsort(seqs, kind="stable")
            return vecs[order].reshape(-1, self.dimension), lens[order].astype(np.int64), seqs[order]
        parts = _gather_objects(self.local.export(), self.group)
        vecs = np.concatenate([p[0] for p in parts]) if parts else np.zeros((0, self.dimension))
        lens = np.concatenate([p[1] for p in parts]).astype(np.int64)
        seqs = np.concatenate([p[2] for p in parts]).astype(np.int64)
        order = np.argsort(seqs, kind="stable")
        return vecs[order].reshape(-1, self.dimension), lens[order], seqs[order]

    def newest(self, count: int):
        """Vectors and lengths of the most recently inserted records (predictor.py:165-168)."""
        if self.replicated:
            if count <= 0:
                return np.zeros((0, self.dimension)), np.zeros(0, np.int64)
            return self.local.newest(count)
        vecs, lens, seqs = self.local.export()
        keep = np.argsort(seqs)[-count:] if count > 0 else np.zeros(0, np.int64)
        parts = _gather_objects((vecs[keep], lens[keep], seqs[keep]), self.group)
        vecs = np.concatenate([p[0] for p in parts]).reshape(-1, self.dimension)
        lens = np.concatenate([p[1] for p in parts]).astype(np.int64)
        seqs = np.concatenate([p[2] for p in parts]).astype(np.int64)
        order = np.argsort(seqs)[-count:] if count > 0 else np.zeros(0, np.int64)
        return vecs[order], lens[order]

    def save(self, path):
        """JSON-lines snapshot (predictor.py:170-178), written by rank 0."""
        import json
        vecs, lens, seqs = self.export()
        if self.rank == 0:
            with open(path, "w") as fh:
                for i in range(len(seqs)):
                    fh.write(json.dumps({"seq": int(seqs[i]), "len": int(lens[i]),
                                         "vector": [float(x) for x in vecs[i]]}) + "\n")

    @classmethod
    def load(cls, path, dimension: int, capacity: int, group=None, dtype=np.float64,
             layout: str = "rows") -> "ShardedVectorStore":
        """predictor.py:180-189: re-adds the records in file order (new seqs from 0)."""
        import json
        vecs, lens = [], []
        with open(path) as fh:
            for line in fh:
                line = line.strip()
                if line:
                    rec = json.loads(line)
                    vecs.append(rec["vector"])
                    lens.append(int(rec["len"]))
        store = cls(dimension, capacity, group=group, dtype=dtype, layout=layout)
        if vecs:
            store.add_batch(np.asarray(vecs, dtype=np.float64), lens)
        return store

    def shard_path(self, path) -> str:
        return f"{path}.shard{self.rank}of{self.world}.npz"

    def save_binary(self, path):
        """Per-shard binary snapshot: each rank writes its own records (master dtype,
        original sequence numbers) and the global next_seq to ``shard_path(path)``."""
        vecs, lens, seqs = self.local.export()
        order = np.argsort(seqs)
        np.savez(self.shard_path(path), vectors=vecs[order].astype(self.dtype), lens=lens[order],
                 seqs=seqs[order], dimension=self.dimension, capacity=self.capacity, world=self.world,
                 rank=self.rank, next_seq=self.next_seq, layout=self.layout)

    @classmethod
    def load_binary(cls, path, group=None) -> "ShardedVectorStore":
        """Restore a save_binary snapshot on the same number of ranks: every shard gets
        its records back under their sequence numbers (same slots, global FIFO order
        and next_seq), so searches and later evictions equal the saved store's."""
        import torch.distributed as dist
        world, rank = dist.get_world_size(group), dist.get_rank(group)
        z = np.load(f"{path}.shard{rank}of{world}.npz")
        if int(z["world"]) != world or int(z["rank"]) != rank:
            raise ValueError("snapshot was written by a different shard layout")
        layout = str(z["layout"]) if "layout" in z.files else "rows"
        store = cls(int(z["dimension"]), int(z["capacity"]), group=group, dtype=z["vectors"].dtype, layout=layout)
        if len(z["lens"]):
            store.local.add_batch(z["vectors"], z["lens"], seqs=z["seqs"])
        store.next_seq = int(z["next_seq"])
        if store.replicated:
            store.local.next_seq = store.next_seq
        return store
