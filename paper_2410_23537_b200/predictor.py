"""Drop-in for ``servesim.predictor`` with a B200 retrieval path.

Reference: /root/reference/pkg/src/servesim/predictor.py.  Same names, argument
meanings and errors.  The hot path — ``VectorStore.search`` (predictor.py:154-163)
and ``LengthPredictor.predict_vector`` (predictor.py:311-325) — runs on the GPU:

* the store is a device FIFO ring (float64 master like the reference, or fp32 for
  fp32 embedding DBs; plus an fp16 coarse copy; slot = seq % cap);
* ``search`` / ``search_batch`` compute the exact top-k by (-sim, seq): a tcgen05
  fp16 coarse scan with a provable candidate margin, then correctly rounded float64
  rescoring of the candidates (sims are the exact dot products of the stored
  vectors, rounded once to float64);
* ``predict_batch`` fuses the aggregate (numpy's summation order, half-even
  rounding) with the float64 all-MLP fallback in one kernel, reading the query in
  its own precision.

With the default float64 store the vectors, ``newest`` (the refit data) and the MLP
inputs are the reference's own float64 values; sims are correctly rounded where the
reference's BLAS dot may differ in the last bit, so results equal the restated oracle
(oracle/pred_oracle.py) exactly and the reference wherever its BLAS rounding does not
flip a threshold or a tie.

Training of the fallback regressor (``FallbackRegressor.fit``, predictor.py:221-264)
and the hashing embedder (predictor.py:66-100) are host-side producers of weights /
query vectors, outside the hot path; they are provided here so the module is a
complete drop-in.
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass

import numpy as np

from . import _lib

_FNV_OFFSET = 0xCBF29CE484222325
_FNV_PRIME = 0x100000001B3
_MASK64 = 0xFFFFFFFFFFFFFFFF
FALLBACK_INIT = 4  # rng.py stream tag
RETRIEVED = "retrieved"
FALLBACK = "fallback"
MAX_K = 1024  # k <= 16: tcgen05 scan path; 16 < k <= 1024: CUDA-core coarse pass (alise_db_topk)


class PredictorError(ValueError):
    pass


def _stream(seed: int, tag: int, *sub: int) -> np.random.Generator:
    """The reference's seeded PCG64 streams (rng.py:20-22)."""
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, tag, *sub])))


@dataclass
class PredictorConfig:
    """predictor.py:38-63."""

    dimension: int = 64
    top_k: int = 8
    similarity_threshold: float = 0.80
    db_capacity: int = 100_000
    max_len: int = 2048
    fallback_hidden: int = 32
    fallback_epochs: int = 150
    fallback_learning_rate: float = 0.05
    allow_untrained: bool = True
    online_refit: bool = True
    refit_epochs: int = 40
    refit_sample_cap: int = 256

    def validate(self):
        checks = [
            (self.dimension >= 1, "dimension must be >= 1"),
            (self.top_k >= 1, "top_k must be >= 1"),
            (self.db_capacity >= self.top_k, "db_capacity must be >= top_k"),
            (-1.0 <= self.similarity_threshold <= 1.0, "similarity_threshold must be in [-1, 1]"),
            (self.max_len >= 1, "max_len must be >= 1"),
        ]
        for ok, msg in checks:
            if not ok:
                raise PredictorError(msg)
        if self.top_k > MAX_K:
            raise PredictorError(f"top_k must be <= {MAX_K}")


def _fnv1a(data: bytes) -> int:
    h = _FNV_OFFSET
    for byte in data:
        h = ((h ^ byte) * _FNV_PRIME) & _MASK64
    return h


class HashingEmbedder:
    """Unigram + bigram FNV-1a feature hashing, L2-normalised (predictor.py:66-100)."""

    def __init__(self, dimension: int = 64):
        if dimension < 1:
            raise PredictorError("dimension must be >= 1")
        self.dimension = dimension

    def embed(self, tokens) -> np.ndarray:
        seq = [int(t) for t in (tokens if tokens is not None else [])]
        if not seq:
            raise PredictorError("cannot embed an empty token sequence")
        v = np.zeros(self.dimension)
        feats = [f"u:{t}" for t in seq] + [f"b:{a}:{b}" for a, b in zip(seq, seq[1:])]
        order = []
        for i, t in enumerate(seq):  # reference interleaves u:t_i then b:t_{i-1}:t_i
            order.append(feats[i])
            if i:
                order.append(feats[len(seq) + i - 1])
        for f in order:
            h = _fnv1a(f.encode())
            v[h % self.dimension] += 1.0 if (h >> 63) & 1 else -1.0
        n = float(np.linalg.norm(v))
        if n == 0.0:
            v[0], n = 1.0, 1.0
        return v / n

    def embed_batch(self, prompts, dtype=None, stream=None):
        """Embed many prompts on the GPU (alise_embed_batch); bit-identical to ``embed``.
        Returns a CUDA tensor [B, dimension] (float64 by default, or float32)."""
        import torch
        lens = [len(p) for p in prompts]
        if any(n == 0 for n in lens):
            raise PredictorError("cannot embed an empty token sequence")
        _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device())
        flat = torch.tensor([int(t) for p in prompts for t in p], dtype=torch.int64)
        offs = torch.tensor(np.concatenate([[0], np.cumsum(lens)]), dtype=torch.int64)
        flat, offs = flat.to(dev), offs.to(dev)
        dtype = dtype or torch.float64
        out = torch.empty((len(prompts), self.dimension), dtype=dtype, device=dev)
        o64 = out if dtype == torch.float64 else None
        o32 = out if dtype == torch.float32 else None
        _lib.call("alise_embed_batch", _lib.ptr(flat), _lib.ptr(offs), len(prompts), self.dimension,
                  _lib.ptr(o64), _lib.ptr(o32), _lib.stream_ptr(stream))
        return out


def load_precomputed_embeddings(path) -> dict:
    """JSON-lines {"id", "vector"}, re-normalised (predictor.py:103-117)."""
    out = {}
    with open(path) as fh:
        for line in fh:
            line = line.strip()
            if not line:
                continue
            rec = json.loads(line)
            v = np.asarray(rec["vector"], dtype=np.float64)
            n = float(np.linalg.norm(v))
            if n == 0:
                raise PredictorError(f"zero vector for id {rec['id']}")
            out[int(rec["id"])] = v / n
    return out


# ----------------------------------------------------------------- device store
DB_F32, DB_F64 = 0, 1  # ALISE_DB_F32 / ALISE_DB_F64 (include/alise_b200.h)
ORDERS = {"exact": 0, "blas": 1}  # ALISE_ORDER_EXACT / ALISE_ORDER_BLAS


def openblas_threads() -> int:
    """OpenBLAS thread count of this host's numpy (what the reference's scan runs on)."""
    try:
        from threadpoolctl import threadpool_info
        for info in threadpool_info():
            if info.get("internal_api") == "openblas":
                return int(info["num_threads"])
    except Exception:
        pass
    import os
    return os.cpu_count() or 1


def _dtype_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float64:
        return DB_F64
    if dt == np.float32:
        return DB_F32
    raise PredictorError(f"unsupported store dtype {dt} (float32 or float64)")


def _torch_dtype(code: int):
    import torch
    return torch.float64 if code == DB_F64 else torch.float32


def _host_lens(lens):
    """Lengths as a host int64 array when they are host data (no device sync)."""
    import torch
    if isinstance(lens, torch.Tensor):
        return None if lens.is_cuda else lens.numpy().astype(np.int64).reshape(-1)
    return np.asarray(lens, dtype=np.int64).reshape(-1)


class VectorStore:
    """FIFO-bounded device store of (vector, observed length) (predictor.py:120-189).

    Same semantics: slot = seq % capacity, ``add`` returns the insert sequence,
    ``search`` returns (sims f64, lens i64, seqs i64) ordered by (-sim, seq).

    ``dtype`` is the master copy's type: float64 (default) keeps the reference's
    np.float64 vectors exactly (predictor.py:126), so sims are the correctly rounded
    dot products of the very vectors the reference stores and ``newest`` returns them
    bit for bit; float32 halves the footprint for fp32 embedding DBs (BASELINE C4).
    Queries are converted to the master type.
    """

    def __init__(self, dimension: int, capacity: int, device: int | None = None, dtype=np.float64,
                 order: str = "exact", blas_threads: int | None = None):
        import torch

        _lib.require_cuda()
        self.dimension = int(dimension)
        self.capacity = int(capacity)
        self.dtype = np.dtype(dtype)
        self._code = _dtype_code(self.dtype)
        self.device = torch.cuda.current_device() if device is None else device
        h = _lib.C.c_void_p()
        _lib.call("alise_db_create_ex", self.device, self.capacity, self.dimension, self._code, _lib.C.byref(h))
        self._h = h.value
        self.size = 0
        self.next_seq = 0
        self.set_order(order, blas_threads)

    def set_order(self, order: str = "exact", blas_threads: int | None = None, ref_capacity: int = 0,
                  ref_size: int = -1):
        """Which float64 sims searches rank by and return: "exact" (the correctly rounded
        dot products; default) or "blas" (the reference's own values: the operation order
        of numpy -> OpenBLAS dgemv_t behind predictor.py:158, so real-arithmetic ties break
        as in the reference; blas_threads = the reference host's OpenBLAS threads)."""
        if order not in ORDERS:
            raise PredictorError(f"order must be one of {sorted(ORDERS)}")
        self.order = order
        self.blas_threads = int(blas_threads or openblas_threads())
        _lib.call("alise_db_set_order", self._h, ORDERS[order], self.blas_threads, int(ref_capacity),
                  int(ref_size))

    def __len__(self):
        return self.size

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            try:
                _lib.lib().alise_db_destroy(h)
            except Exception:
                pass

    def _dev(self):
        import torch
        return torch.device("cuda", self.device)

    def _as_rows(self, vectors):
        """Rows on this store's device in the master dtype, [n, dimension] contiguous."""
        import torch
        v = torch.as_tensor(vectors if isinstance(vectors, torch.Tensor) else np.asarray(vectors))
        return v.to(self._dev(), _torch_dtype(self._code)).reshape(-1, self.dimension).contiguous()

    _STAGE_SLOTS = 32

    def add(self, vector, observed_len: int) -> int:
        """VectorStore.add (predictor.py:135-152): one record, appended without a host
        synchronisation -- the vector, length and sequence number are packed into a
        pinned staging slot, copied with one async H2D on the current stream and
        appended by the ring kernel (a slot is reused once its copy has completed)."""
        import torch

        if observed_len < 1:
            raise PredictorError("observed_len must be >= 1")
        v = np.asarray(vector, dtype=np.float64).reshape(-1)
        if v.size != self.dimension:
            raise PredictorError("vector has the wrong dimension")
        seq = self.next_seq
        if getattr(self, "_stage_h", None) is None:
            esz = 8 if self._code == DB_F64 else 4
            self._stage_vb = (self.dimension * esz + 15) // 16 * 16
            nb = self._stage_vb + 16
            self._stage_h = torch.empty((self._STAGE_SLOTS, nb), dtype=torch.uint8).pin_memory()
            self._stage_d = torch.empty((self._STAGE_SLOTS, nb), dtype=torch.uint8, device=self._dev())
            self._stage_ev = [None] * self._STAGE_SLOTS
            self._stage_i = 0
        r = self._stage_i
        self._stage_i = (r + 1) % self._STAGE_SLOTS
        if self._stage_ev[r] is not None:
            self._stage_ev[r].synchronize()  # the slot's previous copy has left the host buffer
        hv = self._stage_h[r].numpy()
        vb = self._stage_vb
        hv[:vb].view(np.float64 if self._code == DB_F64 else np.float32)[: self.dimension] = v
        hv[vb:vb + 4].view(np.int32)[0] = int(observed_len)
        hv[vb + 8:vb + 16].view(np.int64)[0] = seq
        dv = self._stage_d[r]
        dv.copy_(self._stage_h[r], non_blocking=True)
        if self._stage_ev[r] is None:
            self._stage_ev[r] = torch.cuda.Event()
        self._stage_ev[r].record()
        base = dv.data_ptr()
        _lib.call("alise_db_append", self._h, base, base + vb, base + vb + 8, 1, _lib.stream_ptr())
        self.next_seq += 1
        self.size = min(self.capacity, self.size + 1)
        return seq

    def add_batch(self, vectors, lens, stream=None, seqs=None):
        """Append rows in insert order (batched VectorStore.add).  ``seqs`` (host int64,
        increasing) restores records under their original sequence numbers (snapshots)."""
        import torch

        v = self._as_rows(vectors)
        hl = _host_lens(lens)
        ln = torch.as_tensor(hl if hl is not None else lens).to(self._dev(), torch.int32).reshape(-1).contiguous()
        n = v.shape[0]
        if ln.numel() != n:
            raise PredictorError("vectors and lengths differ in count")
        if n and (hl.min() if hl is not None else int(ln.min().item())) < 1:
            raise PredictorError("observed_len must be >= 1")
        if seqs is not None:
            seqs = np.asarray(seqs, dtype=np.int64).reshape(-1)
            if len(seqs) != n or (n and (seqs[0] < self.next_seq or np.any(np.diff(seqs) <= 0))):
                raise PredictorError("restored sequence numbers must increase past next_seq")
        done = 0
        while done < n:
            m = min(n - done, self.capacity)
            if seqs is None:
                sq = torch.arange(self.next_seq, self.next_seq + m, dtype=torch.int64, device=self._dev())
            else:
                sq = torch.as_tensor(seqs[done:done + m]).to(self._dev())
            _lib.call("alise_db_append", self._h, _lib.ptr(v[done:done + m]), _lib.ptr(ln[done:done + m]),
                      _lib.ptr(sq), m, _lib.stream_ptr(stream))
            self.next_seq = self.next_seq + m if seqs is None else int(seqs[done + m - 1]) + 1
            self.size = min(self.capacity, self.size + m)
            done += m
        return self.next_seq - 1

    def search_batch(self, queries, k: int, stream=None):
        """Exact top-k for a batch.  Returns CUDA tensors (sims f64 [B,k], seqs i64,
        lens i32, counts i32 [B], the queries in the master dtype); rows past
        counts[b] are undefined."""
        import torch

        if k < 1 or k > MAX_K:
            raise PredictorError(f"k must be in [1, {MAX_K}]")
        q = self._as_rows(queries)
        B = q.shape[0]
        dev = self._dev()
        sims = torch.empty((B, k), dtype=torch.float64, device=dev)
        seqs = torch.empty((B, k), dtype=torch.int64, device=dev)
        lens = torch.empty((B, k), dtype=torch.int32, device=dev)
        cnt = torch.empty(B, dtype=torch.int32, device=dev)
        _lib.call("alise_db_topk", self._h, _lib.ptr(q), B, k, _lib.ptr(sims), _lib.ptr(seqs),
                  _lib.ptr(lens), _lib.ptr(cnt), _lib.stream_ptr(stream))
        return sims, seqs, lens, cnt, q

    def search(self, vector, k: int):
        """Top-k by cosine similarity; ties broken by older insert first."""
        if self.size == 0:
            return np.array([]), np.array([], dtype=np.int64), np.array([], dtype=np.int64)
        k = min(k, self.size)
        sims, seqs, lens, cnt, _ = self.search_batch(np.asarray(vector, dtype=np.float64)[None, :], k)
        c = int(cnt[0].item())
        return (sims[0, :c].cpu().numpy(), lens[0, :c].cpu().numpy().astype(np.int64),
                seqs[0, :c].cpu().numpy())

    def set_timing(self, on: bool):
        _lib.call("alise_db_timing", self._h, int(on))

    def kernel_stats(self):
        """(scan_ms, launches, algorithmic flops) since the last call (synchronises)."""
        ms, fl = _lib.C.c_double(), _lib.C.c_double()
        n = _lib.C.c_int64()
        _lib.call("alise_db_kernel_stats", self._h, _lib.C.byref(ms), _lib.C.byref(n), _lib.C.byref(fl))
        return ms.value, n.value, fl.value

    def inexact_count(self) -> int:
        """Candidates whose float64 rounding could not be certified (expected 0)."""
        c = _lib.C.c_uint()
        _lib.call("alise_db_inexact", self._h, _lib.C.byref(c))
        return int(c.value)

    # -- host-side views (not on the hot path) --------------------------------------
    def newest(self, count: int):
        """Vectors and lengths of the most recently inserted records (predictor.py:165-168)."""
        vecs, lens, seqs = self.export()
        order = np.argsort(seqs)[-count:]
        return vecs[order], lens[order]

    def export(self):
        """Copy the live records to the host: (vectors f64 [n,d], lens i64, seqs i64)."""
        import torch

        n = self.size
        if n == 0:
            return np.zeros((0, self.dimension)), np.zeros(0, np.int64), np.zeros(0, np.int64)
        vec = torch.empty((n, self.dimension), dtype=_torch_dtype(self._code), device=self._dev())
        lens = torch.empty(n, dtype=torch.int32, device=self._dev())
        seqs = torch.empty(n, dtype=torch.int64, device=self._dev())
        _lib.call("alise_db_export", self._h, _lib.ptr(vec), _lib.ptr(lens), _lib.ptr(seqs), n,
                  _lib.stream_ptr())
        return (vec.cpu().numpy().astype(np.float64), lens.cpu().numpy().astype(np.int64),
                seqs.cpu().numpy())

    def save(self, path):
        vecs, lens, seqs = self.export()
        with open(path, "w") as fh:
            for i in np.argsort(seqs):
                fh.write(json.dumps({"seq": int(seqs[i]), "len": int(lens[i]),
                                     "vector": [float(x) for x in vecs[i]]}) + "\n")

    def save_binary(self, path):
        """Binary snapshot (npz: master-dtype vectors, lengths, seqs in insert order,
        next_seq) — the GPU-native counterpart of the JSON-lines ``save``
        (predictor.py:170-178)."""
        vecs, lens, seqs = self.export()
        order = np.argsort(seqs)
        np.savez(path, vectors=vecs[order].astype(self.dtype), lens=lens[order], seqs=seqs[order],
                 dimension=self.dimension, capacity=self.capacity, next_seq=self.next_seq)

    @classmethod
    def load_binary(cls, path, capacity: int | None = None, restore_seqs: bool = False) -> "VectorStore":
        """Re-adds the records in insert order: new seqs from 0 like ``load``
        (predictor.py:180-189), or, with restore_seqs, under their original sequence
        numbers (same slots, same FIFO position, same next_seq)."""
        z = np.load(path)
        cap = int(capacity or z["capacity"])
        store = cls(int(z["dimension"]), cap, dtype=z["vectors"].dtype)
        if len(z["lens"]):
            store.add_batch(z["vectors"], z["lens"], seqs=z["seqs"] if restore_seqs else None)
        if restore_seqs and "next_seq" in z:
            store.next_seq = int(z["next_seq"])
        return store

    @classmethod
    def load(cls, path, dimension: int, capacity: int) -> "VectorStore":
        vecs, lens = [], []
        with open(path) as fh:
            for line in fh:
                line = line.strip()
                if line:
                    rec = json.loads(line)
                    vecs.append(rec["vector"])
                    lens.append(int(rec["len"]))
        store = cls(dimension, capacity)
        if vecs:
            store.add_batch(np.asarray(vecs, dtype=np.float64), lens)
        return store


def _as_query_rows(queries, dimension=None):
    """Queries as a contiguous CUDA tensor on the current device, float64 when given in
    float64 (numpy's default: the reference's own vectors), else fp32."""
    import torch
    q = torch.as_tensor(queries if isinstance(queries, torch.Tensor) else np.asarray(queries))
    dt = torch.float64 if q.dtype == torch.float64 else torch.float32
    q = q.to(torch.device("cuda", torch.cuda.current_device()), dt)
    if dimension is not None:
        q = q.reshape(-1, dimension)
    return q.contiguous()


def _query_code(q) -> int:
    import torch
    return DB_F64 if q.dtype == torch.float64 else DB_F32


# ----------------------------------------------------------------- fallback regressor
class FallbackRegressor:
    """One-hidden-layer tanh regressor on log length (predictor.py:192-264)."""

    def __init__(self, dimension: int, hidden: int, seed: int = 0):
        gen = _stream(seed, FALLBACK_INIT)
        lim = math.sqrt(6.0 / (dimension + hidden))
        self.w1 = gen.uniform(-lim, lim, size=(dimension, hidden))
        self.b1 = np.zeros(hidden)
        self.w2 = gen.uniform(-lim, lim, size=hidden) / math.sqrt(hidden)
        self.b2 = 0.0
        self.loss_history: list = []
        self.trained = False
        self._dev_cache = None

    # host-side forward (training only)
    def _forward(self, X):
        h = np.tanh(X @ self.w1 + self.b1)
        return h, h @ self.w2 + self.b2

    def predict_log(self, vector) -> float:
        return float(self._forward(np.asarray(vector, dtype=np.float64)[None, :])[1][0])

    def device_weights(self):
        """float64 CUDA copies of (W1, b1, w2), refreshed when the weights change."""
        import torch
        key = (id(self.w1), id(self.b1), id(self.w2))
        if self._dev_cache is None or self._dev_cache[0] != key:
            d = torch.device("cuda", torch.cuda.current_device())
            self._dev_cache = (key, torch.as_tensor(np.ascontiguousarray(self.w1), dtype=torch.float64).to(d),
                               torch.as_tensor(self.b1, dtype=torch.float64).to(d),
                               torch.as_tensor(self.w2, dtype=torch.float64).to(d))
        return self._dev_cache[1:]

    def predict_len_batch(self, X, max_len: int, stream=None):
        """Batched predict_len on the GPU (float64 MLP, same op order as the oracle).
        X is used in its own precision: float64 input (the reference's vectors) stays
        float64, anything else is read as fp32."""
        import torch
        x = _as_query_rows(X)
        B = x.shape[0]
        dev = x.device
        cnt = torch.zeros(B, dtype=torch.int32, device=dev)
        sims = torch.empty((B, 1), dtype=torch.float64, device=dev)
        lens = torch.empty((B, 1), dtype=torch.int32, device=dev)
        out = torch.empty(B, dtype=torch.int32, device=dev)
        ret = torch.empty(B, dtype=torch.uint8, device=dev)
        W1, b1, w2 = self.device_weights()
        _lib.call("alise_predict_finish_ex", B, 1, _lib.ptr(sims), _lib.ptr(lens), _lib.ptr(cnt), 2.0,
                  _lib.ptr(x), _query_code(x), x.shape[1], _lib.ptr(W1), _lib.ptr(b1), _lib.ptr(w2),
                  float(self.b2), W1.shape[1], int(max_len), math.log(max_len) + 1.0, _lib.ptr(out),
                  _lib.ptr(ret), _lib.stream_ptr(stream))
        return out

    def predict_len(self, vector, max_len: int) -> int:
        return int(self.predict_len_batch(np.asarray(vector, dtype=np.float64)[None, :], max_len)[0].item())

    def fit(self, X, lengths, epochs: int, learning_rate: float):
        """Full-batch gradient descent with backtracking (predictor.py:221-264).
        Host-side weight production (not on the hot path)."""
        X = np.asarray(X, dtype=np.float64)
        y = np.log(np.asarray(lengths, dtype=np.float64))
        n = X.shape[0]

        def evaluate(w1, b1, w2, b2):
            h = np.tanh(X @ w1 + b1)
            err = (h @ w2 + b2) - y
            g = 2.0 * err / n
            dpre = np.outer(g, w2) * (1.0 - h ** 2)
            return float(np.mean(err ** 2)), (X.T @ dpre, dpre.sum(axis=0), h.T @ g, float(g.sum()))

        params = (self.w1, self.b1, self.w2, self.b2)
        loss, grads = evaluate(*params)
        self.loss_history = [loss]
        lr = learning_rate
        for _ in range(epochs):
            step_taken = False
            for _ in range(30):
                trial = tuple(p - lr * g for p, g in zip(params, grads))
                t_loss, t_grads = evaluate(*trial)
                if t_loss <= loss:
                    params, loss, grads, step_taken = trial, t_loss, t_grads, True
                    break
                lr *= 0.5
            self.loss_history.append(loss)
            if step_taken:
                lr = min(lr * 1.25, learning_rate)
        self.w1, self.b1, self.w2, self.b2 = params
        self.b2 = float(self.b2)
        self.trained = True
        self._dev_cache = None
        return self


def train_fallback(corpus, config: PredictorConfig, seed: int = 0, embedder=None) -> FallbackRegressor:
    """predictor.py:267-279."""
    if len(corpus) < 10:
        raise PredictorError("training corpus must have at least 10 examples")
    embedder = embedder or HashingEmbedder(config.dimension)
    X = np.stack([embedder.embed(tokens) for tokens, _ in corpus])
    lengths = [n for _, n in corpus]
    if min(lengths) < 1:
        raise PredictorError("corpus lengths must be >= 1")
    reg = FallbackRegressor(config.dimension, config.fallback_hidden, seed=seed)
    return reg.fit(X, lengths, config.fallback_epochs, config.fallback_learning_rate)


# ----------------------------------------------------------------- length predictor
class _GraphedRequest:
    """One-query predict path captured as a CUDA graph (pinned host in/out buffers)."""

    def __init__(self, predictor):
        import torch
        self.p = predictor
        d = predictor.config.dimension
        self.h_in = torch.zeros(1, d, dtype=torch.float64).pin_memory()
        self.h_out = torch.zeros(1, dtype=torch.int32).pin_memory()
        self.h_ret = torch.zeros(1, dtype=torch.uint8).pin_memory()
        self.d_in = torch.zeros(1, d, dtype=torch.float64, device="cuda")
        self.key = None
        self.graph = None

    def _key(self):
        w = self.p.regressor.device_weights()
        return (self.p.store.size, tuple(int(t.data_ptr()) for t in w), float(self.p.regressor.b2))

    def _capture(self):
        import torch
        # warm-up outside the capture: allocates the store's scratch and sets kernel attributes
        self.p.predict_batch(self.d_in)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.d_in.copy_(self.h_in, non_blocking=True)
            out, ret = self.p.predict_batch(self.d_in)
            self.h_out.copy_(out, non_blocking=True)
            self.h_ret.copy_(ret, non_blocking=True)
        self.graph = g
        self.key = self._key()

    def __call__(self, vector):
        import torch
        if self.graph is None or self._key() != self.key:
            self._capture()
        self.h_in.numpy()[0] = np.asarray(vector, dtype=np.float64)
        self.graph.replay()
        torch.cuda.current_stream().synchronize()
        return int(self.h_out[0]), int(self.h_ret[0])


class LengthPredictor:
    """Retrieval-first length predictor with regressor fallback (predictor.py:286-352)."""

    def __init__(self, config: PredictorConfig, regressor: FallbackRegressor | None = None,
                 embedder: HashingEmbedder | None = None, store: VectorStore | None = None,
                 precomputed: dict | None = None):
        config.validate()
        self.config = config
        self.embedder = embedder or HashingEmbedder(config.dimension)
        self.store = store if store is not None else VectorStore(config.dimension, config.db_capacity)
        if regressor is None and not config.allow_untrained:
            raise PredictorError("no trained fallback and allow_untrained is false")
        self._untrained = regressor is None
        self.regressor = regressor or FallbackRegressor(config.dimension, config.fallback_hidden, seed=0)
        self.precomputed = precomputed or {}
        self._observations = 0
        self._next_refit = 8

    def embed(self, tokens, request_id: int | None = None) -> np.ndarray:
        if request_id is not None and request_id in self.precomputed:
            return self.precomputed[request_id]
        return self.embedder.embed(tokens)

    def predict_batch(self, queries, stream=None):
        """Batched predict_vector: (lengths int32 [B], retrieved uint8 [B]) CUDA tensors.
        The search runs in the store's master dtype; the fallback MLP reads the queries
        in their own precision (float64 for the reference's float64 vectors)."""
        import torch
        cfg = self.config
        q = _as_query_rows(queries, cfg.dimension)
        B = q.shape[0]
        k = cfg.top_k
        if self.store.size > 0:
            sims, _seqs, lens, cnt, _q = self.store.search_batch(q, k, stream=stream)
        else:
            dev = q.device
            sims = torch.empty((B, k), dtype=torch.float64, device=dev)
            lens = torch.empty((B, k), dtype=torch.int32, device=dev)
            cnt = torch.zeros(B, dtype=torch.int32, device=dev)
        return self.finish(sims, lens, cnt, q, stream=stream)

    def finish(self, sims, lens, cnt, q, stream=None):
        """Aggregate + MLP fallback over given (possibly merged) top-k lists; q fp32 or
        float64 [B, dimension] on the device."""
        import torch
        cfg = self.config
        B, k = sims.shape
        out = torch.empty(B, dtype=torch.int32, device=q.device)
        ret = torch.empty(B, dtype=torch.uint8, device=q.device)
        W1, b1, w2 = self.regressor.device_weights()
        _lib.call("alise_predict_finish_ex", B, k, _lib.ptr(sims), _lib.ptr(lens), _lib.ptr(cnt),
                  float(cfg.similarity_threshold), _lib.ptr(q), _query_code(q), cfg.dimension, _lib.ptr(W1),
                  _lib.ptr(b1), _lib.ptr(w2), float(self.regressor.b2), W1.shape[1], int(cfg.max_len),
                  math.log(cfg.max_len) + 1.0, _lib.ptr(out), _lib.ptr(ret), _lib.stream_ptr(stream))
        return out, ret

    def enable_graphs(self, on: bool = True):
        """Serve predict_vector (one request) by replaying a CUDA graph of the whole
        per-request path: query upload, prep, tcgen05 scan, rescoring, finish and the
        result download become one graph launch (re-captured when the DB size or the
        fallback weights change).  top_k > 16 (the CUDA-core search, which synchronises to
        report near-tie overflow) stays eager."""
        self._graph = _GraphedRequest(self) if on and self.config.top_k <= 16 else None

    def predict_vector(self, vector) -> tuple:
        """Predict from an already-embedded prompt; returns (length, provenance)."""
        g = getattr(self, "_graph", None)
        if g is not None and self.store.size > 0:
            length, ret = g(vector)
            return length, (RETRIEVED if ret else FALLBACK)
        out, ret = self.predict_batch(np.asarray(vector, dtype=np.float64)[None, :])
        return int(out[0].item()), (RETRIEVED if int(ret[0].item()) else FALLBACK)

    def predict(self, tokens, request_id: int | None = None) -> tuple:
        vec = self.embed(tokens, request_id)
        length, provenance = self.predict_vector(vec)
        return length, provenance, vec

    def observe(self, vector, actual_len: int):
        """Append a finished request; refit the fallback on a geometric schedule."""
        self.store.add(vector, actual_len)
        self._observations += 1
        if self.config.online_refit and self._observations >= self._next_refit:
            self._refit()
            cap = self.config.refit_sample_cap
            self._next_refit = min(self._next_refit * 2, self._observations + cap)

    def _refit(self):
        X, lens = self.store.newest(self.config.refit_sample_cap)
        reg = FallbackRegressor(self.config.dimension, self.config.fallback_hidden, seed=self._observations)
        reg.fit(X, lens, self.config.refit_epochs, self.config.fallback_learning_rate)
        self.regressor = reg


def eval_accuracy(pairs, bin_width: int, latencies_ms=None) -> dict:
    """Bucketed accuracy and mean relative error (predictor.py:355-374)."""
    if bin_width < 1:
        raise PredictorError("bin_width must be >= 1")
    pairs = list(pairs)
    if not pairs:
        raise PredictorError("no prediction pairs to evaluate")
    hits = sum(1 for p, a in pairs if p // bin_width == a // bin_width)
    rel = sum(abs(p - a) / a for p, a in pairs) / len(pairs)
    return {"count": len(pairs), "accuracy": hits / len(pairs), "pred_error": rel,
            "mean_latency_ms": float(np.mean(latencies_ms)) if latencies_ms else 0.0}

