"""Restated CPU oracle for the retrieval length predictor — TEST INFRASTRUCTURE ONLY.

Reference: /root/reference/pkg/src/servesim/predictor.py
  * VectorStore.search        :154-163  (sims = vecs @ q, argpartition, lexsort)
  * LengthPredictor.predict_vector :311-325 (threshold, clip, weighted mean, round, clamp)
  * FallbackRegressor._forward / predict_len :209-219

Why restated rather than called: the reference's arithmetic lives in numpy /
OpenBLAS (absent from /root/reference; numpy 2.3.5 + scipy-openblas 0.3.30 here),
whose dot-product summation order is unspecified, and ``argpartition`` picks an
arbitrary subset of rows tied at the k-boundary.  The restatement
pins what the north star asks for:
  * sims = the correctly rounded float64 value of the exact dot product
    (fp32 x fp32 products are exact in float64; float64 products are split exactly
    into two doubles (Dekker); summed with math.fsum);
  * order = full (-sim, seq) sort, so ties are broken by insert order everywhere;
  * aggregate = numpy's own ops on the same arrays (summation order: sequential for
    n < 8, 8-accumulator tree for n >= 8 — see tests/test_oracle_pred.py);
  * MLP = float64, separate multiply/add, hidden pre-activations summed over the
    input dimension in index order, output summed over hidden units in index order.
It agrees with the raw reference wherever the reference is well defined
(untied top-k, lengths) — checked against tests/golden/pred_golden.npz.
"""
from __future__ import annotations

import math

import numpy as np


def _two_prod(a, b):
    """Elementwise a*b = p + e exactly (Veltkamp/Dekker; float64 arrays in the normal
    range).  Entries whose products leave the safe range are returned in `bad`."""
    p = a * b
    c = 134217729.0  # 2^27 + 1
    ta = c * a
    ah = ta - (ta - a)
    al = a - ah
    tb = c * b
    bh = tb - (tb - b)
    bl = b - bh
    e = ((ah * bh - p) + ah * bl + al * bh) + al * bl
    mag = np.abs(p)
    bad = (p != 0) & ((mag < 2.0 ** -900) | (mag > 2.0 ** 900) | (np.abs(a) > 2.0 ** 995) | (np.abs(b) > 2.0 ** 995))
    return p, e, bad


def exact_dot(a, b, f64: bool = False) -> float:
    """Correctly rounded float64 dot product: of two fp32 vectors (products exact in
    float64), or with f64=True of two float64 vectors (products split exactly)."""
    if not f64:
        a = np.asarray(a, dtype=np.float32).astype(np.float64)
        b = np.asarray(b, dtype=np.float32).astype(np.float64)
        return math.fsum((a * b).tolist())
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    p, e, bad = _two_prod(a, b)
    if bad.any():  # exact rational arithmetic for out-of-range products
        from fractions import Fraction
        tot = sum((Fraction(x) * Fraction(y) for x, y in zip(a.tolist(), b.tolist())), Fraction(0))
        return float(tot)  # Fraction -> float rounds correctly (half-even)
    return math.fsum(p.tolist() + e.tolist())


def _rows(db, f64):
    return np.asarray(db, dtype=np.float64) if f64 else np.asarray(db, dtype=np.float32)


def search_exact(db32, lens, seqs, q32, k: int, f64: bool = False):
    """Exact top-k by (-sim, seq) over fp32 rows (or float64 rows with f64=True).
    Returns (sims f64, lens, seqs)."""
    db = _rows(db32, f64)
    n = db.shape[0]
    if n == 0:
        return np.array([]), np.array([], dtype=np.int64), np.array([], dtype=np.int64)
    k = min(k, n)
    qr = _rows(q32, f64)
    q = qr.astype(np.float64)
    coarse = db.astype(np.float64) @ q           # |error| <= ~dim * 2^-53 * |q| * max|v|
    margin = 1e-9 * max(1.0, float(np.abs(q).sum())) * max(1.0, float(np.abs(db).max()))
    kth = np.partition(coarse, n - k)[n - k]
    cand = np.flatnonzero(coarse >= kth - 2 * margin)
    exact = np.array([exact_dot(db[r], qr, f64) for r in cand])
    order = np.lexsort((np.asarray(seqs)[cand], -exact))[:k]
    pick = cand[order]
    return exact[order], np.asarray(lens)[pick].astype(np.int64), np.asarray(seqs)[pick].astype(np.int64)


def search_exact_batch(db32, lens, seqs, Q32, k: int, chunk: int = 256, f64: bool = False):
    """search_exact for a batch (one BLAS GEMM for the coarse pass).
    Returns lists of (sims, lens, seqs) per query."""
    db = _rows(db32, f64)
    db64 = db.astype(np.float64)
    Q = _rows(Q32, f64)
    n = db.shape[0]
    kk = min(k, n)
    out = []
    amax = float(np.abs(db).max()) if n else 1.0
    for c0 in range(0, len(Q), chunk):
        Qc = Q[c0:c0 + chunk].astype(np.float64)
        coarse = db64 @ Qc.T
        for j in range(Qc.shape[0]):
            col = coarse[:, j]
            margin = 1e-9 * max(1.0, float(np.abs(Qc[j]).sum())) * max(1.0, amax)
            kth = np.partition(col, n - kk)[n - kk]
            cand = np.flatnonzero(col >= kth - 2 * margin)
            exact = np.array([exact_dot(db[r], Q[c0 + j], f64) for r in cand])
            order = np.lexsort((np.asarray(seqs)[cand], -exact))[:kk]
            pick = cand[order]
            out.append((exact[order], np.asarray(lens)[pick].astype(np.int64),
                        np.asarray(seqs)[pick].astype(np.int64)))
    return out


_BLAS = None


def _blas_lib():
    global _BLAS
    if _BLAS is None:
        import ctypes
        import os
        import subprocess
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "liboracle_blas.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(here, "blas_order.c")):
            subprocess.run(["make", "-s", "-C", here], check=True)
        lib = ctypes.CDLL(so)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.oracle_blas_gemv.argtypes = [vp, i64, i64, vp, vp, i32]
        _BLAS = lib
    return _BLAS


def blas_gemv(V, x, threads: int):
    """V @ x (V float64 [n, d] row-major) in the reference BLAS's operation order
    (oracle/blas_order.c: numpy -> OpenBLAS 0.3.30 dgemv_t on x86-64)."""
    V = np.ascontiguousarray(V, dtype=np.float64)
    x = np.ascontiguousarray(x, dtype=np.float64)
    y = np.empty(V.shape[0])
    if V.shape[0]:
        _blas_lib().oracle_blas_gemv(V.ctypes.data, V.shape[0], V.shape[1], x.ctypes.data, y.ctypes.data, threads)
    return y


def search_blas(slots, lens, seqs, q, k: int, threads: int):
    """VectorStore.search (predictor.py:154-163) verbatim in algorithm, with the scan's
    float64 sims in the reference BLAS order: rows are the ring slots in slot order
    (the reference's self._vecs[:size]); argpartition + lexsort as the reference."""
    n = len(slots)
    if n == 0:
        return np.array([]), np.array([], dtype=np.int64), np.array([], dtype=np.int64)
    sims = blas_gemv(slots, q, threads)
    k = min(k, n)
    idx = np.argpartition(-sims, k - 1)[:k]
    order = np.lexsort((np.asarray(seqs)[idx], -sims[idx]))
    idx = idx[order]
    return sims[idx], np.asarray(lens)[idx].astype(np.int64), np.asarray(seqs)[idx].astype(np.int64)


def aggregate(sims, lens, s0: float, max_len: int):
    """predict_vector's retrieval branch (predictor.py:314-324).

    Returns the length, or None when no neighbour qualifies (-> fallback MLP).
    """
    sims = np.asarray(sims, dtype=np.float64)
    if sims.size == 0:
        return None
    qualify = sims >= s0
    if not qualify.any():
        return None
    w = np.clip(sims[qualify], 0.0, None)
    vals = np.asarray(lens)[qualify].astype(np.float64)
    if w.sum() > 0.0:
        pred = float((w * vals).sum() / w.sum())
    else:
        pred = float(vals.mean())
    return int(min(max(round(pred), 1), max_len))


def mlp_forward(X, W1, b1, w2, b2):
    """Batched float64 MLP in the canonical order the CUDA kernel uses."""
    X = np.asarray(X, dtype=np.float64)
    W1 = np.asarray(W1, dtype=np.float64)
    acc = np.zeros((X.shape[0], W1.shape[1]))
    for d in range(X.shape[1]):
        acc = acc + X[:, d:d + 1] * W1[d]
    h = np.tanh(acc + np.asarray(b1, dtype=np.float64))
    out = np.zeros(X.shape[0])
    for j in range(h.shape[1]):
        out = out + h[:, j] * float(w2[j])
    return out + float(b2)


def mlp_predict_len(X, W1, b1, w2, b2, max_len: int):
    """FallbackRegressor.predict_len (predictor.py:217-219) for a batch."""
    out = mlp_forward(X, W1, b1, w2, b2)
    cap = math.log(max_len) + 1.0
    raw = np.exp(np.minimum(out, cap))
    return np.clip(np.rint(raw), 1, max_len).astype(np.int64)


def predict_batch(db32, lens, seqs, Q32, W1, b1, w2, b2, k=8, s0=0.80, max_len=2048, f64: bool = False):
    """Full predict_vector for a batch (search + aggregate, else MLP).  With f64=True the
    rows and queries are float64 (the reference's own store and MLP inputs)."""
    fallback = mlp_predict_len(_rows(Q32, f64).astype(np.float64), W1, b1, w2, b2, max_len)
    out_len = np.empty(len(Q32), dtype=np.int64)
    retrieved = np.zeros(len(Q32), dtype=bool)
    for i, q in enumerate(Q32):
        s, ln, _ = search_exact(db32, lens, seqs, q, k, f64=f64)
        a = aggregate(s, ln, s0, max_len)
        if a is None:
            out_len[i] = fallback[i]
        else:
            out_len[i] = a
            retrieved[i] = True
    return out_len, retrieved
