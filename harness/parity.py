"""Parity checks shared by the GPU tests and bench.py (checker side only: the oracle
is the reference restated in oracle/; nothing here is on the product path).

* KV: decode a host slab's (layer, K|V) plane records and compare codes, the (scale,
  zero) its fp16 (min, max) pair expands to, and the fp16 KV after the upload with
  the C oracle (oracle/kvquant_ref.c, kvmanager.py:108-154), plane by plane.
* Predictor: exact top-k (seqs, lens, float64 sims) and predicted lengths of sampled
  queries against oracle/pred_oracle.py (predictor.py:154-163, 311-325)."""
from __future__ import annotations

import ctypes
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
_C = None


def c_oracle():
    """ctypes handle of oracle/liboracle_kv.so (built on demand with make)."""
    global _C
    if _C is None:
        so = os.path.join(ROOT, "oracle", "liboracle_kv.so")
        src = os.path.join(ROOT, "oracle", "kvquant_ref.c")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
            subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle")], check=True)
        lib = ctypes.CDLL(so)
        vp, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        lib.oracle_quantize_f64.argtypes = [vp, i64, i64, i32, vp, vp, vp]
        lib.oracle_quantize_f16.argtypes = [vp, i64, i64, i32, vp, vp, vp, vp]
        lib.oracle_dequantize.argtypes = [vp, vp, vp, i64, i64, vp]
        _C = lib
    return _C


def c_quantize(lib, x, bits):
    """Run the C oracle on a 2D float16/float64 array: (codes, scale [r,1], zero [r,1])."""
    x = np.ascontiguousarray(x)
    r, n = x.shape
    codes = np.empty((r, n), np.uint8)
    scale = np.empty((r, 1))
    zero = np.empty((r, 1))
    if x.dtype == np.float16:
        scratch = np.empty(n)
        st = lib.oracle_quantize_f16(x.ctypes.data, r, n, bits, codes.ctypes.data, scale.ctypes.data,
                                     zero.ctypes.data, scratch.ctypes.data)
    else:
        x = x.astype(np.float64)
        st = lib.oracle_quantize_f64(x.ctypes.data, r, n, bits, codes.ctypes.data, scale.ctypes.data,
                                     zero.ctypes.data)
    if st != 0:
        raise ValueError(f"oracle quantize failed ({st})")
    return codes, scale, zero


def plane_records(lay, slab):
    """Yield (plane, codes bytes, fp16 (min, -max) pairs) of every (layer, K|V) plane of a
    slab: chunk records are [codes, native order][(min, -max) per group], sections
    256-byte aligned."""
    g = lay.geometry()
    planes = lay.layers * 2
    ppc = -(-planes // g["n_chunks"])
    per_codes = lay.tokens * lay.hidden // (2 if lay.packed else 1)
    rows_pp = g["rows"] // planes
    a256 = lambda x: (x + 255) // 256 * 256
    for p in range(planes):
        c, j = divmod(p, ppc)
        np_ = min(ppc, planes - c * ppc)
        base = c * g["chunk_bytes"]
        codes = slab[base + j * per_codes: base + (j + 1) * per_codes]
        pbase = base + a256(np_ * per_codes) + j * rows_pp * 4
        yield p, codes, slab[pbase: pbase + rows_pp * 4].view(np.float16).reshape(-1, 2)


def kv_check_planes(lay, src_h, slab, out_h, planes=None, threads=8):
    """Compare the given planes (default all) of one job: src_h / out_h are the job's KV
    before the offload and after the upload ([layers, 2, T, hidden] fp16, host), slab
    its host slab.  Returns (planes checked, values checked, mismatching planes)."""
    from oracle import kv_oracle as ko
    lib = c_oracle()
    kind = "contig" if lay.kind == "rows" else lay.kind
    want = set(range(lay.layers * 2) if planes is None else planes)
    bad = []

    def check(rec):
        p, codes, mm = rec
        if p not in want:
            return
        layer, s = divmod(p, 2)
        x = src_h[layer, s][None, None]
        rows = ko.view_rows(x, kind, group=lay.group, head_dim=lay.head_dim)
        absmax = getattr(lay, "mode", "asymmetric") == "absmax"
        if absmax:   # restated symmetric mode (parity unpinned by the reference)
            c_ref, s_ref, z_ref = ko.quantize_rows_absmax(rows, lay.bits)
        else:
            c_ref, s_ref, z_ref = c_quantize(lib, rows, lay.bits)
        codes = np.asarray(codes)
        if lay.packed:
            codes = np.stack([codes & 15, codes >> 4], axis=1).reshape(-1)
        got = ko.view_rows(codes.reshape(x.shape), kind, group=lay.group, head_dim=lay.head_dim)
        solve = ko.params_absmax if absmax else ko.params_from_minmax
        scale, zero = solve(mm[:, 0].astype(np.float64), -mm[:, 1].astype(np.float64), lay.bits)
        deq = np.empty(rows.shape)
        lib.oracle_dequantize(c_ref.ctypes.data, s_ref.ctypes.data, z_ref.ctypes.data, rows.shape[0], rows.shape[1],
                              deq.ctypes.data)
        back = ko.view_rows(out_h[layer, s][None, None], kind, group=lay.group, head_dim=lay.head_dim)
        if not (np.array_equal(got, c_ref) and np.array_equal(scale, s_ref[:, 0])
                and np.array_equal(zero, z_ref[:, 0]) and np.array_equal(back, deq.astype(np.float16))):
            bad.append(p)

    with ThreadPoolExecutor(threads) as ex:   # the C oracle releases the GIL
        list(ex.map(check, plane_records(lay, slab)))
    per_plane = lay.tokens * lay.hidden
    return len(want), len(want) * per_plane, sorted(bad)


def pred_search_fp32(db32, lens, Q32, k: int, chunk: int = 64):
    """Exact top-k by (-sim, seq) of fp32 queries over an fp32 DB (seq = row index):
    an fp32 BLAS pass with a rigorous margin (any summation order errs by at most
    dim 2^-24 sum|p| <= dim 2^-24 |v| |q|) picks the candidates, which are rescored
    with the correctly rounded float64 dot (oracle/pred_oracle.exact_dot)."""
    from oracle import pred_oracle as po
    n, d = db32.shape
    kk = min(k, n)
    vmax = 0.0
    for r0 in range(0, n, 65536):  # float64 row norms without a float64 copy of the DB
        blk = db32[r0:r0 + 65536].astype(np.float64)
        vmax = max(vmax, float(np.sqrt((blk * blk).sum(axis=1).max())))
    out = []
    for c0 in range(0, len(Q32), chunk):
        Qc = np.ascontiguousarray(Q32[c0:c0 + chunk], dtype=np.float32)
        coarse = db32 @ Qc.T
        for j in range(Qc.shape[0]):
            col = coarse[:, j].astype(np.float64)
            margin = 1.01 * (d + 2) * 2.0 ** -24 * vmax * float(np.linalg.norm(Qc[j].astype(np.float64)))
            kth = np.partition(col, n - kk)[n - kk]
            cand = np.flatnonzero(col >= kth - 2 * margin)
            exact = np.array([po.exact_dot(db32[r], Qc[j]) for r in cand])
            o = np.lexsort((cand, -exact))[:kk]
            out.append((exact[o], np.asarray(lens)[cand[o]].astype(np.int64), cand[o].astype(np.int64)))
    return out


def pred_check(db32, lens, Q32, idx, sims, seqs, slens, cnt, out_len, out_ret, W1, b1, w2, b2, k=8, s0=0.80,
               max_len=2048):
    """Compare GPU results (host arrays, rows idx of the batch) with the oracle: top-k
    seqs, lens and sims bit-exact, predicted lengths and provenance exact.  Returns the
    list of mismatching query indices."""
    from oracle import pred_oracle as po
    ref = pred_search_fp32(db32, lens, Q32[idx], k)
    mlp = po.mlp_predict_len(Q32[idx].astype(np.float64), W1, b1, w2, b2, max_len)
    bad = []
    for j, (i, (es, el, eq)) in enumerate(zip(idx, ref)):
        c = int(cnt[i])
        a = po.aggregate(es, el, s0, max_len)
        want_len, want_ret = (mlp[j], False) if a is None else (a, True)
        if not (c == len(eq) and np.array_equal(seqs[i, :c], eq) and np.array_equal(slens[i, :c], el)
                and np.array_equal(sims[i, :c], es) and int(out_len[i]) == int(want_len)
                and bool(out_ret[i]) == want_ret):
            bad.append(int(i))
    return bad


def kv_roundtrip_planes(lay, planes_src: dict, planes_out: dict):
    """planes_src / planes_out: {plane: [tokens, hidden] fp16 host array} before the
    offload and after the upload.  Returns the planes whose round trip differs from
    fp16(oracle dequantize(oracle quantize(src))) (kvmanager.py:108-154)."""
    from oracle import kv_oracle as ko
    lib = c_oracle()
    kind = "contig" if lay.kind == "rows" else lay.kind
    bad = []
    for p, x in planes_src.items():
        rows = ko.view_rows(np.asarray(x)[None, None], kind, group=lay.group, head_dim=lay.head_dim)
        c, s, z = c_quantize(lib, rows, lay.bits)
        deq = np.empty(rows.shape)
        lib.oracle_dequantize(c.ctypes.data, s.ctypes.data, z.ctypes.data, rows.shape[0], rows.shape[1],
                              deq.ctypes.data)
        back = ko.view_rows(np.asarray(planes_out[p])[None, None], kind, group=lay.group, head_dim=lay.head_dim)
        if not np.array_equal(back, deq.astype(np.float16)):
            bad.append(p)
    return bad
