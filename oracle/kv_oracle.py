"""Numpy restatement of the reference KV quantizer — TEST INFRASTRUCTURE ONLY.

Restates ``servesim.kvmanager`` (reference ``pkg/src/servesim/kvmanager.py``):
  * ``quantize``   kvmanager.py:108-149  (row min/max, scale/zero, snap loop, codes)
  * ``dequantize`` kvmanager.py:152-154
  * ``kv_bytes`` / ``quantized_kv_bytes`` kvmanager.py:61-82

The reference iterates the scale-snap map over *all* rows until every row is
a fixed point (or 32 passes).  Because a fixed point stays fixed, that equals
applying the map to each row independently until it is fixed or 32 passes
have run; this restatement does it per row with an explicit active mask,
which is also exactly what the CUDA kernel does (one row per thread group).

Everything is IEEE float64 with separate multiply/add (numpy never fuses),
``np.rint`` is round-half-to-even and ``x / scale`` is a correctly rounded
division — the properties the bit-exact CUDA kernel reproduces.

This module is also the ``kind: "port"`` CPU baseline timed by ``bench.py``.
"""
from __future__ import annotations

import math

import numpy as np

SCALE_ZP_BYTES = 8  # kvmanager.py:24


def quantize_rows(x, bits: int):
    """Quantize each row of a 2D array. Returns (codes u8, scale f64 (R,1), zero f64 (R,1)).

    Errors follow kvmanager.py:120-128 (ValueError).
    """
    if bits not in (4, 8):
        raise ValueError("bits must be 4 or 8")
    a = np.asarray(x, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if a.ndim != 2 or a.size == 0:
        raise ValueError("expected a non-empty channel-major 2D tensor")
    if not np.isfinite(a).all():
        raise ValueError("tensor contains non-finite values")
    qmax = float(2 ** bits - 1)
    s, z = params_from_minmax(a.min(axis=1), a.max(axis=1), bits)
    codes = np.clip(np.rint(a / s[:, None] + z[:, None]), 0.0, qmax).astype(np.uint8)
    return codes, s[:, None].copy(), z[:, None].copy()


def params_from_minmax(lo, hi, bits: int):
    """(scale, zero) per row from the row (min, max), kvmanager.py:130-146.  The data
    plane's transfer slabs store only the fp16 (min, max) of each group and recompute
    (scale, zero) with exactly this solve on upload."""
    qmax = float(2 ** bits - 1)
    lo = np.asarray(lo, dtype=np.float64).copy()
    hi = np.asarray(hi, dtype=np.float64).copy()
    flat = hi == lo
    # kvmanager.py:135-136 (degenerate rows: scale 1, zero -min)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(flat, 1.0, (hi - lo) / qmax)
        z = np.where(flat, -lo, np.rint(-lo / s))
    # kvmanager.py:141-146, per row: s <- (s*(qmax-z) - s*(0-z)) / qmax until fixed, <=32 passes
    active = ~flat
    for _ in range(32):
        if not active.any():
            break
        sa, za = s[active], z[active]
        nxt = (sa * (qmax - za) - sa * (0.0 - za)) / qmax
        moved = nxt != sa
        idx = np.flatnonzero(active)
        s[idx] = nxt
        active[idx[~moved]] = False
    return s, z


def params_absmax(lo, hi, bits: int):
    """(scale, zero) of the symmetric absmax mode from the row (min, max) -- the north
    star's alternative group-wise scheme.  PARITY UNPINNED: the reference has no such
    mode, so this restates the formula itself: a = max|x| = max(|min|, |max|),
    scale = a / (2^(b-1) - 1) (one correctly rounded float64 division; 1 when a == 0),
    zero = 2^(b-1); codes and values then use the reference's own formulas
    (kvmanager.py:148, :154)."""
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    a = np.maximum(np.abs(lo), np.abs(hi))
    qs = float(2 ** (bits - 1) - 1)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = np.where(a == 0.0, 1.0, a / qs)
    return s, np.full_like(s, float(2 ** (bits - 1)))


def quantize_rows_absmax(x, bits: int):
    """Symmetric absmax quantization of each row (see params_absmax); same errors and
    output layout as quantize_rows."""
    if bits not in (4, 8):
        raise ValueError("bits must be 4 or 8")
    a = np.asarray(x, dtype=np.float64)
    if a.ndim == 1:
        a = a.reshape(1, -1)
    if a.ndim != 2 or a.size == 0:
        raise ValueError("expected a non-empty channel-major 2D tensor")
    if not np.isfinite(a).all():
        raise ValueError("tensor contains non-finite values")
    qmax = float(2 ** bits - 1)
    s, z = params_absmax(a.min(axis=1), a.max(axis=1), bits)
    codes = np.clip(np.rint(a / s[:, None] + z[:, None]), 0.0, qmax).astype(np.uint8)
    return codes, s[:, None].copy(), z[:, None].copy()


def dequantize_rows(codes, scale, zero):
    """kvmanager.py:152-154: scale * (q - zero) in float64."""
    return np.asarray(scale, np.float64) * (np.asarray(codes).astype(np.float64)
                                            - np.asarray(zero, np.float64))


def kv_bytes(num_layers: int, hidden: int, tokens: int, bytes_per_value: int = 2) -> int:
    """kvmanager.py:61-66."""
    return 2 * num_layers * hidden * bytes_per_value * tokens


def quantized_kv_bytes(num_layers: int, hidden: int, tokens: int, bits: int) -> int:
    """kvmanager.py:69-82."""
    if tokens == 0:
        return 0
    ch = 2 * num_layers * hidden
    return math.ceil(bits / 8) * ch * tokens + ch * SCALE_ZP_BYTES


# ---- layout views used by the KV data plane (see DESIGN.md §KV layout) -------------
# A job's KV lives in HBM as kv[layer][kv][token][hidden] fp16 (hidden = heads*head_dim).
# Each group kind is a 2D (rows, row_len) view of it; the oracle is always
# quantize_rows(view).

def view_rows(kv, kind: str, group: int = 0, head_dim: int = 0):
    """Return the 2D row view (copy) of a [L,2,T,Hd] array for a group kind.

    kind "contig": rows are runs of `group` consecutive hidden values of one token.
    kind "channel": rows are (layer, kv, hidden column) along tokens (reference accounting).
    kind "head": rows are (layer, kv, head) over tokens x head_dim.
    """
    L, two, T, Hd = kv.shape
    if kind == "contig":
        return kv.reshape(-1, group)
    if kind == "channel":
        return np.ascontiguousarray(kv.transpose(0, 1, 3, 2)).reshape(L * two * Hd, T)
    if kind == "head":
        H = Hd // head_dim
        v = kv.reshape(L, two, T, H, head_dim).transpose(0, 1, 3, 2, 4)
        return np.ascontiguousarray(v).reshape(L * two * H, T * head_dim)
    raise ValueError(kind)


def rows_to_native(codes_rows, shape, kind: str, group: int = 0, head_dim: int = 0):
    """Inverse of view_rows for code arrays: back to [L,2,T,Hd] element order."""
    L, two, T, Hd = shape
    if kind == "contig":
        return codes_rows.reshape(shape)
    if kind == "channel":
        return np.ascontiguousarray(codes_rows.reshape(L, two, Hd, T).transpose(0, 1, 3, 2))
    if kind == "head":
        H = Hd // head_dim
        v = codes_rows.reshape(L, two, H, T, head_dim).transpose(0, 1, 3, 2, 4)
        return np.ascontiguousarray(v).reshape(shape)
    raise ValueError(kind)
