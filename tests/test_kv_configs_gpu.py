"""GPU parity at the BASELINE.json KV configurations' own shapes (not scaled down).

* C1 (configs[0]): 4 layers x 8 heads x 128 x 512 tokens fp16, INT8/INT4, per-head,
  per-channel and per-(token, head) views, through the drop-in quantize/dequantize and
  through the device slab -- SHA-256-equal to the REFERENCE's own outputs
  (tests/golden/kv_c1_full.npz, made by tests/golden/make_golden.py).
* C2 (configs[1]): one whole Llama-2-7B job (32 x 2 x 2048 x 4096 = 1 GiB fp16), INT8
  g=128, quantize+offload to pinned host memory, upload+dequantize back: every one of
  the 64 (layer, K|V) planes bit-exact against the C oracle -- codes, the (scale, zero)
  the host slab's fp16 (min, max) pair expands to, and the fp16 KV after the round trip.
  The reference accounting layout (per channel along 2048 tokens) the same way.
* C3 (configs[2]): INT4 g=64 packed at the ShareGPT p95 length (1488 tokens).
Reference: kvmanager.py:108-154 (quantize / dequantize)."""
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import pytest

from oracle import kv_oracle as ko
from tests.conftest import GOLDEN, c_quantize, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]

C1 = dict(layers=4, tokens=512, heads=8, head_dim=128)
C1_LAYOUTS = (("head", 0), ("channel", 0), ("contig", 128))


@pytest.fixture(scope="module")
def km():
    from paper_2410_23537_b200 import kvmanager
    return kvmanager


@pytest.fixture(scope="module")
def c1():
    from harness import synthetic
    z = np.load(os.path.join(GOLDEN, "kv_c1_full.npz"))
    kv = synthetic.kv_job(C1["layers"], C1["tokens"], C1["heads"] * C1["head_dim"], seed=0, job=0, group=128)
    assert ko_digest(kv) == str(z["kv_digest"]), "synthetic C1 input differs from the golden's"
    return kv, z


def ko_digest(a) -> str:
    import hashlib
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


@pytest.mark.parametrize("kind,group", C1_LAYOUTS)
@pytest.mark.parametrize("bits", [8, 4])
def test_c1_true_shape_dropin_api(km, c1, kind, group, bits):
    kv, z = c1
    tag = f"{kind}{group or ''}_b{bits}"
    view = ko.view_rows(kv, kind, group=group, head_dim=C1["head_dim"])
    assert list(view.shape) == z[tag + "_shape"].tolist()
    qt = km.quantize(view, bits)
    assert ko_digest(qt.values) == str(z[tag + "_codes_digest"]), np.argwhere(qt.values[:2] != z[tag + "_codes_head"])[:5]
    assert ko_digest(qt.scale) == str(z[tag + "_scale_digest"])
    assert ko_digest(qt.zero) == str(z[tag + "_zero_digest"])
    assert ko_digest(km.dequantize(qt)) == str(z[tag + "_deq_digest"])


@pytest.mark.parametrize("kind,group", C1_LAYOUTS)
@pytest.mark.parametrize("bits,packed", [(8, False), (4, True)])
def test_c1_true_shape_device_slab(km, c1, kind, group, bits, packed):
    """KV tensor -> alise_kv_quantize -> slab -> alise_kv_dequantize -> fp16 KV, per-head /
    per-channel / per-(token, head): codes and fp16 output equal the reference's."""
    import torch
    kv, z = c1
    tag = f"{kind}{group or ''}_b{bits}"
    k = "rows" if kind == "contig" else kind
    lay = km.KVLayout(C1["layers"], C1["tokens"], C1["heads"] * C1["head_dim"], C1["head_dim"], kind=k,
                      group=group or 128, bits=bits, packed=packed)
    g = lay.geometry()
    src = torch.from_numpy(kv).cuda()
    slab = torch.zeros(g["slab_bytes"], dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    km._lib.call("alise_kv_quantize", km._lib.C.byref(lay.desc()), km._lib.ptr(src), km._lib.ptr(slab),
                 km._lib.ptr(flag), km._lib.stream_ptr())
    out = torch.zeros_like(src)
    km._lib.call("alise_kv_dequantize", km._lib.C.byref(lay.desc()), km._lib.ptr(slab), km._lib.ptr(out),
                 km._lib.stream_ptr())
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    codes = _slab_codes(lay, slab.cpu().numpy(), kv.shape)
    assert ko_digest(ko.view_rows(codes, kind, group=group, head_dim=C1["head_dim"])) == \
        str(z[tag + "_codes_digest"])
    got = ko.view_rows(out.cpu().numpy(), kind, group=group, head_dim=C1["head_dim"])
    assert ko_digest(got) == str(z[tag + "_deq16_digest"])


def _plane_records(lay, slab):
    """Yield (plane index, codes bytes, fp16 (min, -max) pairs) of every (layer, K|V)
    plane of a slab: chunk records are [codes, native order][(min, -max) per group],
    sections 256-byte aligned."""
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


def _slab_codes(lay, slab, shape):
    parts = [c for _, c, _ in _plane_records(lay, slab)]
    native = np.concatenate(parts)
    if lay.packed:
        native = np.stack([native & 15, native >> 4], axis=1).reshape(-1)
    return native.reshape(shape)


def _job_parity(km, c_oracle, lay, kind, kv, threads=8):
    """Offload a whole job to pinned host memory and upload it back through the swap
    engine; check every plane against the C oracle.  Returns (planes, mismatching planes)."""
    import torch
    g = lay.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine()
    try:
        addr = pool.alloc(g["slab_bytes"])
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        eng.offload(lay, kv, addr, flag=flag)
        torch.cuda.synchronize()
        assert int(flag.item()) == 0
        slab = pool.view(addr, g["slab_bytes"])
        out = torch.zeros_like(kv)
        eng.upload(lay, addr, out)
        torch.cuda.synchronize()
        src_h = kv.cpu().numpy()
        out_h = out.cpu().numpy()
        bad = []

        def check(rec):
            p, codes, mm = rec
            layer, s = divmod(p, 2)
            x = src_h[layer, s][None, None]                   # [1, 1, T, hidden]
            rows = ko.view_rows(x, kind, group=lay.group, head_dim=lay.head_dim)
            c_ref, s_ref, z_ref = c_quantize(c_oracle, rows, lay.bits)
            if lay.packed:
                codes = np.stack([codes & 15, codes >> 4], axis=1).reshape(-1)
            got = ko.view_rows(np.asarray(codes).reshape(x.shape), kind, group=lay.group, head_dim=lay.head_dim)
            scale, zero = ko.params_from_minmax(mm[:, 0].astype(np.float64), -mm[:, 1].astype(np.float64), lay.bits)
            deq = np.empty(rows.shape)
            c_oracle.oracle_dequantize(c_ref.ctypes.data, s_ref.ctypes.data, z_ref.ctypes.data, rows.shape[0],
                                       rows.shape[1], deq.ctypes.data)
            back = ko.view_rows(out_h[layer, s][None, None], kind, group=lay.group, head_dim=lay.head_dim)
            ok = (np.array_equal(got, c_ref) and np.array_equal(scale, s_ref[:, 0])
                  and np.array_equal(zero, z_ref[:, 0]) and np.array_equal(back, deq.astype(np.float16)))
            if not ok:
                bad.append(p)

        with ThreadPoolExecutor(threads) as ex:   # the C oracle releases the GIL
            list(ex.map(check, _plane_records(lay, slab)))
        return lay.layers * 2, bad
    finally:
        eng.close()
        pool.close()


@pytest.mark.slow
def test_c2_whole_job_offload_upload_bit_exact(km, c_oracle):
    """C2: one whole 1 GiB Llama-2-7B job, INT8 g=128, every plane bit-exact."""
    from harness import synthetic
    lay = km.KVLayout(32, 2048, 4096, 128, kind="rows", group=128, bits=8)
    kv = synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=3, group=128)
    planes, bad = _job_parity(km, c_oracle, lay, "contig", kv)
    assert planes == 64 and not bad, bad


@pytest.mark.slow
def test_c2_reference_channel_layout_t2048(km, c_oracle):
    """The reference's accounting layout (kvmanager.py:72-75: one (scale, zero) per
    (layer, K|V, hidden channel) over the tokens) at T = 2048, 4 layers."""
    from harness import synthetic
    lay = km.KVLayout(4, 2048, 4096, 128, kind="channel", bits=8)
    kv = synthetic.kv_job_torch(4, 2048, 4096, seed=0, job=5, group=128)
    planes, bad = _job_parity(km, c_oracle, lay, "channel", kv)
    assert planes == 8 and not bad, bad


@pytest.mark.slow
def test_c3_int4_g64_packed_p95_job(km, c_oracle):
    """C3: INT4 g=64 packed two per byte, a ShareGPT p95-length job (1488 tokens)."""
    from harness import synthetic
    lay = km.KVLayout(8, 1488, 4096, 128, kind="rows", group=64, bits=4, packed=True)
    kv = synthetic.kv_job_torch(8, 1488, 4096, seed=0, job=11, group=64)
    planes, bad = _job_parity(km, c_oracle, lay, "contig", kv)
    assert planes == 16 and not bad, bad
