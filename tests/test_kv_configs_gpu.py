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
import numpy as np
import pytest

from oracle import kv_oracle as ko
from tests.conftest import GOLDEN, have_gpu

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


def _slab_codes(lay, slab, shape):
    from harness import parity
    parts = [c for _, c, _ in parity.plane_records(lay, slab)]
    native = np.concatenate(parts)
    if lay.packed:
        native = np.stack([native & 15, native >> 4], axis=1).reshape(-1)
    return native.reshape(shape)


def _job_parity(km, lay, kv):
    """Offload a whole job to pinned host memory and upload it back through the swap
    engine; check every plane against the C oracle (harness/parity.py)."""
    import torch
    from harness import parity
    g = lay.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine()
    try:
        addr = pool.alloc(g["slab_bytes"])
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        eng.offload(lay, kv, addr, flag=flag)
        torch.cuda.synchronize()
        assert int(flag.item()) == 0
        out = torch.zeros_like(kv)
        eng.upload(lay, addr, out)
        torch.cuda.synchronize()
        planes, _values, bad = parity.kv_check_planes(lay, kv.cpu().numpy(), pool.view(addr, g["slab_bytes"]),
                                                      out.cpu().numpy())
        return planes, bad
    finally:
        eng.close()
        pool.close()


@pytest.mark.slow
def test_c2_whole_job_offload_upload_bit_exact(km):
    """C2: one whole 1 GiB Llama-2-7B job, INT8 g=128, every plane bit-exact."""
    from harness import synthetic
    lay = km.KVLayout(32, 2048, 4096, 128, kind="rows", group=128, bits=8)
    kv = synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=3, group=128)
    planes, bad = _job_parity(km, lay, kv)
    assert planes == 64 and not bad, bad


@pytest.mark.slow
def test_c2_reference_channel_layout_t2048(km):
    """The reference's accounting layout (kvmanager.py:72-75: one (scale, zero) per
    (layer, K|V, hidden channel) over the tokens) at T = 2048, 4 layers."""
    from harness import synthetic
    lay = km.KVLayout(4, 2048, 4096, 128, kind="channel", bits=8)
    kv = synthetic.kv_job_torch(4, 2048, 4096, seed=0, job=5, group=128)
    planes, bad = _job_parity(km, lay, kv)
    assert planes == 8 and not bad, bad


@pytest.mark.slow
def test_c3_int4_g64_packed_p95_job(km):
    """C3: INT4 g=64 packed two per byte, a ShareGPT p95-length job (1488 tokens)."""
    from harness import synthetic
    lay = km.KVLayout(8, 1488, 4096, 128, kind="rows", group=64, bits=4, packed=True)
    kv = synthetic.kv_job_torch(8, 1488, 4096, seed=0, job=11, group=64)
    planes, bad = _job_parity(km, lay, kv)
    assert planes == 16 and not bad, bad


# ----------------------------------------------------------------- C4 at its own shape
@pytest.mark.slow
def test_c4_full_db_1m_x_768_batch_4096():
    """C4 (configs[3]): 1M x 768 fp32 DB with 1000 planted duplicate groups, one batch of
    4096 queries through LengthPredictor.predict_batch; 256 sampled queries plus one
    query aimed at each of 100 planted duplicate groups (11-way exact ties) checked
    against the oracle: top-8 seqs/lens/sims bit-exact, predicted lengths exact."""
    import torch

    from harness import parity, synthetic
    from paper_2410_23537_b200 import predictor as pr
    N, D, B = 1_000_000, 768, 4096
    db, lens = synthetic.predictor_db_torch(N, D, seed=0, dup_groups=1000, device="cuda")
    Q = synthetic.predictor_queries_torch(db, B, seed=1)
    # queries aimed at planted groups: rows that occur more than once (hash of the row)
    h = db @ torch.randn(D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(3))
    uniq, inv, counts = torch.unique(h, return_inverse=True, return_counts=True)
    dup_rows = torch.nonzero(counts[inv] > 1).flatten()
    grp_first = {}
    for r in dup_rows.tolist():
        grp_first.setdefault(int(inv[r]), r)
    targets = list(grp_first.values())[:100]
    gq = torch.Generator(device="cuda").manual_seed(4)
    Q[:100] = db[targets] + 0.01 * torch.randn((len(targets), D), device="cuda", generator=gq)
    Q[:100] /= Q[:100].norm(dim=1, keepdim=True)
    store = pr.VectorStore(D, N, dtype=np.float32)
    store.add_batch(db, lens)
    reg = pr.FallbackRegressor(D, 32, seed=0)
    reg.b2 = 5.0
    p = pr.LengthPredictor(pr.PredictorConfig(dimension=D, db_capacity=N), regressor=reg, store=store)
    sims, seqs, slens, cnt, _ = store.search_batch(Q, 8)
    out, ret = p.predict_batch(Q)
    torch.cuda.synchronize()
    g = np.random.default_rng(0)
    idx = np.concatenate([np.arange(100), np.sort(g.choice(np.arange(100, B), 256, replace=False))])
    bad = parity.pred_check(db.cpu().numpy(), lens.cpu().numpy(), Q.cpu().numpy(), idx, sims.cpu().numpy(),
                            seqs.cpu().numpy(), slens.cpu().numpy(), cnt.cpu().numpy(), out.cpu().numpy(),
                            ret.cpu().numpy(), reg.w1, reg.b1, reg.w2, reg.b2)
    assert not bad, bad[:10]
    assert len(targets) == 100 and int(ret[:100].sum()) == 100
