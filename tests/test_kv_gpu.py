"""GPU parity: the CUDA quantizer / dequantizer / swap path vs the oracle and the
reference golden vectors.  Bar: codes, scale, zero bit-exact; dequantized float64
bit-exact; fp16 dequant = fp16(reference float64) (0 ulp)."""
import numpy as np
import pytest

from oracle import kv_oracle as ko
from tests.conftest import c_quantize, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]

C1_CASES = [("contig", 32), ("contig", 64), ("channel", 0), ("head", 0)]


@pytest.fixture(scope="module")
def km():
    from paper_2410_23537_b200 import kvmanager
    return kvmanager


def _layout(km, kv, kind, group, bits, packed=False, ppc=0):
    L, _, T, Hd = kv.shape
    k = "rows" if kind == "contig" else kind
    return km.KVLayout(L, T, Hd, 32, kind=k, group=group or 128, bits=bits, packed=packed,
                       planes_per_chunk=ppc)


def _slab_to_rows(km, layout, slab, shape, kind, group, head_dim):
    """Decode a host/device slab into (codes in reference row order, scale, zero).  A chunk
    record is [codes, native order][fp16 (min, -max) per group]; (scale, zero) follow from
    (min, max) by the reference solve (oracle params_from_minmax)."""
    import math
    g = layout.geometry()
    L, two, T, Hd = shape
    planes = L * two
    ppc = math.ceil(planes / g["n_chunks"]) if layout.planes_per_chunk <= 0 else min(layout.planes_per_chunk, planes)
    rows_pp = g["rows"] // planes
    per_plane_codes = T * Hd // (2 if layout.packed else 1)
    a256 = lambda x: (x + 255) // 256 * 256
    codes, mms = [], []
    for c in range(g["n_chunks"]):
        np_ = min(ppc, planes - c * ppc)
        base = c * g["chunk_bytes"]
        cs = a256(np_ * per_plane_codes)
        codes.append(slab[base: base + np_ * per_plane_codes])
        mms.append(slab[base + cs: base + cs + np_ * rows_pp * 4].view(np.float16).reshape(-1, 2))
    native = np.concatenate(codes)
    if layout.packed:
        lo, hi = native & 15, native >> 4
        native = np.stack([lo, hi], axis=1).reshape(-1)
    native = native.reshape(shape)
    rows = ko.view_rows(native, kind, group=group, head_dim=head_dim)
    mm = np.concatenate(mms).astype(np.float64)
    scale, zero = ko.params_from_minmax(mm[:, 0], -mm[:, 1], layout.bits)
    return rows, scale[:, None], zero.astype(np.float32).astype(np.float64)[:, None]


# ----------------------------------------------------------------- drop-in API
@pytest.mark.parametrize("kind,group", C1_CASES)
@pytest.mark.parametrize("bits", [4, 8])
def test_quantize_dropin_matches_reference_golden(km, kv_golden, kind, group, bits):
    kv = kv_golden["c1_kv"]
    view = ko.view_rows(kv, kind, group=group, head_dim=32)
    qt = km.quantize(view, bits)
    tag = f"c1_{kind}{group or ''}_b{bits}"
    assert qt.values.dtype == np.uint8 and qt.scale.shape == (view.shape[0], 1)
    assert np.array_equal(qt.values, kv_golden[tag + "_codes"])
    assert np.array_equal(qt.scale, kv_golden[tag + "_scale"])
    assert np.array_equal(qt.zero, kv_golden[tag + "_zero"])
    assert np.array_equal(km.dequantize(qt), kv_golden[tag + "_deq"])


def test_quantize_dropin_float64_cases(km, kv_golden):
    for i in range(40):
        x = kv_golden[f"f64_{i}_x"]
        bits = int(kv_golden[f"f64_{i}_bits"])
        qt = km.quantize(x, bits)
        assert np.array_equal(qt.values, kv_golden[f"f64_{i}_codes"]), i
        assert np.array_equal(qt.scale, kv_golden[f"f64_{i}_scale"]), i
        assert np.array_equal(qt.zero, kv_golden[f"f64_{i}_zero"]), i
        assert np.array_equal(km.dequantize(qt), kv_golden[f"f64_{i}_deq"]), i


def test_reference_known_answers_through_gpu(km):
    # pkg/tests/test_kvmanager.py:53-126, run through the CUDA path
    qt = km.quantize(np.array([[0.0, 1.0]]), 8)
    assert qt.scale[0, 0] == 1.0 / 255.0 and qt.zero[0, 0] == 0.0
    assert qt.values[0].tolist() == [0, 255]
    deq = km.dequantize(qt)
    assert deq[0, 1] == 1.0 and deq[0, 0] == 0.0
    gen = np.random.default_rng(5)
    for _ in range(50):
        c = float(gen.uniform(-750, 750))
        x = np.full((1, int(gen.integers(1, 40))), c)
        for bits in (4, 8):
            assert np.array_equal(km.dequantize(km.quantize(x, bits)), x)
    gen = np.random.default_rng(17)
    for i in range(100):
        bits = 4 if i % 2 else 8
        length = int(gen.integers(1, 513))
        sc = 10.0 ** gen.uniform(-2, 2)
        x = gen.uniform(-sc, sc, size=(3, length))
        if i % 3 == 1:
            x = np.abs(x)
        elif i % 3 == 2:
            x = -np.abs(x)
        qt = km.quantize(x, bits)
        assert np.all(np.abs(x - km.dequantize(qt)) <= qt.scale / 2 + 1e-9)
        ref = ko.quantize_rows(x, bits)
        assert np.array_equal(qt.values, ref[0]) and np.array_equal(qt.scale, ref[1])
    gen = np.random.default_rng(29)
    for i in range(60):
        bits = 4 if i % 2 else 8
        x = gen.uniform(-1, 1, size=(2, int(gen.integers(2, 257))))
        y1 = km.dequantize(km.quantize(x, bits))
        qt2 = km.quantize(y1, bits)
        assert np.array_equal(km.quantize(x, bits).values, qt2.values)
        assert np.array_equal(y1, km.dequantize(qt2))
    with pytest.raises(ValueError):
        km.quantize(np.ones((1, 4)), 5)
    with pytest.raises(ValueError):
        km.quantize(np.ones((1, 0)), 8)
    with pytest.raises(ValueError):
        km.quantize(np.array([[1.0, np.nan]]), 8)
    with pytest.raises(ValueError):
        km.quantize(np.array([[1.0, np.inf]], dtype=np.float16), 8)


@pytest.mark.parametrize("row_len", [8, 16, 24, 64, 96, 128, 200, 256, 264, 1000, 65536])
@pytest.mark.parametrize("bits", [4, 8])
def test_quantize_fp16_row_lengths_vs_c_oracle(km, c_oracle, row_len, bits):
    g = np.random.default_rng(row_len * 10 + bits)
    rows = max(3, min(4000, 400000 // row_len))
    x = (g.standard_normal((rows, row_len)) * 10.0 ** g.uniform(-3, 3, size=(rows, 1))).astype(np.float16)
    x[::5] = np.abs(x[::5]) + np.float16(200)
    x[1::9] = -np.abs(x[1::9]) - np.float16(1000)
    x[2::11] = x[2::11, :1]
    qt = km.quantize(x, bits)
    c, s, z = c_quantize(c_oracle, x, bits)
    assert np.array_equal(qt.values, c)
    assert np.array_equal(qt.scale, s)
    assert np.array_equal(qt.zero, z)


def test_quantize_1d_and_float32(km):
    x = np.linspace(-3, 7, 1001).astype(np.float32)
    qt = km.quantize(x, 8)
    ref = ko.quantize_rows(x, 8)
    assert qt.values.shape == (1, 1001)
    assert np.array_equal(qt.values, ref[0]) and np.array_equal(qt.scale, ref[1])


def test_dequantize_fp16_is_one_rounding_of_reference(km, kv_golden):
    import torch
    kv = kv_golden["c1_kv"]
    view = ko.view_rows(kv, "contig", group=64, head_dim=32)
    qt = km.quantize(view, 8)
    out = km.dequantize_tensor(qt, out_dtype=torch.float16).cpu().numpy()
    assert np.array_equal(out, km.dequantize(qt).astype(np.float16))


# ----------------------------------------------------------------- KV data plane
@pytest.mark.parametrize("kind,group", C1_CASES)
@pytest.mark.parametrize("bits,packed", [(8, False), (4, False), (4, True)])
def test_kv_device_slab_matches_reference(km, kv_golden, kind, group, bits, packed):
    import torch
    kv = kv_golden["c1_kv"]
    layout = _layout(km, kv, kind, group, bits, packed, ppc=1)
    g = layout.geometry()
    src = torch.from_numpy(kv).cuda()
    slab = torch.zeros(g["slab_bytes"], dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    km._lib.call("alise_kv_quantize", km._lib.C.byref(layout.desc()), km._lib.ptr(src), km._lib.ptr(slab),
                 km._lib.ptr(flag), km._lib.stream_ptr())
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    rows, scale, zero = _slab_to_rows(km, layout, slab.cpu().numpy(), kv.shape, kind, group, 32)
    tag = f"c1_{kind}{group or ''}_b{bits}"
    assert np.array_equal(rows, kv_golden[tag + "_codes"])
    assert np.array_equal(scale, kv_golden[tag + "_scale"])
    assert np.array_equal(zero, kv_golden[tag + "_zero"])
    out = torch.empty_like(src)
    km._lib.call("alise_kv_dequantize", km._lib.C.byref(layout.desc()), km._lib.ptr(slab), km._lib.ptr(out),
                 km._lib.stream_ptr())
    ref = ko.rows_to_native(kv_golden[tag + "_deq"], kv.shape, kind, group=group, head_dim=32)
    assert np.array_equal(out.cpu().numpy(), ref.astype(np.float16))


@pytest.mark.parametrize("mode", ["staged", "zerocopy"])
@pytest.mark.parametrize("kind,group,bits,packed", [("contig", 64, 8, False), ("contig", 32, 4, True),
                                                    ("channel", 0, 8, False), ("head", 0, 4, False)])
def test_swap_round_trip_through_host(km, kv_golden, mode, kind, group, bits, packed):
    import torch
    kv = kv_golden["c1_kv"]
    layout = _layout(km, kv, kind, group, bits, packed, ppc=1)
    g = layout.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine(mode=mode)
    try:
        src = torch.from_numpy(kv).cuda()
        addr = pool.alloc(g["slab_bytes"])
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        eng.offload(layout, src, addr, flag=flag)
        torch.cuda.synchronize()
        rows, scale, zero = _slab_to_rows(km, layout, pool.view(addr, g["slab_bytes"]).copy(), kv.shape,
                                          kind, group, 32)
        tag = f"c1_{kind}{group or ''}_b{bits}"
        assert np.array_equal(rows, kv_golden[tag + "_codes"])
        assert np.array_equal(scale, kv_golden[tag + "_scale"])
        out = torch.zeros_like(src)
        eng.upload(layout, addr, out)
        torch.cuda.synchronize()
        ref = ko.rows_to_native(kv_golden[tag + "_deq"], kv.shape, kind, group=group, head_dim=32)
        assert np.array_equal(out.cpu().numpy(), ref.astype(np.float16))
    finally:
        eng.close()
        pool.close()


def test_device_memory_state_moves_real_bytes(km, kv_golden):
    import torch
    kv = kv_golden["c1_kv"]
    layout = _layout(km, kv, "contig", 64, 8)
    m = km.ModelConfig("toy", 4, 2, 128)
    link = km.quantized_kv_bytes(m, 64, 8)
    gpu_b = km.kv_bytes(m, 64)
    ms = km.DeviceMemoryState(gpu_capacity=10 * gpu_b, cpu_capacity=10 * link, pcie_bytes_per_ms=25e6,
                              host_pool_bytes=1 << 24)
    src = torch.from_numpy(kv).cuda()
    ms.bind(7, src, layout)
    ms.reserve_gpu(gpu_b)
    cmd = ms.start_offload(7, link, gpu_b, now_us=0)
    assert cmd.complete_us == ms.transfer_us(link)
    ms.complete(cmd)
    assert ms.gpu_used == 0 and ms.cpu_used == link
    src.zero_()
    cmd = ms.start_upload(7, link, gpu_b, now_us=cmd.complete_us)
    ms.complete(cmd)
    assert ms.cpu_used == 0 and ms.gpu_used == gpu_b
    ref = ko.rows_to_native(kv_golden["c1_contig64_b8_deq"], kv.shape, "contig", group=64)
    assert np.array_equal(src.cpu().numpy(), ref.astype(np.float16))


def test_nonfinite_kv_flagged_at_complete(km):
    import torch
    layout = km.KVLayout(1, 16, 64, 32, kind="rows", group=64, bits=8)
    kv = torch.randn(1, 2, 16, 64, device="cuda").half()
    kv[0, 1, 3, 5] = float("inf")
    ms = km.DeviceMemoryState(gpu_capacity=1 << 30, cpu_capacity=1 << 30, pcie_bytes_per_ms=25e6,
                              host_pool_bytes=1 << 20)
    ms.bind(1, kv, layout)
    ms.reserve_gpu(4096)
    cmd = ms.start_offload(1, 2048, 4096, 0)
    with pytest.raises(ValueError):
        ms.complete(cmd)


@pytest.mark.slow
def test_llama7b_job_round_trip_properties(km):
    """Full C2-size job (1 GiB fp16): bit-exact against the C oracle on sampled rows,
    and the reference's error bound |x - deq| <= scale/2 on every element."""
    import torch
    from harness import synthetic
    layout = km.KVLayout(32, 2048, 4096, 128, kind="rows", group=128, bits=8)
    kv = synthetic.kv_job_torch(32, 2048, 4096, seed=0, job=3, group=128)
    g = layout.geometry()
    slab = torch.empty(g["slab_bytes"], dtype=torch.uint8, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    km._lib.call("alise_kv_quantize", km._lib.C.byref(layout.desc()), km._lib.ptr(kv), km._lib.ptr(slab),
                 km._lib.ptr(flag), km._lib.stream_ptr())
    out = torch.empty_like(kv)
    km._lib.call("alise_kv_dequantize", km._lib.C.byref(layout.desc()), km._lib.ptr(slab), km._lib.ptr(out),
                 km._lib.stream_ptr())
    torch.cuda.synchronize()
    err = (kv.float() - out.float()).abs().view(-1, 128).amax(dim=1)
    span = (kv.float().view(-1, 128).amax(1) - kv.float().view(-1, 128).amin(1))
    # |x - deq| <= scale/2 (+ fp16 output rounding of the dequantized value)
    bound = span / 255 / 2 + kv.float().view(-1, 128).abs().amax(1) * 2 ** -11 + 1e-6
    assert bool((err <= bound).all())


@pytest.mark.slow
def test_c5_replay_matches_reference_ledger():
    """Config-5 replay (tests/golden/c5_swaps.json.gz, recorded from the reference
    simulator): every swap call moves real quantized KV through DeviceMemoryState, the
    ledger equals the reference after every call, and sampled planes of each job's KV
    after its first round trip equal the oracle's quantize/dequantize of its original."""
    import os

    from harness import replay
    from tests.conftest import GOLDEN
    rec = replay.load(os.path.join(GOLDEN, "c5_swaps.json.gz"))
    out = replay.replay(rec, replica=3, max_events=1200)
    assert out["swaps_out"] > 100 and out["data_checked"] > 10
    assert out["data_mismatches"] == 0


@pytest.mark.parametrize("bits", [4, 8])
def test_constant_divisor_division_is_ddiv_rn(bits):
    """qmath.cuh qdiv (hoisted reciprocal) == __ddiv_rn bit for bit: random doubles over
    the whole exponent range, the snap loop's operands (s*(qmax-z) - s*(-z) for fp16
    (min, max) pairs) and the special values."""
    import torch
    from paper_2410_23537_b200 import _lib
    g = np.random.default_rng(bits)
    qmax = float((1 << bits) - 1)
    parts = [g.standard_normal(1 << 20) * np.exp2(g.integers(-1070, 1020, 1 << 20)),
             g.integers(1, 1 << 62, 1 << 20, dtype=np.int64).view(np.float64)]
    mn = g.standard_normal(1 << 20).astype(np.float16).astype(np.float64) * 100
    mx = mn + np.abs(g.standard_normal(1 << 20).astype(np.float16).astype(np.float64)) * 100 + 2.0 ** -20
    s = (mx - mn) / qmax
    z = np.rint(-mn / s)
    parts += [mx - mn, s * (qmax - z) - s * (0 - z)]
    parts.append(np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 5e-324, 1.7e308, qmax, -qmax, 1.0]))
    x = np.concatenate(parts)
    x = x[np.isfinite(x) | np.isnan(x)]
    xd = torch.from_numpy(x).cuda()
    bad = torch.zeros(1, dtype=torch.int64, device="cuda")
    _lib.call("alise_selftest_qdiv", _lib.ptr(xd), x.size, bits, _lib.ptr(bad), _lib.stream_ptr())
    torch.cuda.synchronize()
    # NaN inputs compare by bits too (both paths return the canonical quiet NaN)
    assert int(bad.item()) == 0


# ----------------------------------------------------------------- token-range (delta) transfers
@pytest.mark.parametrize("group,bits,packed,ppc", [(128, 8, False, 0), (64, 4, True, 3), (64, 8, False, 1)])
def test_delta_offload_equals_full_offload(km, group, bits, packed, ppc):
    """Offloading a job in token ranges (as it grows) writes exactly the bytes of one full
    offload; uploading in ranges restores exactly the full upload (kvmanager.py:108-154
    applied per (token, group) row)."""
    import torch
    from harness import synthetic
    L, T, H = 3, 96, 4096
    kv = synthetic.kv_job_torch(L, T, H, seed=0, job=5, group=group, device="cuda")
    lay = km.KVLayout(L, T, H, 128, kind="rows", group=group, bits=bits, packed=packed, planes_per_chunk=ppc)
    g = lay.geometry()
    pool = km.HostSlabPool(2 * g["slab_bytes"] + 8192)
    eng = km.KVSwapEngine()
    try:
        full, delta = pool.alloc(g["slab_bytes"]), pool.alloc(g["slab_bytes"])
        pool.view(full, g["slab_bytes"])[:] = 0
        pool.view(delta, g["slab_bytes"])[:] = 0
        flag = torch.zeros(1, dtype=torch.int32, device="cuda")
        eng.offload(lay, kv, full, flag=flag)
        for t0, t1 in [(0, 8), (8, 40), (40, 41), (41, 96)]:
            eng.offload(lay, kv, delta, flag=flag, tokens=(t0, t1))
        torch.cuda.synchronize()
        assert np.array_equal(pool.view(full, g["slab_bytes"]), pool.view(delta, g["slab_bytes"]))
        ref = torch.zeros_like(kv)
        eng.upload(lay, full, ref)
        out = torch.zeros_like(kv)
        for t0, t1 in [(0, 33), (33, 96)]:
            eng.upload(lay, delta, out, tokens=(t0, t1))
        part = torch.zeros_like(kv)
        eng.upload(lay, delta, part, tokens=(0, 50))
        torch.cuda.synchronize()
        assert torch.equal(out, ref)
        assert torch.equal(part[:, :, :50], ref[:, :, :50]) and not part[:, :, 50:].any()
        assert int(flag.item()) == 0
    finally:
        eng.close()
        pool.close()


def test_delta_transfer_errors(km):
    import torch
    lay = km.KVLayout(1, 32, 256, 64, kind="channel", bits=8)
    eng = km.KVSwapEngine()
    pool = km.HostSlabPool(1 << 20)
    try:
        kv = torch.zeros(1, 2, 32, 256, dtype=torch.float16, device="cuda")
        addr = pool.alloc(lay.geometry()["slab_bytes"])
        with pytest.raises(ValueError):
            eng.offload(lay, kv, addr, tokens=(0, 8))     # groups span tokens
        lay = km.KVLayout(1, 32, 256, 64, kind="rows", group=64, bits=8)
        with pytest.raises(ValueError):
            eng.offload(lay, kv, addr, tokens=(8, 40))    # beyond the token capacity
        with pytest.raises(ValueError):
            eng.upload(lay, addr, kv, tokens=(5, 5))      # empty range
    finally:
        eng.close()
        pool.close()


def test_c5_replay_delta_offload_same_ledger():
    """Config-5 replay with incremental (delta) offload: the ledger still equals the
    reference after every call, fewer bytes cross the link, and after every upload
    sampled planes of each job's KV equal the oracle's quantize/dequantize of its
    ORIGINAL values (each token is quantized once; a full re-offload would re-quantize
    fp16-rounded dequantized values)."""
    import os

    from harness import replay
    from tests.conftest import GOLDEN
    rec = replay.load(os.path.join(GOLDEN, "c5_swaps.json.gz"))
    full = replay.replay(rec, replica=3, max_events=900, check_data=False)
    dlt = replay.replay(rec, replica=3, max_events=900, delta=True)
    assert dlt["data_mismatches"] == 0 and dlt["data_checked"] > 50
    assert dlt["link_bytes_moved"] < full["link_bytes_moved"]


# ----------------------------------------------------------------- absmax mode
@pytest.mark.parametrize("bits", [4, 8])
def test_absmax_dropin_matches_restated_oracle(km, kv_golden, bits):
    """mode="absmax" (symmetric, north star; parity against the restated oracle --
    the reference has no such mode): codes / scale / zero / float64 values bit-exact on
    the C1 views and on float64 rows incl. all-zero and single-sign rows."""
    kv = kv_golden["c1_kv"]
    cases = [ko.view_rows(kv, kind, group=g, head_dim=32) for kind, g in C1_CASES]
    g = np.random.default_rng(bits)
    x = g.standard_normal((40, 96)) * 10.0 ** g.uniform(-2, 2, size=(40, 1))
    x[5] = 0.0
    x[6] = np.abs(x[6]) + 3.0
    x[7] = 7.0
    cases.append(x)
    for v in cases:
        qt = km.quantize(v, bits, mode="absmax")
        c, s, z = ko.quantize_rows_absmax(v, bits)
        assert np.array_equal(qt.values, c) and np.array_equal(qt.scale, s) and np.array_equal(qt.zero, z)
        assert np.array_equal(km.dequantize(qt), ko.dequantize_rows(c, s, z))


@pytest.mark.parametrize("kind,group,bits,packed", [("contig", 64, 4, True), ("contig", 128, 8, False),
                                                    ("channel", 0, 8, False), ("head", 0, 4, True)])
def test_absmax_swap_round_trip(km, kind, group, bits, packed):
    """KV data plane in absmax mode: quantize+offload to pinned host, upload+dequantize;
    every plane vs the restated oracle (codes, the (scale, zero) the slab's fp16
    (min, max) expands to, fp16 output)."""
    import torch

    from harness import parity, synthetic
    L, T, H = 4, 160, 1024
    k = "rows" if kind == "contig" else kind
    lay = km.KVLayout(L, T, H, 128, kind=k, group=group or 128, bits=bits, packed=packed, mode="absmax")
    kv = synthetic.kv_job_torch(L, T, H, seed=3, job=1, group=group or 64)
    g = lay.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine()
    try:
        addr = pool.alloc(g["slab_bytes"])
        eng.offload(lay, kv, addr)
        torch.cuda.synchronize()
        out = torch.zeros_like(kv)
        eng.upload(lay, addr, out)
        torch.cuda.synchronize()
        planes, _vals, bad = parity.kv_check_planes(lay, kv.cpu().numpy(), pool.view(addr, g["slab_bytes"]),
                                                    out.cpu().numpy())
        assert planes == 2 * L and not bad, bad
    finally:
        eng.close()
        pool.close()


# ----------------------------------------------------------------- column kinds, ragged T
@pytest.mark.parametrize("kind,bits,packed", [("channel", 8, False), ("channel", 4, True), ("head", 8, False),
                                              ("head", 4, False)])
@pytest.mark.parametrize("T", [1, 5, 37, 300, 6017, 12900])
def test_cols_ragged_tokens_through_host(km, kind, bits, packed, T):
    """Column kinds at token counts that leave cluster ranks empty or partial (T < 8,
    T not a multiple of 8 x 16) and beyond the single-pass kernel's shared-memory limit
    (T = 12900 takes the two-pass kernel): every plane vs the C oracle through pinned host."""
    import torch

    from harness import parity, synthetic
    L, H = 1, 256
    lay = km.KVLayout(L, T, H, 128, kind=kind, bits=bits, packed=packed)
    kv = synthetic.kv_job_torch(L, T, H, seed=T, job=2, group=64)
    g = lay.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine()
    try:
        addr = pool.alloc(g["slab_bytes"])
        eng.offload(lay, kv, addr)
        torch.cuda.synchronize()
        out = torch.zeros_like(kv)
        eng.upload(lay, addr, out)
        torch.cuda.synchronize()
        planes, _vals, bad = parity.kv_check_planes(lay, kv.cpu().numpy(), pool.view(addr, g["slab_bytes"]),
                                                    out.cpu().numpy())
        assert planes == 2 * L and not bad, bad
    finally:
        eng.close()
        pool.close()


# ----------------------------------------------------------------- snap-loop cycles
@pytest.mark.parametrize("bits,group", [(4, 64), (8, 128), (8, 64)])
def test_snap_loop_cycles_match_the_reference_loop(km, bits, group):
    """Rows whose snap loop never settles (2-, 3- and 4-cycles, ~0.7% of real-valued
    rows) end at the reference's 32nd iterate: the kernels read it off the detected
    cycle (qmath.cuh snap_scale).  The rows are selected on the host by running the
    reference's loop and kept only if still moving after 8 passes; they go through the
    drop-in quantize (tile kernel), the transfer slab (k_expand_params on upload) and
    must equal the oracle (plain 32-pass loop) bit for bit."""
    import torch

    from harness import synthetic
    kv = synthetic.kv_job(8, 256, 1024, seed=bits + group, job=4, group=group)
    x = kv.reshape(-1, group).astype(np.float64)
    q = float(2 ** bits - 1)
    mn, mx = x.min(1), x.max(1)
    live = mx != mn
    s = np.where(live, (mx - mn) / q, 1.0)
    z = np.where(live, np.rint(-mn / s), -mn)
    for _ in range(8):
        s = np.where(live, (s * (q - z) - s * (0.0 - z)) / q, 1.0)
    s9 = np.where(live, (s * (q - z) - s * (0.0 - z)) / q, 1.0)
    moving = np.flatnonzero(live & (s9 != s))
    assert len(moving) > 20, len(moving)
    rows = x[moving]
    qt = km.quantize(rows, bits)
    c, sc, zc = ko.quantize_rows(rows, bits)
    assert np.array_equal(qt.scale, sc) and np.array_equal(qt.zero, zc) and np.array_equal(qt.values, c)
    # through a transfer slab (fp16 (min, max) -> k_expand_params on upload)
    L, T = 1, 2 * len(moving) // (1024 // group) + 2
    T = (T + 1) // 2 * 2
    plane = np.zeros((L, 2, T, 1024), dtype=np.float16)
    flat = plane.reshape(-1, group)
    flat[:len(moving)] = rows.astype(np.float16)
    lay = km.KVLayout(L, T, 1024, 128, kind="rows", group=group, bits=bits, packed=bits == 4)
    g = lay.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine()
    try:
        src = torch.from_numpy(plane).cuda()
        addr = pool.alloc(g["slab_bytes"])
        eng.offload(lay, src, addr)
        out = torch.zeros_like(src)
        eng.upload(lay, addr, out)
        torch.cuda.synchronize()
        c4, s4, z4 = ko.quantize_rows(flat.astype(np.float64), bits)
        ref = ko.dequantize_rows(c4, s4, z4).astype(np.float16).reshape(plane.shape)
        assert np.array_equal(out.cpu().numpy(), ref)
    finally:
        eng.close()
        pool.close()


@pytest.mark.parametrize("head_dim,hidden", [(16, 256), (64, 384), (128, 384), (256, 512)])
@pytest.mark.parametrize("bits,packed", [(8, False), (4, True)])
def test_head_kind_widths_through_host(km, head_dim, hidden, bits, packed):
    """Per-head groups of every width the kernels dispatch on: 16/64 (64-column cluster
    strips), 128 (128-column strips), 256 (generic path), with hidden sizes that are
    not multiples of 128 -- every plane vs the C oracle through pinned host."""
    import torch

    from harness import parity, synthetic
    L, T = 1, 37
    lay = km.KVLayout(L, T, hidden, head_dim, kind="head", bits=bits, packed=packed)
    kv = synthetic.kv_job_torch(L, T, hidden, seed=head_dim, job=3, group=16)
    g = lay.geometry()
    pool = km.HostSlabPool(g["slab_bytes"] + 4096)
    eng = km.KVSwapEngine()
    try:
        addr = pool.alloc(g["slab_bytes"])
        eng.offload(lay, kv, addr)
        torch.cuda.synchronize()
        out = torch.zeros_like(kv)
        eng.upload(lay, addr, out)
        torch.cuda.synchronize()
        planes, _vals, bad = parity.kv_check_planes(lay, kv.cpu().numpy(), pool.view(addr, g["slab_bytes"]),
                                                    out.cpu().numpy())
        assert planes == 2 * L and not bad, bad
    finally:
        eng.close()
        pool.close()
