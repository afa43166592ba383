"""CPU: pin the KV oracle (numpy + C restatements) to the reference's golden vectors
and to the reference's own known-answer tests (pkg/tests/test_kvmanager.py)."""
import numpy as np
import pytest

from oracle import kv_oracle as ko
from tests.conftest import c_quantize

C1_CASES = [("contig", 32), ("contig", 64), ("channel", 0), ("head", 0)]


@pytest.mark.parametrize("kind,group", C1_CASES)
@pytest.mark.parametrize("bits", [4, 8])
def test_numpy_oracle_matches_reference_golden(kv_golden, kind, group, bits):
    kv = kv_golden["c1_kv"]
    view = ko.view_rows(kv, kind, group=group, head_dim=32)
    codes, scale, zero = ko.quantize_rows(view, bits)
    tag = f"c1_{kind}{group or ''}_b{bits}"
    assert np.array_equal(codes, kv_golden[tag + "_codes"])
    assert np.array_equal(scale, kv_golden[tag + "_scale"])
    assert np.array_equal(zero, kv_golden[tag + "_zero"])
    assert np.array_equal(ko.dequantize_rows(codes, scale, zero), kv_golden[tag + "_deq"])


@pytest.mark.parametrize("kind,group", C1_CASES)
@pytest.mark.parametrize("bits", [4, 8])
def test_c_oracle_matches_reference_golden(kv_golden, c_oracle, kind, group, bits):
    kv = kv_golden["c1_kv"]
    view = ko.view_rows(kv, kind, group=group, head_dim=32)
    codes, scale, zero = c_quantize(c_oracle, view, bits)
    tag = f"c1_{kind}{group or ''}_b{bits}"
    assert np.array_equal(codes, kv_golden[tag + "_codes"])
    assert np.array_equal(scale, kv_golden[tag + "_scale"])
    assert np.array_equal(zero, kv_golden[tag + "_zero"])


def test_oracles_match_reference_float64_cases(kv_golden, c_oracle):
    for i in range(40):
        x = kv_golden[f"f64_{i}_x"]
        bits = int(kv_golden[f"f64_{i}_bits"])
        for codes, scale, zero in (ko.quantize_rows(x, bits), c_quantize(c_oracle, x, bits)):
            assert np.array_equal(codes, kv_golden[f"f64_{i}_codes"])
            assert np.array_equal(scale, kv_golden[f"f64_{i}_scale"])
            assert np.array_equal(zero, kv_golden[f"f64_{i}_zero"])


def test_layout_views_invert(kv_golden):
    kv = kv_golden["c1_kv"]
    for kind, group in C1_CASES:
        v = ko.view_rows(kv, kind, group=group, head_dim=32)
        back = ko.rows_to_native(v, kv.shape, kind, group=group, head_dim=32)
        assert np.array_equal(back, kv)


def test_c_vs_numpy_oracle_random_fp16(c_oracle):
    g = np.random.default_rng(11)
    for bits in (4, 8):
        x = (g.standard_normal((2000, 64)) * 10.0 ** g.uniform(-3, 3, size=(2000, 1))).astype(np.float16)
        x[::7] = np.abs(x[::7]) + np.float16(300)
        x[::13] = x[::13, :1]
        a = ko.quantize_rows(x, bits)
        b = c_quantize(c_oracle, x, bits)
        for u, v in zip(a, b):
            assert np.array_equal(u, v)


# ---- reference known answers (pkg/tests/test_kvmanager.py:52-126), restated -------
def test_unit_interval_known_answer():
    codes, scale, zero = ko.quantize_rows(np.array([[0.0, 1.0]]), 8)
    assert scale[0, 0] == 1.0 / 255.0 and zero[0, 0] == 0.0
    assert codes[0].tolist() == [0, 255]
    deq = ko.dequantize_rows(codes, scale, zero)
    assert deq[0, 1] == 1.0 and deq[0, 0] == 0.0


def test_errors():
    with pytest.raises(ValueError):
        ko.quantize_rows(np.ones((1, 4)), 5)
    with pytest.raises(ValueError):
        ko.quantize_rows(np.ones((1, 0)), 8)
    with pytest.raises(ValueError):
        ko.quantize_rows(np.array([[1.0, np.nan]]), 8)


def test_accounting_known_answers(kv_golden):
    from paper_2410_23537_b200 import kvmanager as km
    rows = kv_golden["acc"]
    i = 0
    for name in ("opt-2.7b", "opt-6.7b", "opt-13b"):
        m = km.MODEL_PRESETS[name]
        for t in (0, 1, 7, 128, 2048):
            for b in (4, 8):
                assert tuple(rows[i]) == (t, b, km.kv_bytes(m, t), km.quantized_kv_bytes(m, t, b))
                assert km.kv_bytes(m, t) == ko.kv_bytes(m.num_layers, m.hidden_size, t)
                assert km.quantized_kv_bytes(m, t, b) == ko.quantized_kv_bytes(m.num_layers, m.hidden_size, t, b)
                i += 1
    assert km.quantized_kv_bytes(km.MODEL_PRESETS["opt-13b"], 128, 8) == 52_428_800 + 3_276_800


# ----------------------------------------------------------------- absmax (restated)
def test_absmax_oracle_properties():
    """The symmetric absmax restatement (parity unpinned by the reference): zero point
    2^(b-1), scale = max|x| / (2^(b-1) - 1), codes symmetric about the zero point,
    round-trip error <= scale / 2, all-zero rows exact."""
    g = np.random.default_rng(9)
    for bits in (4, 8):
        x = g.standard_normal((50, 64)) * 10.0 ** g.uniform(-3, 3, size=(50, 1))
        x[3] = 0.0
        x[7] = np.abs(x[7])
        c, s, z = ko.quantize_rows_absmax(x, bits)
        qs = 2 ** (bits - 1) - 1
        assert (z == 2 ** (bits - 1)).all()
        a = np.abs(x).max(axis=1, keepdims=True)
        assert np.array_equal(s[a > 0], (a / qs)[a > 0]) and s[3, 0] == 1.0
        assert c.min() >= 2 ** (bits - 1) - qs and c.max() <= 2 ** (bits - 1) + qs
        y = ko.dequantize_rows(c, s, z)
        assert (np.abs(y - x) <= s / 2 * (1 + 1e-12)).all()
        assert (y[3] == 0).all()
        assert np.array_equal(ko.quantize_rows_absmax(-x, bits)[0].astype(int), 2 ** bits - c.astype(int))
