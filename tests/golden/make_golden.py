"""Generate golden vectors from the REFERENCE servesim package (run in the build
container, where /root/reference exists; the fixtures travel, the reference does not).

    python tests/golden/make_golden.py

Writes tests/golden/kv_golden.npz, kv_c1_full.npz and pred_golden.npz.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from harness import refsim  # noqa: E402

refsim.import_servesim()

from servesim import kvmanager as rk  # noqa: E402
from servesim import predictor as rp  # noqa: E402

from harness import synthetic  # noqa: E402
from oracle import kv_oracle  # noqa: E402


def kv_golden():
    out = {}
    # C1-shaped (scaled down): kv[2][2][64][128] fp16, head_dim 32
    L, T, Hd, D = 2, 64, 128, 32
    kv = synthetic.kv_job(L, T, Hd, seed=0, job=0, group=32)
    out["c1_kv"] = kv
    for kind, group in (("contig", 32), ("contig", 64), ("channel", 0), ("head", 0)):
        view = kv_oracle.view_rows(kv, kind, group=group, head_dim=D)
        for bits in (4, 8):
            qt = rk.quantize(view, bits)
            tag = f"c1_{kind}{group or ''}_b{bits}"
            out[tag + "_codes"] = qt.values
            out[tag + "_scale"] = qt.scale
            out[tag + "_zero"] = qt.zero
            out[tag + "_deq"] = rk.dequantize(qt)
    # float64 cases in the style of test_kvmanager.py:70-118 (mixed signs, single-sign,
    # magnitudes 1e-2..1e2, lengths 1..300)
    g = np.random.default_rng(2024)
    for i in range(40):
        bits = 4 if i % 2 else 8
        length = int(g.integers(1, 301))
        sc = 10.0 ** g.uniform(-2, 2)
        x = g.uniform(-sc, sc, size=(3, length))
        if i % 3 == 1:
            x = np.abs(x)
        elif i % 3 == 2:
            x = -np.abs(x) - 50.0
        qt = rk.quantize(x, bits)
        out[f"f64_{i}_x"] = x
        out[f"f64_{i}_bits"] = np.array(bits)
        out[f"f64_{i}_codes"] = qt.values
        out[f"f64_{i}_scale"] = qt.scale
        out[f"f64_{i}_zero"] = qt.zero
        out[f"f64_{i}_deq"] = rk.dequantize(qt)
    # accounting known answers
    ms = rk.MODEL_PRESETS
    acc = []
    for name in ("opt-2.7b", "opt-6.7b", "opt-13b"):
        for t in (0, 1, 7, 128, 2048):
            for b in (4, 8):
                acc.append((t, b, rk.kv_bytes(ms[name], t), rk.quantized_kv_bytes(ms[name], t, b)))
    out["acc"] = np.array(acc, dtype=np.int64)
    np.savez_compressed(os.path.join(HERE, "kv_golden.npz"), **out)
    print("kv_golden:", len(out), "arrays")


C1_FULL = dict(layers=4, tokens=512, heads=8, head_dim=128)
C1_FULL_LAYOUTS = (("head", 0), ("channel", 0), ("contig", 128))


def digest(a) -> str:
    import hashlib
    a = np.ascontiguousarray(a)
    return hashlib.sha256(a.dtype.str.encode() + str(a.shape).encode() + a.tobytes()).hexdigest()


def c1_full_kv():
    c = C1_FULL
    return synthetic.kv_job(c["layers"], c["tokens"], c["heads"] * c["head_dim"], seed=0, job=0, group=128)


def kv_c1_full():
    """BASELINE config 1 at its own shape: 4 layers x 8 heads x 128 dim x 512 tokens fp16,
    INT8 (and INT4) per-head (64 x 65536), per-channel (8192 x 512) and per-(token, head)
    (32768 x 128) views through the REFERENCE quantize/dequantize.  The outputs are kept
    as SHA-256 digests (bit-exact comparisons) plus the first rows in full."""
    kv = c1_full_kv()
    out = {"kv_digest": np.array(digest(kv))}
    for kind, group in C1_FULL_LAYOUTS:
        view = kv_oracle.view_rows(kv, kind, group=group, head_dim=C1_FULL["head_dim"])
        for bits in (4, 8):
            qt = rk.quantize(view, bits)
            deq = rk.dequantize(qt)
            tag = f"{kind}{group or ''}_b{bits}"
            out[tag + "_shape"] = np.array(view.shape)
            for name, arr in (("codes", qt.values), ("scale", qt.scale), ("zero", qt.zero), ("deq", deq),
                              ("deq16", deq.astype(np.float16))):
                out[f"{tag}_{name}_digest"] = np.array(digest(arr))
            out[tag + "_codes_head"] = qt.values[:2]
            out[tag + "_scale_head"] = qt.scale[:64]
            out[tag + "_zero_head"] = qt.zero[:64]
    np.savez_compressed(os.path.join(HERE, "kv_c1_full.npz"), **out)
    print("kv_c1_full:", len(out), "arrays")


def pred_golden():
    out = {}
    for tag, n, dim, nq, dups in (("d64", 3000, 64, 96, 20), ("d768", 1500, 768, 64, 10)):
        db, lens = synthetic.predictor_db(n, dim, seed=1, dup_groups=dups, dup_size=11)
        q = synthetic.predictor_queries(db, nq, seed=1)
        cfg = rp.PredictorConfig(dimension=dim, top_k=8, similarity_threshold=0.80,
                                 db_capacity=4096, max_len=2048)
        store = rp.VectorStore(dim, cfg.db_capacity)
        for v, ln in zip(db.astype(np.float64), lens):
            store.add(v, int(ln))
        reg = rp.FallbackRegressor(dim, 32, seed=0)
        reg.b2 = 5.0
        pred = rp.LengthPredictor(cfg, regressor=reg, store=store)
        sims, slens, seqs, plen, prov, mlp = [], [], [], [], [], []
        for v in q.astype(np.float64):
            s, l_, sq = store.search(v, 8)
            sims.append(s); slens.append(l_); seqs.append(sq)
            a, b = pred.predict_vector(v)
            plen.append(a); prov.append(b == rp.RETRIEVED)
            mlp.append(reg.predict_len(v, cfg.max_len))
        out[f"{tag}_db"] = db
        out[f"{tag}_lens"] = lens
        out[f"{tag}_q"] = q
        out[f"{tag}_sims"] = np.array(sims)
        out[f"{tag}_slens"] = np.array(slens)
        out[f"{tag}_seqs"] = np.array(seqs)
        out[f"{tag}_pred"] = np.array(plen)
        out[f"{tag}_retrieved"] = np.array(prov)
        out[f"{tag}_mlp"] = np.array(mlp)
        out[f"{tag}_W1"] = reg.w1
        out[f"{tag}_b1"] = reg.b1
        out[f"{tag}_w2"] = reg.w2
        out[f"{tag}_b2"] = np.array(reg.b2)
    # a trained regressor (train_fallback on hashed pseudo-prompts)
    from servesim import workload as rw
    corpus = []
    g = np.random.default_rng(5)
    for i in range(200):
        n_out = int(np.clip(np.rint(g.lognormal(5.0, 1.2)), 1, 2048))
        corpus.append((rw.make_prompt_tokens(0, i, n_out), n_out))
    cfg = rp.PredictorConfig(dimension=64, fallback_epochs=60)
    reg = rp.train_fallback(corpus, cfg, seed=0)
    emb = rp.HashingEmbedder(64)
    X = np.stack([emb.embed(t) for t, _ in corpus])
    out["trained_X"] = X
    out["trained_W1"] = reg.w1
    out["trained_b1"] = reg.b1
    out["trained_w2"] = reg.w2
    out["trained_b2"] = np.array(reg.b2)
    out["trained_len"] = np.array([reg.predict_len(x, 2048) for x in X])
    out["trained_loss"] = np.array(reg.loss_history)
    out["corpus_lens"] = np.array([n for _, n in corpus])
    np.savez_compressed(os.path.join(HERE, "pred_golden.npz"), **out)
    print("pred_golden:", len(out), "arrays")


if __name__ == "__main__":
    which = sys.argv[1:] or ["kv", "c1full", "pred"]
    if "kv" in which:
        kv_golden()
    if "c1full" in which:
        kv_c1_full()
    if "pred" in which:
        pred_golden()
