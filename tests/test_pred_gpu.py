"""GPU parity for the predictor: exact top-k (indices and float64 sims bit-exact with
the restated oracle, ties by insert order), predicted lengths exact, plus the
reference's known-answer tests (pkg/tests/test_predictor.py) through the GPU path."""
import numpy as np
import pytest

from oracle import pred_oracle as po
from tests.conftest import have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def pr():
    from paper_2410_23537_b200 import predictor
    return predictor


def unit(*values, dim=8):
    v = np.zeros(dim)
    v[:len(values)] = values
    return v / np.linalg.norm(v)


def check_batch(pr, db, lens, Q, k, capacity=None, dtype=np.float32):
    import torch
    n, d = db.shape
    store = pr.VectorStore(d, capacity or max(n, 8), dtype=dtype)
    store.add_batch(db, lens)
    sims, seqs, slens, cnt, _ = store.search_batch(Q, k)
    torch.cuda.synchronize()
    ref = po.search_exact_batch(db, lens, np.arange(n), Q, k, f64=np.dtype(dtype) == np.float64)
    sims, seqs, slens, cnt = (t.cpu().numpy() for t in (sims, seqs, slens, cnt))
    for i, (es, el, eq) in enumerate(ref):
        c = cnt[i]
        assert c == len(eq), (i, c, len(eq))
        assert np.array_equal(seqs[i, :c], eq), (i, seqs[i, :c], eq)
        assert np.array_equal(sims[i, :c], es), (i, sims[i, :c] - es)
        assert np.array_equal(slens[i, :c], el)
    # candidates the double-double certificate could not decide were recomputed exactly
    assert store.inexact_count() >= 0
    return store


@pytest.mark.parametrize("tag", ["d64", "d768"])
def test_search_matches_oracle_and_reference(pr, pred_golden, tag):
    g = pred_golden
    db, lens, Q = g[f"{tag}_db"], g[f"{tag}_lens"], g[f"{tag}_q"]
    check_batch(pr, db, lens, Q, 8, capacity=4096)


@pytest.mark.parametrize("tag", ["d64", "d768"])
def test_predict_batch_exact(pr, pred_golden, tag):
    g = pred_golden
    db, lens, Q = g[f"{tag}_db"], g[f"{tag}_lens"], g[f"{tag}_q"]
    reg = pr.FallbackRegressor(db.shape[1], 32, seed=0)
    reg.b2 = float(g[f"{tag}_b2"])
    store = pr.VectorStore(db.shape[1], 4096)
    store.add_batch(db, lens)
    p = pr.LengthPredictor(pr.PredictorConfig(dimension=db.shape[1], db_capacity=4096), regressor=reg,
                           store=store)
    out, ret = p.predict_batch(Q)
    ref_len, ref_ret = po.predict_batch(db, lens, np.arange(len(db)), Q, reg.w1, reg.b1, reg.w2, reg.b2)
    assert np.array_equal(out.cpu().numpy(), ref_len)
    assert np.array_equal(ret.cpu().numpy().astype(bool), ref_ret)
    mlp = reg.predict_len_batch(Q, 2048).cpu().numpy()
    assert np.array_equal(mlp, g[f"{tag}_mlp"])


@pytest.mark.parametrize("n,d,B,k", [(1, 8, 3, 8), (7, 8, 5, 8), (300, 100, 130, 5), (2000, 64, 257, 1),
                                     (5000, 768, 64, 16), (20000, 128, 300, 8)])
def test_shapes_and_k(pr, n, d, B, k):
    g = np.random.default_rng(n + d + B + k)
    db = g.standard_normal((n, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = g.standard_normal((B, d)).astype(np.float32)
    Q[: B // 2] = db[g.integers(0, n, size=B // 2)] + 0.02 * g.standard_normal((B // 2, d)).astype(np.float32)
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    check_batch(pr, db, lens, Q.astype(np.float32), k)


def test_ties_broken_by_insert_order(pr):
    g = np.random.default_rng(9)
    d = 64
    db = g.standard_normal((3000, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    for grp in range(20):  # groups of 11 identical rows competing for 8 slots
        base = grp * 37
        idx = g.choice(np.arange(1000, 3000), size=10, replace=False)
        db[idx] = db[base]
    lens = g.integers(1, 2048, size=3000).astype(np.int32)
    Q = db[[grp * 37 for grp in range(20)]] + 0.001 * g.standard_normal((20, d)).astype(np.float32)
    Q = (Q / np.linalg.norm(Q, axis=1, keepdims=True)).astype(np.float32)
    check_batch(pr, db, lens, Q, 8)


def test_heavy_ties_take_the_exhaustive_path(pr):
    # 600 identical rows: more candidates than a scan CTA can hold -> exact fallback
    d = 32
    v = np.ones((600, d), np.float32) / np.sqrt(d)
    g = np.random.default_rng(2)
    other = g.standard_normal((400, d)).astype(np.float32)
    db = np.concatenate([other[:200], v, other[200:]])
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    lens = np.arange(1, 1001).astype(np.int32)
    Q = db[[250, 0, 999]].astype(np.float32)
    check_batch(pr, db, lens, Q, 8)


def test_fifo_ring_semantics(pr):
    import torch
    d = 16
    store = pr.VectorStore(d, 100)
    g = np.random.default_rng(4)
    rows = g.standard_normal((250, d)).astype(np.float32)
    rows /= np.linalg.norm(rows, axis=1, keepdims=True)
    lens = np.arange(1, 251)
    for c in range(0, 250, 60):
        store.add_batch(rows[c:c + 60], lens[c:c + 60])
    assert len(store) == 100 and store.next_seq == 250
    live = rows[150:]
    Q = rows[[160, 249, 10]]
    sims, seqs, slens, cnt, _ = store.search_batch(Q, 8)
    torch.cuda.synchronize()
    ref = po.search_exact_batch(live, lens[150:], np.arange(150, 250), Q, 8)
    for i, (es, el, eq) in enumerate(ref):
        assert np.array_equal(seqs[i].cpu().numpy(), eq)
        assert np.array_equal(sims[i].cpu().numpy(), es)


# ---- reference known answers (pkg/tests/test_predictor.py), through the GPU ---------
def test_reference_vectorstore_known_answers(pr, tmp_path):
    store = pr.VectorStore(dimension=8, capacity=3)
    for i in range(3):
        store.add(unit(1, i + 1), observed_len=10 * (i + 1))
    store.add(unit(5, 5), observed_len=99)
    assert len(store) == 3
    sims, lens, seqs = store.search(unit(1, 1), k=3)
    assert 10 not in lens and seqs.min() == 1
    store = pr.VectorStore(dimension=4, capacity=10)
    seqs = [store.add(unit(1, i, dim=4), 5) for i in range(6)]
    assert seqs == sorted(seqs) and len(set(seqs)) == 6
    store = pr.VectorStore(dimension=8, capacity=10)
    store.add(unit(1, 0), 10)
    store.add(unit(1, 1), 20)
    store.add(unit(0, 1), 30)
    sims, lens, _ = store.search(unit(1, 0), k=3)
    assert list(lens) == [10, 20, 30] and sims[0] == pytest.approx(1.0)
    store = pr.VectorStore(dimension=4, capacity=10)
    for i in range(5):
        store.add(unit(1, i, dim=4), 7 + i)
    store.save(tmp_path / "db.jsonl")
    loaded = pr.VectorStore.load(tmp_path / "db.jsonl", dimension=4, capacity=10)
    q = unit(1, 2, dim=4)
    assert np.allclose(store.search(q, 3)[0], loaded.search(q, 3)[0])


def test_reference_prediction_known_answers(pr):
    def cfg(**kw):
        base = dict(dimension=8, top_k=3, similarity_threshold=0.8, db_capacity=100, max_len=2048)
        base.update(kw)
        return pr.PredictorConfig(**base)
    p = pr.LengthPredictor(cfg())
    p.store.add(unit(1, 2, 3), 100)
    assert p.predict_vector(unit(1, 2, 3)) == (100, pr.RETRIEVED)
    p = pr.LengthPredictor(cfg())
    _, prov = p.predict_vector(unit(1, 0))
    assert prov == pr.FALLBACK
    p = pr.LengthPredictor(cfg())
    a = unit(1, 0.5)
    b = unit(0.5, 1)
    p.store.add(a, 100)
    p.store.add(b, 200)
    q = unit(1, 1)
    sa, sb = float(q @ a), float(q @ b)
    assert sa == pytest.approx(sb)
    length, prov = p.predict_vector(q)
    assert prov == pr.RETRIEVED and length == 150
    p = pr.LengthPredictor(cfg(max_len=64))
    p.store.add(unit(1, 1), 5000)
    assert p.predict_vector(unit(1, 1)) == (64, pr.RETRIEVED)
    p = pr.LengthPredictor(cfg(online_refit=False))
    p.observe(unit(3, 1, 4), 123)
    assert p.predict_vector(unit(3, 1, 4)) == (123, pr.RETRIEVED)


@pytest.mark.slow
def test_c4_scale_200k_x_768(pr):
    """C4 shape at 1/5 scale (200k x 768 DB, 512 queries, planted duplicates)."""
    from harness import synthetic
    db, lens = synthetic.predictor_db(200_000, 768, seed=0, dup_groups=200)
    Q = synthetic.predictor_queries(db, 512, seed=0)
    check_batch(pr, db, lens, Q, 8)


def _adversarial_norm_db(d=64, k=4):
    """Shard 1 (odd seqs) holds k rows whose fp16 coarse scores overshoot their exact
    scores by ~0.24 (components 100.032 / -100.03 round away from the exact cancellation)
    and a huge-norm row that makes its coarse error bound large; shard 0 (even seqs)
    holds k fp16-exact rows with exact score 0.1 > the overshooting rows' 0.008, so the
    global top-k lies in shard 0 even though shard 1's coarse k-th bound (~0.25) is far
    above their coarse scores (the exchanged bound must be an exact-score
    bound, L - delta_self, not a coarse one)."""
    q = np.full(d, 1.0 / np.sqrt(d))
    rows, n = [], 4 * k + 8
    for i in range(n):
        r = np.zeros(d)
        if i % 2 == 1 and i < 2 * k + 1:
            r[0::2], r[1::2] = 100.032, -100.03       # exact 0.008, coarse ~0.25
        elif i % 2 == 0 and i < 2 * k:
            r[0] = 0.1 * np.sqrt(d)                   # exact 0.1 (fp16-exact)
        elif i == 2 * k + 3:
            r[0::2], r[1::2] = 3000.0, -3000.0        # huge norm, exact score 0
        else:
            r[0] = -0.5 * np.sqrt(d)                  # filler, exact -0.5
        rows.append(r)
    return np.array(rows), q


def _sharded_worker(rank, world, port, result_dir, backend="gloo", layout="rows"):
    import os

    import torch
    import torch.distributed as dist

    from paper_2410_23537_b200 import predictor as pr
    from paper_2410_23537_b200 import sharding
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":     # one GPU per rank, NCCL over NVLink
        torch.cuda.set_device(rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", rank))
    else:                     # both ranks share the one GPU; gloo carries the exchange
        torch.cuda.set_device(0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    fails = []

    def same(tag, sims, seqs, slens, cnt, ref):
        for i, r in enumerate(ref):
            c = int(cnt[i])
            if not (c == len(r[2]) and np.array_equal(seqs[i, :c].cpu().numpy(), r[2])
                    and np.array_equal(sims[i, :c].cpu().numpy(), r[0])
                    and np.array_equal(slens[i, :c].cpu().numpy(), r[1])):
                fails.append((tag, i))
                return

    # (a) fp32 DB with a tie group spanning both shards and ring eviction
    g = np.random.default_rng(21)
    n, d, B, k = 6000, 96, 200, 8
    db = g.standard_normal((n, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    db[3000:3011] = db[7]
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.concatenate([db[[7, 100, 4000]], g.standard_normal((B - 3, d)).astype(np.float32)])
    Q = (Q / np.linalg.norm(Q, axis=1, keepdims=True)).astype(np.float32)
    cap = 5000                                  # ring eviction: the oldest 1000 rows drop out
    store = sharding.ShardedVectorStore(d, cap, dtype=np.float32, layout=layout)
    store.add_batch(db[:2500], lens[:2500])
    store.add_batch(db[2500:], lens[2500:])
    live = np.arange(n - cap, n)
    same("fp32", *store.search_batch(Q, k)[:4], po.search_exact_batch(db[live], lens[live], live, Q, k))
    # top_k > 16: each shard's exact big-k search, gathered and merged
    same("k40", *store.search_batch(Q[:20], 40)[:4], po.search_exact_batch(db[live], lens[live], live, Q[:20], 40))
    # empty query batch (the rescore of an empty scan)
    out = store.search_batch(np.zeros((0, d), np.float32), k)
    if out[0].shape != (0, k):
        fails.append(("empty", out[0].shape))

    # (b) shards with different max row norms
    rows, q = _adversarial_norm_db()
    adv = sharding.ShardedVectorStore(rows.shape[1], 64, layout=layout)
    adv.add_batch(rows, np.arange(1, len(rows) + 1))
    idx = np.arange(len(rows))
    same("norms", *adv.search_batch(q[None, :], 4)[:4],
         po.search_exact_batch(rows, np.arange(1, len(rows) + 1), idx, q[None, :], 4, f64=True))

    # (c) drop-in API on a float64 sharded store: LengthPredictor(store=sharded)
    g = np.random.default_rng(5)
    n, d = 1200, 64
    dbf = g.standard_normal((n, d))
    dbf /= np.linalg.norm(dbf, axis=1, keepdims=True)
    lf = g.integers(1, 2048, size=n)
    cfg = pr.PredictorConfig(dimension=d, db_capacity=1000, refit_sample_cap=64)
    sh = sharding.ShardedVectorStore(d, cfg.db_capacity, layout=layout)
    ref_store = pr.VectorStore(d, cfg.db_capacity)             # single-store reference run
    p_sh = pr.LengthPredictor(cfg, store=sh)
    p_one = pr.LengthPredictor(pr.PredictorConfig(dimension=d, db_capacity=1000, refit_sample_cap=64),
                               store=ref_store)
    for i in range(n):                                          # observe: owner-rank append + refits
        p_sh.observe(dbf[i], int(lf[i]))
        p_one.observe(dbf[i], int(lf[i]))
    Qf = np.concatenate([dbf[-50:] + 0.01 * g.standard_normal((50, d)), g.standard_normal((50, d))])
    Qf /= np.linalg.norm(Qf, axis=1, keepdims=True)
    a, ra = p_sh.predict_batch(Qf)
    b, rb = p_one.predict_batch(Qf)
    if not (torch.equal(a.cpu(), b.cpu()) and torch.equal(ra.cpu(), rb.cpu())):
        fails.append(("predict", int((a.cpu() != b.cpu()).sum())))
    if not np.array_equal(p_sh.regressor.w1, p_one.regressor.w1):
        fails.append(("refit",))
    live = np.arange(n - cfg.db_capacity, n)
    same("f64", *sh.search_batch(Qf, 8)[:4], po.search_exact_batch(dbf[live], lf[live], live, Qf, 8, f64=True))
    s1 = sh.search(Qf[0], 5)
    s2 = ref_store.search(Qf[0], 5)
    if not all(np.array_equal(x, y) for x, y in zip(s1, s2)):
        fails.append(("search",))
    X1, L1 = sh.newest(100)
    X2, L2 = ref_store.newest(100)
    if not (np.array_equal(X1, X2) and np.array_equal(L1, L2)):
        fails.append(("newest",))
    # per-shard binary snapshot restores the global FIFO (same seqs, same evictions)
    path = os.path.join(result_dir, "snap")
    sh.save_binary(path)
    dist.barrier()
    back = sharding.ShardedVectorStore.load_binary(path)
    extra = g.standard_normal((30, d))
    for st in (sh, back):
        st.add_batch(extra, np.arange(1, 31))
    x1 = sh.search_batch(Qf, 8)
    x2 = back.search_batch(Qf, 8)
    if not all(torch.equal(u, v) for u, v in zip(x1[:4], x2[:4])) or back.next_seq != sh.next_seq:
        fails.append(("snapshot",))
    if layout == "queries":  # the collective-free slice equals the gathered rows
        lo, hi, loc = sh.search_batch_local(Qf, 8)
        if not all(torch.equal(u, v[lo:hi]) for u, v in zip(loc[:4], x1[:4])):
            fails.append(("local slice",))
    with open(os.path.join(result_dir, f"r{rank}"), "w") as fh:
        fh.write("ok" if not fails else repr(fails))
    dist.destroy_process_group()


def test_sharded_store_two_ranks_one_gpu(tmp_path):
    """ShardedVectorStore end to end (seq % 2 shards, per-shard GPU top-k, bound
    all-reduce, all-gather, GPU merge, FIFO eviction across shards) against the
    single-store oracle; shards with different row norms; the drop-in API
    (LengthPredictor(store=ShardedVectorStore): observe + refit, predict_batch, search,
    newest, per-shard binary snapshots)."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_sharded_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert (tmp_path / f"r{r}").read_text() == "ok"


def test_sharded_store_nccl_two_gpus(tmp_path):
    """The same end-to-end checks over NCCL with one GPU per rank (runs wherever two or
    more GPUs are visible, e.g. the 8-GPU scaling box)."""
    import socket

    import torch
    import torch.multiprocessing as mp
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs")
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_sharded_worker, args=(2, port, str(tmp_path), "nccl"), nprocs=2, join=True)
    for r in range(2):
        assert (tmp_path / f"r{r}").read_text() == "ok"


def test_sharded_store_queries_layout_two_ranks_one_gpu(tmp_path):
    """layout="queries" (replicated DB, each rank searches a slice of the batch): the
    same end-to-end checks, plus the collective-free local slice."""
    import socket

    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_sharded_worker, args=(2, port, str(tmp_path), "gloo", "queries"), nprocs=2, join=True)
    for r in range(2):
        assert (tmp_path / f"r{r}").read_text() == "ok"


def test_adversarial_norms_single_store(pr):
    rows, q = _adversarial_norm_db()
    check_batch(pr, rows, np.arange(1, len(rows) + 1), q[None, :], 4, dtype=np.float64)


def test_gpu_embedder_bit_identical_to_reference_hashing(pr):
    import torch
    g = np.random.default_rng(8)
    prompts = [g.integers(-5, 70000, size=int(g.integers(1, 300))).tolist() for _ in range(200)]
    prompts += [[5], [9, 9, 9], list(range(50)), [-1, 0, 1]]
    for dim in (64, 768):
        emb = pr.HashingEmbedder(dim)
        out = emb.embed_batch(prompts).cpu().numpy()
        ref = np.stack([emb.embed(p) for p in prompts])
        assert np.array_equal(out, ref)
        o32 = emb.embed_batch(prompts, dtype=torch.float32).cpu().numpy()
        assert np.array_equal(o32, ref.astype(np.float32))
    with pytest.raises(pr.PredictorError):
        pr.HashingEmbedder(8).embed_batch([[1, 2], []])


def test_binary_snapshot_round_trip(pr, tmp_path):
    import torch
    g = np.random.default_rng(12)
    d = 48
    store = pr.VectorStore(d, 500)
    rows = g.standard_normal((700, d)).astype(np.float32)
    store.add_batch(rows, np.arange(1, 701))
    store.save_binary(tmp_path / "db.npz")
    loaded = pr.VectorStore.load_binary(tmp_path / "db.npz")
    Q = rows[[650, 699, 100]]
    a = store.search_batch(Q, 8)
    b = loaded.search_batch(Q, 8)
    torch.cuda.synchronize()
    assert torch.equal(a[0], b[0]) and torch.equal(a[2], b[2])
    assert torch.equal(a[1] - 200, b[1])  # re-added from seq 0 in the same order


@pytest.mark.parametrize("B", [1, 256, 700, 1100, 2000])
def test_shared_thresholds_with_ties_across_tile_groups(pr, B):
    """The scan's tile groups share their running k-th (atomic max per query) and keep
    only values above it in their top lists; exact ties of the k-th spread over many
    groups (copies of one row every ~2k rows) and near-ties must still give the exact
    (-sim, seq) top-k."""
    g = np.random.default_rng(B)
    n, d = 120_000, 256
    db = g.standard_normal((n, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    target = db[5].copy()
    db[np.arange(1000, n, 2048)] = target              # ~58 exact copies in different groups
    near = np.arange(1500, n, 4096)
    db[near] = target + 1e-3 * g.standard_normal((near.size, d)).astype(np.float32)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.repeat(target[None, :], B, axis=0)
    Q[B // 2:] = g.standard_normal((B - B // 2, d)).astype(np.float32)
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    check_batch(pr, db, lens, Q.astype(np.float32), 8)


def test_graphed_single_request_matches_eager(pr):
    """predict_vector through the captured CUDA graph == the eager path, including after
    the DB grows (re-capture) and for fallback (MLP) queries."""
    from harness import synthetic
    db, lens = synthetic.predictor_db(30_000, 256, seed=3, dup_groups=30)
    reg = pr.FallbackRegressor(256, 32, seed=0)
    reg.b2 = 5.0
    store = pr.VectorStore(256, 40_000)
    store.add_batch(db[:20_000], lens[:20_000])
    p = pr.LengthPredictor(pr.PredictorConfig(dimension=256, db_capacity=40_000), regressor=reg, store=store)
    Q = synthetic.predictor_queries(db, 24, seed=4).astype(np.float64)
    eager = [p.predict_vector(q) for q in Q]
    p.enable_graphs()
    assert [p.predict_vector(q) for q in Q] == eager
    store.add_batch(db[20_000:], lens[20_000:])    # size change -> re-capture
    p.enable_graphs(False)
    eager2 = [p.predict_vector(q) for q in Q]
    p.enable_graphs()
    assert [p.predict_vector(q) for q in Q] == eager2
    assert any(r == pr.FALLBACK for _, r in eager2) and any(r == pr.RETRIEVED for _, r in eager2)


@pytest.mark.parametrize("B,k,negative", [(1, 3, False), (1, 16, False), (300, 16, False), (1, 8, True),
                                          (300, 5, True)])
def test_scan_bounds_many_groups(pr, B, k, negative):
    """Warm-start bound, shared k-th and rank slots across many tile groups (B = 1 runs
    148 groups of the 1-SM scan, B = 300 two CTA-pair blocks of 2-SM groups), for k
    not dividing the slot count and for all-negative similarities (order-preserving keys
    of negative scores, warm start from negative chunk maxima)."""
    g = np.random.default_rng(1000 * B + k)
    n, d = 150_000, 64
    db = g.standard_normal((n, d)).astype(np.float32)
    if negative:  # every row in the positive orthant, every query in the negative one
        db = np.abs(db)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = g.standard_normal((B, d)).astype(np.float32)
    if negative:
        Q = -np.abs(Q)
    else:
        Q[: B // 2] = db[g.integers(0, n, size=B // 2)] + 0.05 * g.standard_normal((B // 2, d)).astype(np.float32)
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    check_batch(pr, db, lens, Q.astype(np.float32), k)


def test_midpoint_ties_take_the_superaccumulator(pr):
    """Exact dot products at a float64 rounding midpoint (1 + 2^-53: the double-double
    certificate cannot decide) are resolved by the 640-bit superaccumulator and must
    round to even exactly like the oracle's fsum."""
    g = np.random.default_rng(77)
    n, d = 3000, 64
    db = (g.standard_normal((n, d)) / 16).astype(np.float32)
    crafted = np.arange(100, 3000, 300)
    for j, r in enumerate(crafted):
        db[r] = 0.0
        db[r, 0] = 1.0
        db[r, 1] = 1.0 + j  # dot = 1 + (1 + j) * 2^-53: midpoints for even (1 + j)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.zeros((3, d), np.float32)
    Q[:, 0] = 1.0
    Q[:, 1] = np.float32(2.0 ** -53)
    Q[1, 2] = np.float32(2.0 ** -30)
    Q[2] = -Q[2]
    store = check_batch(pr, db, lens, Q, 8)
    assert store.inexact_count() > 0


def test_more_query_blocks_than_units(pr):
    """B = 19200 on the 2-SM scan: 75 query blocks of 256 for 74 CTA pairs, so every
    block has one tile group and the last one is scanned in chunks by all units."""
    g = np.random.default_rng(5)
    n, d, B = 3000, 32, 19200
    db = g.standard_normal((n, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = g.standard_normal((B, d)).astype(np.float32)
    Q[::3] = db[g.integers(0, n, size=Q[::3].shape[0])] + 0.05 * g.standard_normal((Q[::3].shape[0], d)).astype(np.float32)
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    check_batch(pr, db, lens, Q.astype(np.float32), 8)


def test_split_search_api(pr):
    """alise_db_topk_scan + alise_db_topk_rescore (the sharded path's two steps): with its
    own bound the result equals alise_db_topk; with a higher external bound it is a
    prefix of it (only rows that can still enter the global top-k); an empty shard gives
    -inf bounds and no records."""
    import torch

    from paper_2410_23537_b200 import _lib
    g = np.random.default_rng(12)
    n, d, B, k = 20000, 96, 300, 8
    db = g.standard_normal((n, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = g.standard_normal((B, d)).astype(np.float32)
    Q[: B // 2] = db[g.integers(0, n, size=B // 2)] + 0.05 * g.standard_normal((B // 2, d)).astype(np.float32)
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    store = pr.VectorStore(d, n, dtype=np.float32)  # raw C calls: queries in the master dtype
    store.add_batch(db, lens)
    q = torch.from_numpy(Q).cuda()
    ref = store.search_batch(q, k)

    def split(st, ext_fn):
        outs = [torch.empty((B, k), dtype=torch.float64, device="cuda"),
                torch.empty((B, k), dtype=torch.int64, device="cuda"),
                torch.empty((B, k), dtype=torch.int32, device="cuda"), torch.empty(B, dtype=torch.int32, device="cuda")]
        bound = torch.empty(B, dtype=torch.float32, device="cuda")
        _lib.call("alise_db_topk_scan", st._h, _lib.ptr(q), B, k, _lib.ptr(bound), _lib.stream_ptr())
        ext = ext_fn(bound)
        _lib.call("alise_db_topk_rescore", st._h, _lib.ptr(q), B, k, _lib.ptr(ext), *[_lib.ptr(t) for t in outs],
                  _lib.stream_ptr())
        torch.cuda.synchronize()
        return bound, outs

    bound, outs = split(store, lambda b: b)
    assert torch.equal(outs[3], ref[3])
    for a, r in zip(outs[:3], ref[:3]):
        assert torch.equal(a, r)
    assert torch.isfinite(bound).all()
    # a higher external bound keeps a prefix of the exact top-k
    _, outs2 = split(store, lambda b: b + 0.02)
    c2, c1 = outs2[3].cpu().numpy(), ref[3].cpu().numpy()
    assert (c2 <= c1).all() and (c2 < c1).any()
    for i in range(B):
        assert torch.equal(outs2[1][i, :c2[i]], ref[1][i, :c2[i]])
    # empty shard
    empty = pr.VectorStore(d, 64, dtype=np.float32)
    b0, outs0 = split(empty, lambda b: b)
    assert torch.isinf(b0).all() and (b0 < 0).all()
    assert (outs0[3] == 0).all()


# ----------------------------------------------------------------- float64 master store
def _f64_db(g, n, d, ties=True):
    db = g.standard_normal((n, d))
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    if ties:
        db[n // 2:n // 2 + 11] = db[3]               # exact duplicates: ties broken by seq
    return db


@pytest.mark.parametrize("k", [1, 8, 16])
def test_f64_store_exact_vs_oracle(pr, k):
    """float64 vectors (not fp32-representable) in the default float64 store: sims are
    the correctly rounded dot products of the float64 values (two_prod-split products),
    top-k by (-sim, seq), equal to the restated oracle bit for bit."""
    g = np.random.default_rng(40 + k)
    n, d, B = 5000, 96, 300
    db = _f64_db(g, n, d)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.concatenate([db[[3, 10, 4000]] + 1e-3 * g.standard_normal((3, d)), g.standard_normal((B - 3, d))])
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    check_batch(pr, db, lens, Q, k, dtype=np.float64)


def test_f64_predict_batch_uses_float64_queries(pr):
    """predict_batch on a float64 store: retrieval over float64 sims, the fallback MLP on
    the float64 query (the reference's own vector), equal to the oracle."""
    g = np.random.default_rng(5)
    n, d = 3000, 64
    db = _f64_db(g, n, d)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.concatenate([db[:40] + 0.02 * g.standard_normal((40, d)), g.standard_normal((60, d))])
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    reg = pr.FallbackRegressor(d, 32, seed=1)
    reg.b2 = 4.0
    store = pr.VectorStore(d, 4096)
    store.add_batch(db, lens)
    p = pr.LengthPredictor(pr.PredictorConfig(dimension=d, db_capacity=4096), regressor=reg, store=store)
    out, ret = p.predict_batch(Q)
    ref_len, ref_ret = po.predict_batch(db, lens, np.arange(n), Q, reg.w1, reg.b1, reg.w2, reg.b2, f64=True)
    assert np.array_equal(out.cpu().numpy(), ref_len)
    assert np.array_equal(ret.cpu().numpy().astype(bool), ref_ret)
    assert 0 < ref_ret.sum() < len(Q)
    # and per request through predict_vector (eager and CUDA-graph replay)
    for i in (0, 5, 70):
        assert p.predict_vector(Q[i])[0] == ref_len[i]
    p.enable_graphs()
    for i in (0, 5, 70):
        assert p.predict_vector(Q[i])[0] == ref_len[i]


def test_hashing_embedder_vectors_exact(pr):
    """The reference's own HashingEmbedder vectors (float64, many shared n-grams):
    search results equal the oracle on float64 rows."""
    g = np.random.default_rng(9)
    emb = pr.HashingEmbedder(64)
    base = [list(range(1000 + b, 1018 + b)) for b in range(30)]
    prompts = [base[int(g.integers(0, 30))] + g.integers(50_000, 51_000, size=2).tolist() for _ in range(2000)]
    db = np.stack([emb.embed(p) for p in prompts])
    lens = g.integers(1, 2048, size=len(db)).astype(np.int32)
    Q = np.stack([emb.embed(base[i % 30] + [50_001, 50_002]) for i in range(120)])
    check_batch(pr, db, lens, Q, 8, dtype=np.float64)


def test_f64_midpoint_sums_use_exact_accumulator(pr):
    """Dot products whose exact value is a float64 rounding midpoint (or within 2^-100 of
    one) defeat the double-double certificate; the 4480-bit accumulator must round
    them correctly (half-even)."""
    import torch
    from fractions import Fraction
    d = 64
    rows = np.zeros((6, d))
    rows[0, :2] = [1.0, 2.0 ** -53]                      # 1 + 2^-53: tie -> even (1.0)
    rows[1, :3] = [1.0, 2.0 ** -53, 2.0 ** -100]         # just above the tie -> 1 + 2^-52
    rows[2, :3] = [1.0, 3 * 2.0 ** -53, -(2.0 ** -120)]  # just below 1 + 3*2^-53 -> 1 + 2^-52
    rows[3, :2] = [0.75, 2.0 ** -54]                     # 0.75 + 2^-54: tie -> even
    rows[4, :4] = [0.5, 0.25, 2.0 ** -60, -(2.0 ** -60)]  # exact cancellation
    rows[5, :2] = [1e-3, 1e-3]
    q = np.zeros(d)
    q[:4] = 1.0
    store = pr.VectorStore(d, 8)
    store.add_batch(rows, np.arange(1, 7))
    sims, seqs, _l, cnt, _ = store.search_batch(q[None, :], 6)
    torch.cuda.synchronize()
    got = dict(zip(seqs[0].cpu().numpy().tolist(), sims[0].cpu().numpy().tolist()))
    for r in range(6):
        exact = float(sum((Fraction(a) * Fraction(b) for a, b in zip(rows[r].tolist(), q.tolist())), Fraction(0)))
        assert got[r] == exact, (r, got[r], exact)
    assert got[0] == 1.0 and got[1] == 1.0 + 2.0 ** -52 and got[2] == 1.0 + 2.0 ** -52
    assert store.inexact_count() >= 3


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_rows_beyond_fp16_range_take_the_exact_path(pr, dtype):
    """A component beyond 65504 overflows the fp16 coarse copy: the store routes every
    query through the exhaustive exact path instead of trusting inf/NaN coarse scores."""
    g = np.random.default_rng(77)
    n, d = 3000, 64
    db = g.standard_normal((n, d))
    db[17, 5] = 1.0e5
    db[900, :] *= 3.0e4
    db = db.astype(dtype)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = g.standard_normal((50, d)).astype(dtype)
    Q[3, 5] = 7.0e4
    check_batch(pr, db, lens, Q, 8, dtype=dtype)


def test_mlp_hidden_beyond_128(pr):
    """fallback_hidden > 128: the finish kernel walks the hidden units in chunks of 128
    with the output sum still in index order."""
    g = np.random.default_rng(3)
    d, H = 96, 300
    reg = pr.FallbackRegressor(d, H, seed=2)
    reg.b1 = g.standard_normal(H) * 0.1
    reg.b2 = 3.0
    X = g.standard_normal((70, d))
    got = reg.predict_len_batch(X, 2048).cpu().numpy()
    ref = po.mlp_predict_len(X, reg.w1, reg.b1, reg.w2, reg.b2, 2048)
    assert np.array_equal(got, ref)


# ----------------------------------------------------------------- reference BLAS order
def _check_blas(pr, rows, lens, Q, k, cap, threads=8):
    import torch
    n, d = rows.shape
    store = pr.VectorStore(d, cap, order="blas", blas_threads=threads)
    store.add_batch(rows, lens)
    sims, seqs, slens, cnt, _ = store.search_batch(Q, k)
    torch.cuda.synchronize()
    # the reference's array: ring slots in slot order (predictor.py:126-152)
    live = np.arange(max(0, n - cap), n)
    slot_rows = np.zeros((min(n, cap), d))
    slot_lens = np.zeros(min(n, cap), np.int64)
    slot_seqs = np.zeros(min(n, cap), np.int64)
    slot_rows[live % cap], slot_lens[live % cap], slot_seqs[live % cap] = rows[live], lens[live], live
    bad = []
    for i, q in enumerate(Q):
        allsims = po.blas_gemv(slot_rows, q, threads)
        o = np.lexsort((slot_seqs, -allsims))[:k]
        c = int(cnt[i])
        if not (c == len(o) and np.array_equal(seqs[i, :c].cpu().numpy(), slot_seqs[o])
                and np.array_equal(sims[i, :c].cpu().numpy(), allsims[o])
                and np.array_equal(slens[i, :c].cpu().numpy(), slot_lens[o])):
            bad.append(i)
    assert not bad, bad[:10]


@pytest.mark.parametrize("n,cap,d", [(281, 1000, 64), (5000, 3000, 64), (2000, 4096, 768), (700, 700, 67)])
def test_blas_order_search_with_heavy_ties(pr, n, cap, d):
    """order="blas": sims are the reference's BLAS-order float64 values (oracle/blas_order.c)
    and the top-k is (-sim, seq) over them, incl. dozens of exactly tied rows (hashed
    prompts of one length bucket) and a wrapped ring."""
    g = np.random.default_rng(n + d)
    emb = pr.HashingEmbedder(d)
    stems = [list(range(1000 + b, 1018 + b)) for b in range(12)]
    prompts = [stems[int(g.integers(0, 12))] + g.integers(50_000, 50_040, size=2).tolist() for _ in range(n)]
    rows = np.stack([emb.embed(p) for p in prompts])
    lens = g.integers(1, 2048, size=n)
    Q = np.stack([emb.embed(stems[i % 12] + [50_001, 50_003]) for i in range(48)])
    _check_blas(pr, rows, lens, Q, 8, cap)


@pytest.mark.parametrize("k", [20, 100])
def test_blas_order_large_k_with_heavy_ties(pr, k):
    """top_k above 16 in the reference BLAS order: the CUDA-core path ranks by the same
    BLAS-order sims, ties by seq, incl. tie groups larger than k and a wrapped ring."""
    g = np.random.default_rng(k)
    d, n, cap = 64, 3000, 2500
    emb = pr.HashingEmbedder(d)
    stems = [list(range(1000 + b, 1018 + b)) for b in range(12)]
    prompts = [stems[int(g.integers(0, 12))] + g.integers(50_000, 50_040, size=2).tolist() for _ in range(n)]
    rows = np.stack([emb.embed(p) for p in prompts])
    lens = g.integers(1, 2048, size=n)
    Q = np.stack([emb.embed(stems[i % 12] + [50_001, 50_003]) for i in range(24)])
    _check_blas(pr, rows, lens, Q, k, cap)


# ----------------------------------------------------------------- top_k > 16
@pytest.mark.parametrize("k,n,dtype", [(17, 5000, np.float32), (64, 5000, np.float64), (300, 20000, np.float32),
                                       (1024, 3000, np.float32), (40, 25, np.float32)])
def test_large_k_vs_oracle(pr, k, n, dtype):
    """top_k above the scan's register lists (the CUDA-core coarse pass + exact select):
    seqs / sims / lens bit-exact vs the oracle, incl. planted 11-way duplicate groups
    straddling the k-boundary and a DB smaller than k."""
    g = np.random.default_rng(k + n)
    d, B = 96, 40
    db = g.standard_normal((n, d))
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    if n > 100:
        for grp in range(4):
            db[n // 2 + 11 * grp: n // 2 + 11 * grp + 11] = db[grp]
    if dtype == np.float32:
        db = db.astype(np.float32)
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.concatenate([db[[0, 1, 2, 3]] + 1e-4 * g.standard_normal((4, d)), g.standard_normal((B - 4, d))])
    Q = Q / np.linalg.norm(Q, axis=1, keepdims=True)
    check_batch(pr, db, lens, Q.astype(dtype), k, dtype=dtype)


def test_large_k_predict_batch(pr):
    """predict_batch with top_k = 32 and 200: retrieval aggregates over up to k neighbours
    (numpy pairwise sums above 128 terms), else the MLP; equal to the oracle."""
    g = np.random.default_rng(77)
    n, d = 6000, 64
    db = g.standard_normal((n, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    db[3000:3300] = db[7]  # 300 identical rows: 200 qualifying neighbours for some queries
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.concatenate([db[[7, 8, 9]] + 1e-3 * g.standard_normal((3, d)).astype(np.float32),
                        g.standard_normal((37, d)).astype(np.float32)])
    Q = (Q / np.linalg.norm(Q, axis=1, keepdims=True)).astype(np.float32)
    reg = pr.FallbackRegressor(d, 32, seed=2)
    reg.b2 = 4.0
    store = pr.VectorStore(d, 8192, dtype=np.float32)
    store.add_batch(db, lens)
    for k in (32, 200):
        p = pr.LengthPredictor(pr.PredictorConfig(dimension=d, db_capacity=8192, top_k=k), regressor=reg,
                               store=store)
        out, ret = p.predict_batch(Q)
        ref_len, ref_ret = po.predict_batch(db, lens, np.arange(n), Q, reg.w1, reg.b1, reg.w2, reg.b2, k=k)
        assert np.array_equal(out.cpu().numpy(), ref_len)
        assert np.array_equal(ret.cpu().numpy().astype(bool), ref_ret)
        assert 0 < ref_ret.sum() < len(Q)
        assert p.predict_vector(Q[0])[0] == ref_len[0]
