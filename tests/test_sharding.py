"""CPU multi-process (gloo, world_size 2) coverage of the N>1 host logic: KV job
placement (LPT, no collective) and the predictor's seq-sharded DB + all-gather +
(-sim, seq) merge, checked against the single-process oracle."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from oracle import pred_oracle as po
from paper_2410_23537_b200 import sharding
from harness import synthetic


def test_lpt_balances_c3_jobs():
    ctx = synthetic.sharegpt_job_tokens(256, seed=0)
    assert int(ctx.sum()) == 120_699  # SURVEY §8(d) C3 token count (seed 0)
    for g in (1, 2, 4, 8):
        bins = sharding.lpt_assign(list(ctx), g)
        assert sorted(i for b in bins for i in b) == list(range(256))
        loads = [int(ctx[b].sum()) for b in bins]
        assert (max(loads) - min(loads)) / (sum(loads) / g) < 0.01


def test_shard_fifo_equals_global_fifo():
    C, G, N = 120, 4, 1000
    seqs = np.arange(N)
    live_global = set(seqs[-C:])
    live = set()
    for r in range(G):
        mine = seqs[sharding.shard_rows(seqs, r, G)]
        live |= set(mine[-(C // G):])   # per-shard ring of C/G slots keeps its newest
    assert live == live_global


def test_query_slices_partition_the_batch():
    """layout="queries": the ranks' slices are disjoint, ordered and cover the batch."""
    import types
    for B in (0, 1, 7, 8, 9, 4096):
        for G in (1, 2, 3, 8):
            sl = [sharding.ShardedVectorStore.query_slice(types.SimpleNamespace(world=G, rank=r), B)
                  for r in range(G)]
            assert [i for lo, hi in sl for i in range(lo, hi)] == list(range(B))
            assert all(hi - lo <= -(-B // G) for lo, hi in sl)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, result_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    g = np.random.default_rng(5)
    n, d, B, k = 900, 32, 12, 8
    db = g.standard_normal((n, d)).astype(np.float32)
    db /= np.linalg.norm(db, axis=1, keepdims=True)
    db[500:511] = db[3]          # tie group across both shards
    lens = g.integers(1, 2048, size=n).astype(np.int32)
    Q = np.concatenate([db[[3, 10]], g.standard_normal((B - 2, d)).astype(np.float32)])
    Q /= np.linalg.norm(Q, axis=1, keepdims=True)
    seqs = np.arange(n)
    mine = sharding.shard_rows(seqs, rank, world)
    local = po.search_exact_batch(db[mine], lens[mine], seqs[mine], Q, k)
    sims = torch.zeros((B, k), dtype=torch.float64)
    sq = torch.zeros((B, k), dtype=torch.int64)
    ln = torch.zeros((B, k), dtype=torch.int32)
    cnt = torch.zeros(B, dtype=torch.int32)
    for i, (s, l_, q_) in enumerate(local):
        c = len(q_)
        sims[i, :c] = torch.from_numpy(s)
        sq[i, :c] = torch.from_numpy(q_)
        ln[i, :c] = torch.from_numpy(l_.astype(np.int32))
        cnt[i] = c
    # the sharded search's bound exchange: each shard's local k-th is a lower bound of
    # the global k-th; after the max all-reduce only records at or above it are kept
    # (exact sims here, so no coarse-error margin), and the merge is still exact
    bound = torch.full((B,), -np.inf, dtype=torch.float32)
    for i in range(B):
        if cnt[i] == k:
            bound[i] = float(np.nextafter(np.float32(sims[i, k - 1].item()), np.float32(-np.inf)))
    sharding.all_reduce_max(bound)
    for i in range(B):
        keep = int((sims[i, :cnt[i]] >= bound[i].double()).sum())
        cnt[i] = keep
    gs, gq, gl, gc = sharding.all_gather_records((sims, sq, ln, cnt))
    o_sim, o_seq, o_len, o_cnt = sharding.merge_topk_host(gs.numpy(), gq.numpy(), gl.numpy(), gc.numpy(), k)
    ref = po.search_exact_batch(db, lens, seqs, Q, k)
    ok = all(np.array_equal(o_seq[i], r[2]) and np.array_equal(o_sim[i], r[0]) and
             np.array_equal(o_len[i], r[1]) for i, r in enumerate(ref))
    with open(os.path.join(result_dir, f"r{rank}"), "w") as fh:
        fh.write("ok" if ok else "bad")
    dist.destroy_process_group()


def test_sharded_topk_gloo_world2(tmp_path):
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        assert (tmp_path / f"r{r}").read_text() == "ok"
