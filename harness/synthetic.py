"""Seeded synthetic inputs for the BASELINE.json configs (no datasets, no network).

KV values follow SURVEY.md §8(d) C1: standard normal, every 16th hidden channel x40
(outliers), 1% of groups constant, 10% of groups single-sign (|x| + U(0, 500)).
Job lengths follow the reference's ShareGPT preset (workload.py:121-130:
lognormal input mu 4.6 s 1.1, output mu 5.0 s 1.2, clamped to [1, 2048]) drawn
from the reference's PCG64 stream layout (rng.py:20-22, TRACE_LENGTHS = 2).
"""
from __future__ import annotations

import numpy as np

TRACE_LENGTHS = 2      # rng.py stream tag
SHAREGPT = dict(input_mu=4.6, input_sigma=1.1, output_mu=5.0, output_sigma=1.2, max_len=2048)


def stream(seed: int, tag: int, *sub: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed, tag, *sub])))


def kv_job(layers: int, tokens: int, hidden: int, seed: int = 0, job: int = 0, group: int = 64,
           dtype=np.float16) -> np.ndarray:
    """One job's KV as [layers, 2, tokens, hidden] with the C1 value mix."""
    g = np.random.default_rng([seed, job])
    x = g.standard_normal((layers, 2, tokens, hidden), dtype=np.float32)
    x[..., ::16] *= 40.0
    flat = x.reshape(-1, group)
    ng = flat.shape[0]
    pick = g.random(ng)
    const = pick < 0.01
    single = (pick >= 0.01) & (pick < 0.11)
    flat[const] = flat[const, :1]
    flat[single] = np.abs(flat[single]) + g.uniform(0.0, 500.0, size=(int(single.sum()), 1)).astype(np.float32)
    return x.astype(dtype)


def kv_job_torch(layers: int, tokens: int, hidden: int, seed: int = 0, job: int = 0,
                 group: int = 64, device="cuda"):
    """Same distribution generated directly on the device (for GiB-scale benches)."""
    import torch

    gen = torch.Generator(device=device)
    gen.manual_seed(seed * 1_000_003 + job)
    x = torch.randn((layers, 2, tokens, hidden), generator=gen, device=device, dtype=torch.float32)
    x[..., ::16] *= 40.0
    flat = x.view(-1, group)
    pick = torch.rand(flat.shape[0], generator=gen, device=device)
    const = pick < 0.01
    single = (pick >= 0.01) & (pick < 0.11)
    flat[const] = flat[const, :1].expand(-1, group)
    off = torch.rand((flat.shape[0], 1), generator=gen, device=device) * 500.0
    flat[single] = flat[single].abs() + off[single]
    return x.to(torch.float16)


def sharegpt_job_tokens(n_jobs: int = 256, seed: int = 0) -> np.ndarray:
    """Context tokens (input + output) of n_jobs ShareGPT-like requests."""
    g = stream(seed, TRACE_LENGTHS)
    p = SHAREGPT
    ins = g.lognormal(p["input_mu"], p["input_sigma"], size=n_jobs)
    outs = g.lognormal(p["output_mu"], p["output_sigma"], size=n_jobs)
    ins = np.clip(np.rint(ins), 1, p["max_len"]).astype(int)
    outs = np.clip(np.rint(outs), 1, p["max_len"]).astype(int)
    return ins + outs


def lpt_assign(weights, n_bins: int) -> list:
    """Longest-processing-time-first assignment of jobs to GPUs.

    Returns one list of job indices per bin; ties go to the lowest bin index.
    """
    order = sorted(range(len(weights)), key=lambda i: (-weights[i], i))
    loads = [0] * n_bins
    bins = [[] for _ in range(n_bins)]
    for i in order:
        b = min(range(n_bins), key=lambda j: (loads[j], j))
        bins[b].append(i)
        loads[b] += weights[i]
    return [sorted(b) for b in bins]


def predictor_db(n: int, dim: int, seed: int = 0, dup_groups: int = 0, dup_size: int = 11):
    """Unit-norm fp32 DB rows (Gaussian), ShareGPT-like output lengths, planted
    groups of exact duplicate rows (tie tests).  Returns (vecs f32 [n,dim], lens i32 [n])."""
    g = np.random.default_rng([seed, 77])
    v = g.standard_normal((n, dim), dtype=np.float32)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    for k in range(dup_groups):
        base = int(g.integers(0, n - dup_size))
        idx = g.choice(n, size=dup_size - 1, replace=False)
        v[idx] = v[base]
    lens = np.clip(np.rint(g.lognormal(SHAREGPT["output_mu"], SHAREGPT["output_sigma"], size=n)),
                   1, SHAREGPT["max_len"]).astype(np.int32)
    return v, lens


def predictor_queries(db: np.ndarray, b: int, seed: int = 0, near_frac: float = 0.5,
                      noise: float = 0.015):
    """b unit-norm fp32 queries: near-duplicates of DB rows (retrieved) and random
    directions (fall back to the MLP)."""
    g = np.random.default_rng([seed, 78])
    n, dim = db.shape
    nn = int(b * near_frac)
    q = g.standard_normal((b, dim), dtype=np.float32)
    src = g.integers(0, n, size=nn)
    q[:nn] = db[src] + noise * g.standard_normal((nn, dim), dtype=np.float32)
    q /= np.linalg.norm(q, axis=1, keepdims=True)
    return q.astype(np.float32)


def predictor_db_torch(n: int, dim: int, seed: int = 0, dup_groups: int = 0, dup_size: int = 11,
                       device="cuda"):
    """Device-side twin of predictor_db for GiB-scale benches (same distribution
    family, torch generator): unit-norm fp32 rows with planted duplicate groups and
    ShareGPT-like lengths."""
    import torch
    gen = torch.Generator(device=device)
    gen.manual_seed(seed * 7919 + 77)
    v = torch.randn((n, dim), generator=gen, device=device, dtype=torch.float32)
    v /= v.norm(dim=1, keepdim=True)
    if dup_groups:
        src = torch.randint(0, n, (dup_groups,), generator=gen, device=device)
        dst = torch.randint(0, n, (dup_groups, dup_size - 1), generator=gen, device=device)
        v[dst.reshape(-1)] = v[src].repeat_interleave(dup_size - 1, dim=0)
    ln = torch.exp(SHAREGPT["output_mu"] + SHAREGPT["output_sigma"] *
                   torch.randn(n, generator=gen, device=device, dtype=torch.float64))
    lens = ln.round().clamp(1, SHAREGPT["max_len"]).to(torch.int32)
    return v, lens


def predictor_queries_torch(db, b: int, seed: int = 0, near_frac: float = 0.5, noise: float = 0.015):
    import torch
    gen = torch.Generator(device=db.device)
    gen.manual_seed(seed * 7919 + 78)
    n, dim = db.shape
    nn = int(b * near_frac)
    q = torch.randn((b, dim), generator=gen, device=db.device, dtype=torch.float32)
    src = torch.randint(0, n, (nn,), generator=gen, device=db.device)
    q[:nn] = db[src] + noise * torch.randn((nn, dim), generator=gen, device=db.device)
    q /= q.norm(dim=1, keepdim=True)
    return q
