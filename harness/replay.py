"""Config-5 trace replay: drive the real KV data plane with the swap-call stream of the
reference simulator.

``tests/golden/record_c5.py`` runs the reference ``servesim.simcore.run`` (speculative
policy, Alpaca arrivals, Llama-2-13B, INT8 KV, 8 replicas) with a recording
``MemoryState`` and stores every ``start_offload`` / ``start_upload`` / ``complete``
call with the ledger after it.  ``replay`` re-issues those calls, in order, on a
``DeviceMemoryState`` whose jobs are bound to real fp16 KV tensors in HBM, so each
offload quantizes a job and streams it to pinned host memory and each upload brings
it back dequantized.  It checks after every call that the ledger (GPU/CPU bytes,
swap counts and bytes) equals the reference's, and (check_data) that sampled
(layer, K|V) planes of every job's KV after its first round trip -- after every upload
in delta mode -- equal fp16(oracle dequantize(oracle quantize(original))), the C
restatement of kvmanager.py:108-154 (harness/parity.py).
"""
from __future__ import annotations

import gzip
import json
import time

from paper_2410_23537_b200 import kvmanager as km


def load(path):
    with gzip.open(path, "rt") as fh:
        return json.load(fh)


def tokens_of(link_bytes: int, layers: int, hidden: int, bits: int) -> int:
    """Invert quantized_kv_bytes (kvmanager.py:69-82) for the job's token count."""
    ch = 2 * layers * hidden
    per = (bits + 7) // 8
    t, rem = divmod(link_bytes - ch * km.SCALE_ZP_BYTES, ch * per)
    if rem or t <= 0:
        raise ValueError(f"link bytes {link_bytes} are not a quantized KV footprint")
    return t


def _planes(t, planes, T):
    """Host copies of the given (layer, K|V) planes' first T tokens."""
    return {p: t[p // 2, p % 2, :T].cpu().numpy() for p in planes}


def replay(rec: dict, replica: int = 0, group: int = 128, check_data: bool = True, seed: int = 0,
           max_events: int | None = None, delta: bool = False, return_state: bool = False,
           check_planes=(0, 1, 79)):
    """Replay one replica's swap calls; returns a summary dict.

    delta=True: jobs keep their KV in a tensor of their final (trace-maximum) token
    capacity and DeviceMemoryState(delta=True) re-offloads only the tokens generated
    since a job's host copy was written (same ledger, fewer bytes on the link)."""
    import numpy as np
    import torch

    from harness import parity, synthetic

    layers, hidden, heads = rec["model"]
    planes = [p for p in check_planes if p < 2 * layers]
    bits = rec["bits"]
    events = rec["replicas"][replica]["events"]
    if max_events:
        events = events[:max_events]
    f = {name: i for i, name in enumerate(rec["fields"])}
    # pinned pool: the peak of concurrently held host slabs (+ alignment slack)
    peak_cpu = max(e[f["cpu_used"]] for e in events) if events else 0
    cap = {}
    for e in events:
        if e[0] == "o":
            cap[e[1]] = max(cap.get(e[1], 0), tokens_of(e[2], layers, hidden, bits))
    # delta mode keeps clean host copies beyond the ledger: give the pool the room of
    # every job's capacity slab (it still evicts oldest-first when full)
    pool_bytes = int(peak_cpu * 1.02) + (256 << 20)
    if delta:
        pool_bytes = max(pool_bytes, sum(km.KVLayout(layers, T, hidden, hidden // heads, kind="rows", group=group,
                                                     bits=bits).geometry()["slab_bytes"] + 256
                                         for T in cap.values()) + (256 << 20))
    ms = km.DeviceMemoryState(gpu_capacity=rec["gpu_capacity"], cpu_capacity=rec["cpu_capacity"],
                              pcie_bytes_per_ms=rec["pcie_bytes_per_ms"], host_pool_bytes=pool_bytes,
                              delta=delta)
    dev = torch.device("cuda", torch.cuda.current_device())
    kv = {}          # job -> (tensor, layout)
    orig = {}        # check_data: job -> sampled planes of its original (never re-quantized) KV
    valid = {}       # job -> valid tokens
    expect = {}      # non-delta: jobs whose first round trip is still to be checked
    inflight = {}    # job -> TransferCommand
    mismatches = 0
    data_checked = 0
    moved = 0
    # each job's KV is materialised at its first offloaded size (and its D2D round-trip
    # reference computed) before the timed replay; jobs that decode while resident grow
    # between swaps, which the replay applies outside the timed region
    for e in events:
        op, job, link = e[0], e[1], e[2]
        if op != "o" or job in kv:
            continue
        T = tokens_of(link, layers, hidden, bits)
        t = synthetic.kv_job_torch(layers, T, hidden, seed=seed, job=job, group=group, device=dev)
        if delta:
            full = torch.zeros(layers, 2, cap[job], hidden, dtype=t.dtype, device=dev)
            full[:, :, :T] = t
            t = full
        lay = km.KVLayout(layers, t.shape[2], hidden, hidden // heads, kind="rows", group=group, bits=bits)
        kv[job] = (t, lay)
        valid[job] = T
        if check_data:
            orig[job] = _planes(t, planes, T)
            if not delta:
                expect[job] = True
        ms.bind(job, t, lay, tokens=T)
    ms._ensure()  # engine + pinned pool created before the timed replay
    torch.cuda.synchronize()
    paused = 0.0
    t_start = time.perf_counter()
    for e in events:
        op, job, link, gpu_b, t0, t1 = e[0], e[1], e[2], e[3], e[4], e[5]
        # the engine reserves / releases bytes directly between swap calls (KV growth,
        # admissions, completions); adopt its ledger before each call, check after
        ms.gpu_used, ms.cpu_used = e[f["gpu_before"]], e[f["cpu_before"]]
        if op == "o":
            T = tokens_of(link, layers, hidden, bits)
            if T != valid[job]:
                # the job decoded while resident: grow its KV (engine work, not timed)
                torch.cuda.synchronize()
                tp = time.perf_counter()
                old, lay0 = kv[job]
                extra = synthetic.kv_job_torch(layers, T - valid[job], hidden, seed=seed + 1, job=job,
                                               group=group, device=dev)
                if delta:
                    old[:, :, valid[job]:T] = extra
                    ms.set_tokens(job, T)
                else:
                    t = torch.cat([old, extra], dim=2).contiguous()
                    lay = km.KVLayout(layers, T, hidden, hidden // heads, kind="rows", group=group, bits=bits)
                    kv[job] = (t, lay)
                    ms.bind(job, t, lay)
                if check_data and (delta or job in expect):   # the new tokens are original too
                    ext = _planes(extra, planes, T - valid[job])
                    orig[job] = {p: np.concatenate([orig[job][p], ext[p]]) for p in planes}
                valid[job] = T
                torch.cuda.synchronize()
                paused += time.perf_counter() - tp
            before = ms._host_valid.get(job, 0) if delta and job in ms._kept else 0
            inflight[job] = ms.start_offload(job, link, gpu_b, t0)
            moved += 2 * 2 * layers * hidden * (T - before)
        elif op == "u":
            inflight[job] = ms.start_upload(job, link, gpu_b, t0)
            moved += 2 * 2 * layers * hidden * valid[job]
        else:
            cmd = inflight.pop(job)
            ms.complete(cmd)
            if cmd.direction == "upload" and check_data and (delta or job in expect):
                # a job's first round trip (every upload in delta mode: each token is
                # quantized once, from its original values) vs the oracle, sampled planes
                torch.cuda.synchronize()
                tp = time.perf_counter()
                T = valid[job]
                lay_t = km.KVLayout(layers, T, hidden, hidden // heads, kind="rows", group=group, bits=bits)
                bad = parity.kv_roundtrip_planes(lay_t, orig[job], _planes(kv[job][0], planes, T))
                mismatches += len(bad)
                data_checked += 1
                expect.pop(job, None)
                paused += time.perf_counter() - tp
        got = (ms.gpu_used, ms.cpu_used, ms.swap_in_count, ms.swap_out_count, ms.swap_in_bytes,
               ms.swap_out_bytes)
        want = tuple(e[f[k]] for k in ("gpu_used", "cpu_used", "swap_in_count", "swap_out_count",
                                       "swap_in_bytes", "swap_out_bytes"))
        if got != want:
            raise AssertionError(f"ledger diverged at {e}: got {got} want {want}")
    torch.cuda.synchronize()
    wall = time.perf_counter() - t_start - paused
    modeled_s = (max((e[5] for e in events), default=0) - min((e[4] for e in events), default=0)) / 1e6
    link_total = ms.swap_in_bytes + ms.swap_out_bytes
    out = {"replica": replica, "events": len(events), "swaps_out": ms.swap_out_count,
           "swaps_in": ms.swap_in_count, "link_bytes": link_total, "fp16_bytes_moved": moved,
           "link_bytes_moved": ms.link_bytes_moved, "delta": delta,
           "wall_s": wall, "fp16_GBs": moved / wall / 1e9 if wall else None,
           "link_GBs": link_total / wall / 1e9 if wall else None,
           "modeled_span_s": modeled_s, "data_checked": data_checked, "data_mismatches": mismatches}
    if return_state:  # every job's valid KV at the end (tests)
        out["state"] = {j: kv[j][0][:, :, :valid[j]] for j in kv}
    if ms.host_pool is not None:
        ms.host_pool.close()
    if ms.engine is not None:
        ms.engine.close()
    return out
