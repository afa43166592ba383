"""Pure-Python restatement of the swap scheduler's control plane — TEST INFRASTRUCTURE ONLY.

Restates the reference (``pkg/src/servesim``):
  * ``ewt_ms``            kvmanager.py:276-294
  * ``plan_swaps``        kvmanager.py:297-322 (returns per-entry actions)
  * ``rank_and_plan``     simcore.py:439-462 (_Run._ranked_with_grants)

Used by ``tests/test_control_plane.py`` as the checker of the C++ control plane
(``csrc/control.cpp``) where the reference package is not importable, and by
``bench.py``'s CPU leg as the timed Python baseline.  Pinned to the reference by the
same tests (bit-identical EWT floats and plans on random inputs).
"""
from __future__ import annotations

import math

GPU, CPU, NONE, UPLOADING, OFFLOADING = 0, 1, 2, 3, 4


def ewt_ms(levels, last_promotion_us, remaining_ms, aging_ms: float, now_us: int) -> list:
    out = []
    ahead = 0.0
    for lev, lp, rem in zip(levels, last_promotion_us, remaining_ms):
        if math.isinf(aging_ms):
            promote = math.inf
        else:
            waited_ms = (now_us - lp) / 1000.0
            promote = max(lev * aging_ms - waited_ms, 0.0)
        out.append(min(ahead, promote))
        ahead += rem
    return out


def plan_swaps(residency, need_gpu_bytes, budget: int) -> list:
    """Actions per entry: 0 denied, 1 granted, 2 granted + upload, 3 denied + offload."""
    used = 0
    act = []
    for res, need in zip(residency, need_gpu_bytes):
        if used + need <= budget:
            used += need
            act.append(2 if res == CPU else 1)
        else:
            act.append(3 if res == GPU else 0)
    return act


def rank_and_plan(levels, last_promotion_us, remaining_ms, residency, need_gpu_bytes, aging_ms: float,
                  now_us: int, budget: int):
    """-> (order, actions, ewts) as alise_rank_and_plan."""
    ewts = ewt_ms(levels, last_promotion_us, remaining_ms, aging_ms, now_us)
    by_level: dict = {}
    for pos, (lev, e) in enumerate(zip(levels, ewts)):
        by_level.setdefault(lev, []).append((e, pos))
    order = []
    for lev in sorted(by_level):
        for e, pos in sorted(by_level[lev]):
            if residency[pos] in (UPLOADING, OFFLOADING):
                continue
            order.append(pos)
    act = plan_swaps([residency[i] for i in order], [need_gpu_bytes[i] for i in order], budget)
    return order, act, ewts
