"""BASELINE config 5 on the real data plane.

* Recorded replay (tests/golden/record_c5.py): all 8 replicas' swap-call streams
  re-issued on DeviceMemoryState with real Llama-2-13B KV; the ledger equals the
  reference's after every call, and sampled planes of every job's first round trip
  (every upload in delta mode) equal the oracle's quantize/dequantize.
* Live: the reference simulator itself (simcore.run, speculative, Alpaca) with its
  _Run.memory built as a DeviceMemoryState over real per-job KV (harness/live.py);
  the MetricsReport is identical to the pure reference run's (recorded in the
  fixture), and sampled planes of the swaps equal the oracle's round trip."""
import json
import os

import pytest

from harness import refsim
from tests.conftest import GOLDEN, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def rec():
    from harness import replay
    return replay.load(os.path.join(GOLDEN, "c5_swaps.json.gz"))


@pytest.mark.slow
@pytest.mark.parametrize("delta", [False, True])
def test_c5_replay_all_replicas_oracle_checked(rec, delta):
    from harness import replay
    checked = swaps = 0
    for r in range(len(rec["replicas"])):
        out = replay.replay(rec, replica=r, delta=delta, check_planes=(79,) if delta else (0, 79))
        assert out["data_mismatches"] == 0, (r, out)
        checked += out["data_checked"]
        swaps += out["swaps_out"] + out["swaps_in"]
    assert len(rec["replicas"]) == 8 and checked > 500 and swaps > 10_000


@pytest.mark.parametrize("replica", [0, 5])
def test_c5_live_engine_identical_report(rec, replica):
    if refsim.import_servesim() is None:
        pytest.skip("reference package not importable here")
    from harness import live
    report, stats, _wall = live.run_replica(replica, check_planes=(0, 79), check_every=4)
    assert json.loads(report) == rec["replicas"][replica]["report"]
    assert stats["swaps_out"] > 100 and stats["swaps_in"] > 100
    assert stats["planes_checked"] > 20 and stats["mismatches"] == 0, stats


@pytest.mark.slow
def test_c5_live_engine_all_replicas(rec):
    if refsim.import_servesim() is None:
        pytest.skip("reference package not importable here")
    from harness import live
    for r in range(8):
        report, stats, _wall = live.run_replica(r, check_planes=(79,), check_every=16)
        assert json.loads(report) == rec["replicas"][r]["report"], r
        assert stats["mismatches"] == 0, (r, stats)
