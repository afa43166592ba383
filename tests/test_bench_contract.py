"""CPU: bench.py's reference arm (the reference's numpy algorithm on the host cores)
prints one JSON line with the driver contract's keys; rank > 0 under torchrun prints
nothing."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(env_extra=None):
    env = dict(os.environ)
    env.update(env_extra or {})
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "0", "--cpu-planes", "2"], capture_output=True, text=True, env=env,
                         cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr
    return [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    lines = _run()
    assert len(lines) == 1
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "impl", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] in ("reference", "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_silent():
    assert _run({"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}) == []


def test_swap_schedule_is_hazard_free_and_complete():
    """The timed swap pipeline (bench.swap_schedule): over any number of steps every job
    is offloaded and uploaded once per step, an upload reads the slab its own offload
    wrote (no later offload overwrote it first), and uploads follow their offload."""
    sys.path.insert(0, ROOT)
    import bench
    for n in (1, 2, 7, 8, 9, 17, 64, 256):
        for slabs in (2, 3, 8):
            for lag in range(1, slabs):
                for steps in (1, 2, 3):
                    pend, content, uploaded = [], {}, []
                    offs = 0
                    for st in range(steps):
                        for op, j in bench.swap_schedule(n, slabs, lag, pend, st == steps - 1):
                            s = j % slabs
                            if op == "off":
                                assert content.get(s) is None, (n, slabs, lag, "slab overwritten before upload")
                                content[s] = j
                                offs += 1
                            else:
                                assert content.get(s) == j, (n, slabs, lag, "upload reads another job's slab")
                                content[s] = None
                                uploaded.append(j)
                    assert offs == n * steps and sorted(uploaded) == sorted(list(range(n)) * steps)
                    assert not pend
