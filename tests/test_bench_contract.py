"""bench.py's reference arm on CPU (the driver runs it beside the GPU arm): one JSON line with
the contract's keys, the same (barrier step, value stream) list the GPU arm times, and exit 0
for non-zero ranks under torchrun."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True,
                       text=True, env=e, timeout=600, cwd=ROOT)
    return p


def test_reference_arm_json_line():
    p = _run(["--impl", "reference", "--config", "tiny", "--steps", "3", "--warmup", "1"])
    assert p.returncode == 0, p.stderr
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "impl",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["higher_is_better"] is False
    assert d["config"]["barrier_steps"] == [1, 2, 3]
    assert d["config"]["systems_timed"] == 3 * 64
    assert d["cpu_baseline"]["kind"] == "port" and d["e2e"]["h2d_bytes_per_step"] == 0
    assert d["value"] > 0


def test_reference_arm_other_ranks_exit_quietly():
    p = _run(["--impl", "reference", "--config", "tiny", "--steps", "1", "--warmup", "1"],
             env={"RANK": "1", "WORLD_SIZE": "2"})
    assert p.returncode == 0, p.stderr
    assert not [l for l in p.stdout.splitlines() if l.startswith("{")]
