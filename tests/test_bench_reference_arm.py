"""bench.py on the host alone: the reference arm (the unmodified reference,
baseline/_ref, timed on the CPU) carries the contract's keys, and
``--gpus N`` without torchrun launches N ranks itself."""

from __future__ import annotations

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(r):
    assert r.returncode == 0, r.stderr[-2000:]
    return json.loads(r.stdout.strip().splitlines()[-1])


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300)
    line = _last_json(r)
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["metric"] == "rank-loss train samples/sec" and line["unit"] == "samples/s"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    import refbench

    assert line["cpu_baseline"]["kind"] == ("reference" if refbench.available() else "port")
    assert line["cpu_baseline"]["host"]["logical_cpus"] >= 1


@pytest.mark.parametrize("n", [2, 3])
def test_gpus_n_without_torchrun_launches_n_ranks(n):
    """`bench.py --gpus 8` silently ran one rank.  Now it spawns
    the N ranks (127.0.0.1 rendezvous); the selftest mode checks the launcher
    and the max-over-ranks reduction with gloo."""
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, "bench.py", "--gpus", str(n), "--selftest-launch"],
                       cwd=ROOT, capture_output=True, text=True, timeout=300, env=env)
    line = _last_json(r)
    assert line == {"selftest": True, "n_gpus": n, "ranks_joined": n, "max_rank": n - 1}
