"""CPU checks of bench.py's multi-rank plumbing: `python bench.py --gpus N`
without torchrun re-launches itself as N ranks through torch.distributed.run
on 127.0.0.1 (the driver's launch), and every rank joins one gloo group."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("n", [2, 3])
def test_self_launch_n_ranks(n):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--launch-check"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout          # rank 0 alone prints
    out = json.loads(lines[0])
    assert out["world"] == n
    assert out["rank_sum"] == n * (n + 1) / 2
    assert out["env"]["MASTER_ADDR"] == "127.0.0.1"


def test_reference_arm_runs_full_workload_unscaled():
    """--impl reference times the oracle on the same config as our arm, with
    no sampling or scaling (the one-line contract)."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "config1",
                        "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["impl"] == "reference" and out["steps"] == 2
    assert "no sampling" in out["cpu_baseline"]["sample"]
    assert out["value"] == out["cpu_baseline"]["value"] == out["e2e"]["value"]
    assert out["ms_per_step"] * 1e3 >= out["value"]
