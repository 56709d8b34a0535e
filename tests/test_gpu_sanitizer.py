"""compute-sanitizer memcheck and racecheck over small team-mode calls of
every kernel (both movers), results checked against the oracle inside."""
import os
import shutil
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sanitizer():
    """The compute-sanitizer binary, or skip: not installed, or closed by the
    GPU pool (its wrapper then refuses every run, exit code 86)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    cs = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    if not os.path.exists(cs):
        pytest.skip("compute-sanitizer not installed")
    r = subprocess.run([cs, "--version"], capture_output=True, text=True, timeout=120)
    if r.returncode != 0 or "closed" in (r.stdout + r.stderr):
        pytest.skip("compute-sanitizer unavailable on this pool: " + (r.stdout + r.stderr).strip()[:200])
    return cs


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
@pytest.mark.parametrize("mover", ["tma", "lsu"])
def test_sanitizer_clean(tool, mover):
    cs = _sanitizer()
    import __graft_entry__

    __graft_entry__.build()
    env = dict(os.environ, STRAGGLAR_MOVER=mover, STRAGGLAR_TIMEOUT_MS="120000")
    r = subprocess.run([cs, "--tool", tool, "--error-exitcode", "9", sys.executable,
                        os.path.join(ROOT, "tests", "sanitize_step.py")],
                       env=env, capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert "sanitize step ok" in out


@pytest.mark.parametrize("tool", ["memcheck", "racecheck"])
def test_sanitizer_clean_ipc_ranks(tool):
    """The per-process mode: two ranks (torchrun, each under its own
    compute-sanitizer) exchanging CUDA-IPC peer mappings; every algorithm runs
    once and is checked against the oracle inside tests/mp_rank_sanitize.py."""
    cs = _sanitizer()
    import __graft_entry__

    __graft_entry__.build()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr", "127.0.0.1",
                        "--nproc-per-node", "2", "--no-python", cs, "--tool", tool, "--error-exitcode", "9",
                        sys.executable, os.path.join(ROOT, "tests", "mp_rank_sanitize.py")],
                       capture_output=True, text=True, timeout=900)
    out = r.stdout + r.stderr
    assert r.returncode == 0, out[-3000:]
    assert out.count("mismatches []") == 2, out[-3000:]
