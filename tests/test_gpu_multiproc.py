"""The per-process (CUDA IPC) communicator end to end: n processes, one rank
each, all on cuda:0 (this run has one GPU).  Exercises stragglar_init /
export / import / register_buffer / allreduce / allreduce_ring / barrier /
inject_delay exactly as the NVLink mode uses them; results checked bit for bit
against the oracle in tests/mp_worker.py."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,sigma,count,dtype,mover", [
    (2, 1, 100003, "float32", "lsu"),
    (2, 0, 65536, "bfloat16", "tma"),
    (4, 2, 250001, "int32", "tma"),
    (4, 0, 99999, "float32", "lsu"),
    (6, 4, 123457, "bfloat16", "tma"),   # Appendix-B schedule (even non-power-of-2 n)
    (8, 3, 500001, "float32", "tma"),    # the full n = 8 schedule across 8 processes
    (4, 1, 30001, "float32", "tma"),
    (8, 5, 70001, "bfloat16", "lsu"),    # 8 processes, 16-byte loads/stores
    (4, 3, 400003, "float32", "tma+sub"),  # several slices per CTA (sub-slices), system scope
])
def test_multiprocess_ipc(world, sigma, count, dtype, mover):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.build()
    env = dict(os.environ, STRAGGLAR_MOVER=mover.split("+")[0])
    if mover.endswith("+sub"):
        env["STRAGGLAR_SLICE_BYTES"] = "1024"       # 8 CTAs per rank (mp_worker), ~4 KB slices: 16 per CTA
        env["STRAGGLAR_SUBSLICE_BYTES"] = "4096"
        env["STRAGGLAR_SUBSLICES"] = "16"            # (default 1 at system scope)
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp_worker.py"), str(world), str(sigma), str(count), dtype,
                        str(_port())], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "OK" in r.stdout


def test_watchdog_reports_missing_peer():
    """A rank that never arrives: the spin-waits time out (STRAGGLAR_TIMEOUT_MS),
    the kernel exits and stragglar_check_error reports ERR_TIMEOUT (no hang)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.build()
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp_timeout.py"), str(_port())],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.parametrize("world,sigma,mode", [(2, 1, "schedule"), (4, 2, "schedule"), (4, 0, "direct"), (4, 3, "auto")])
def test_ddp_comm_hook(world, sigma, mode):
    """data-parallel training with StragglAR as the
    gradient AllReduce — DDP comm hook vs DDP's default hook, 3 steps."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.build()
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp_ddp.py"), str(world), str(sigma), str(_port()), mode],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-3000:]


@pytest.mark.parametrize("knob,value", [("STRAGGLAR_SUBSLICE_BYTES", "4096"), ("STRAGGLAR_SUB_MAJOR", "0"),
                                         ("STRAGGLAR_E2E_PIECE_BYTES", "65536")])
def test_layout_mismatch_rejected_at_import(knob, value):
    """Ranks with different layout knobs fail at stragglar_import_handles
    (INVALID_ARG) instead of running with different slice layouts, unit
    orders or host-pipeline pieces."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.build()
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp_layout_mismatch.py"), str(_port()), knob, value],
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


def test_k0_probes_move_the_right_bytes():
    """K0: the probe copies land every byte in the right peer
    segment (push / pull, LSU / TMA) and the flag ping-pong completes."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.build()
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp_probe.py"), str(_port())],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
