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


def test_nccl_log_summary_parses_version_nranks_algos_and_nvls(tmp_path):
    """bench.py's NCCL_DEBUG=INFO reader (the N>1 line's `nccl.log_rank0`): version,
    communicator sizes, the algorithms the tuner logged, and whether NCCL found
    NVLS usable (which gates the NCCL_ALGO=NVLS arm)."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    log = tmp_path / "nccl_bench_r0.123.log"
    log.write_text(
        "host:123:123 [0] NCCL INFO NCCL version 2.28.9+cuda12.9\n"
        "host:123:200 [0] NCCL INFO NVLS multicast support is available on dev 0\n"
        "host:123:200 [0] NCCL INFO ncclCommInitRankConfig comm 0x1 rank 0 nRanks 8 nNodes 1 localRanks 8 localRank 0 MNNVL 0\n"
        "host:123:200 [0] NCCL INFO ncclCommInitRankConfig comm 0x1 rank 0 nranks 8 cudaDev 0 nvmlDev 0 busId 1000 commId 0x2 - Init COMPLETE\n"
        "host:123:200 [0] NCCL INFO AllReduce: opCount 0 sendbuff 0x1 recvbuff 0x1 count 16 datatype 7 op 0 root 0 comm 0x1 [nranks=8] stream 0x3\n"
        "host:123:200 [0] NCCL INFO AllReduce: 268435456 Bytes -> Algo NVLS proto SIMPLE channel{Lo..Hi}={0..15}\n"
        "host:123:200 [0] NCCL INFO AllReduce: 268435456 Bytes -> Algo RING proto SIMPLE channel{Lo..Hi}={0..31}\n")
    out = bench._nccl_log_summary(str(tmp_path / "nccl_bench_r0.*.log"))
    assert out["version"] == "2.28.9+cuda12.9"
    assert out["nranks"] == [8]
    assert out["algos"] == {"NVLS": 1, "RING": 1}
    assert out["nvls_available"] is True and out["files"] == 1
    log.write_text("x NCCL INFO NVLS multicast support is not available on dev 0\n")
    assert bench._nccl_log_summary(str(tmp_path / "nccl_bench_r0.*.log"))["nvls_available"] is False


def test_nvlink_roofline_per_phase():
    """The N>1 line's roofline at config 2, n = 8, with made-up K0 ceilings:
    Phase A (n-2)C per port over T_A, Phase B R*C over T_post."""
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod2", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    C = bench.chunk_bytes(1 << 26, 7, 4)
    assert C == 38_347_936                                   # SURVEY §8(a) sizes table
    r = bench.nvlink_roofline(6 * C, 9 * C, 300.0, 450.0, 800.0, 700.0)
    assert r["bound"] == "nvlink" and r["unit"] == "GB/s"
    assert abs(r["phase_A"]["achieved"] - 6 * C / 300e-6 / 1e9) < 0.1
    assert abs(r["phase_B"]["achieved"] - 9 * C / 450e-6 / 1e9) < 0.1
    assert r["frac"] == r["phase_B"]["frac_k0"] == round(9 * C / 450e-6 / 1e9 / 700.0, 3)
    assert r["phase_A"]["frac_nominal_900"] == round(6 * C / 300e-6 / 1e9 / 900.0, 3)


def test_nvlink_counter_parser():
    import importlib.util

    spec = importlib.util.spec_from_file_location("bench_mod3", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    txt = ("GPU 0: NVIDIA B200 (UUID: GPU-x)\n\t Link 0: Data Tx: 1024 KiB\n\t Link 0: Data Rx: 2048 KiB\n"
           "\t Link 1: Data Tx: 3 KiB\n\t Link 1: Data Rx: 0 KiB\n")
    assert bench.parse_nvlink_counters(txt) == (1027 * 1024.0, 2048 * 1024.0)
    # what this round's one-GPU box prints (profiles/r02/nvlink_gt.txt): no numbers
    assert bench.parse_nvlink_counters("GPU 0: NVIDIA B200\n\t Link 0: Data Tx: N/A\n\t Link 0: Data Rx: N/A\n") is None
