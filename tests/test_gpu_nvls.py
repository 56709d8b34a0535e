"""NEXT row N1(i): the NVLS (multicast) variant.

* One GPU: the multicast instructions and the VMM/multicast plumbing through a
  one-member multicast object (stragglar_nvls_selftest): a reducing load
  through it returns the member's own data, bit for bit, for every dtype.
* One GPU, several processes: the kernel's synchronisation with the multicast
  operations emulated through IPC peer pointers (tests/mp_nvls_emu.py), bit-exact.
* Two or more GPUs: the whole variant (tests/mp_nvls.py), one process per GPU,
  against the plain definition within the north_star tolerance (int32 exact;
  the switch's summation order is unspecified), ranks bitwise identical.
  Skips only with fewer than 2 GPUs."""
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


@pytest.fixture(scope="module")
def S():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import __graft_entry__

    __graft_entry__.build()
    from paper_2505_23523_b200 import stragglar

    return stragglar


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16, torch.int32])
@pytest.mark.parametrize("count", [8, 4096, (1 << 20) + 8])
def test_selftest_one_member_multicast(S, dtype, count):
    torch.cuda.set_device(0)
    if not S.stragglar_nvls_supported():
        pytest.skip("this GPU reports no multicast support")
    g = torch.Generator().manual_seed(count)
    if dtype == torch.int32:
        x = torch.randint(-2**31, 2**31 - 1, (count,), generator=g, dtype=torch.int64).to(torch.int32)
    else:
        x = torch.randn(count, generator=g).to(dtype)
    try:
        y = S.stragglar_nvls_selftest(x)
    except S.StragglarError as e:
        if e.status == 2:
            pytest.skip("the driver creates no multicast object on this GPU (no NVSwitch fabric: "
                        "cuMulticastCreate -> CUDA_ERROR_INVALID_VALUE, scripts/mc_selftest.cu)")
        raise
    assert torch.equal(x.view(torch.int16 if dtype == torch.bfloat16 else torch.int32),
                       y.view(torch.int16 if dtype == torch.bfloat16 else torch.int32))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("dtype", ["float32", "bfloat16", "int32"])
def test_nvls_allreduce_multi_gpu(S, dtype):
    n = torch.cuda.device_count()
    if n < 2:
        pytest.skip(f"{n} GPU visible: the NVLS variant needs >= 2 GPUs (one per rank)")
    world = 8 if n >= 8 else (4 if n >= 4 else 2)
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp_nvls.py"), str(world), "1", str(600_016), dtype,
                        str(_port())], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "OK" in r.stdout


@pytest.mark.parametrize("world,sigma,count,dtype", [
    (2, 1, 40_000, "float32"),
    (4, 2, 250_000, "bfloat16"),
    (6, 5, 123_456, "int32"),
    (8, 3, 524_288, "bfloat16"),      # config 5's shape
])
def test_nvls_protocol_emulated(S, world, sigma, count, dtype):
    """The NVLS kernel's flags / epochs / hand-offs with the multicast operations
    emulated through IPC peer pointers (processes sharing this GPU): bit-exact vs
    the oracle's StragglAR result on every rank, three calls back to back."""
    r = subprocess.run([sys.executable, os.path.join(HERE, "mp_nvls_emu.py"), str(world), str(sigma), str(count), dtype,
                        str(_port())], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
