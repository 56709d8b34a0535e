"""CPU checks of the C-ABI library: it loads, exports every declared symbol,
rejects bad arguments without a GPU, and its own C++ schedule generator
(independent of the oracle) matches Algorithm 1 as the oracle reads it."""
import ctypes
import os
import re

import pytest

from oracle import schedule as OS

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "stragglar.h")


@pytest.fixture(scope="module")
def S():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2505_23523_b200 import stragglar

    return stragglar


def declared_symbols():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(stragglar_\w+)\s*\(", txt, re.M)))


def test_header_declares_api():
    names = declared_symbols()
    for required in ["stragglar_init", "stragglar_allreduce", "stragglar_allreduce_ring", "stragglar_finalize",
                     "stragglar_export_handle", "stragglar_import_handles", "stragglar_team_allreduce"]:
        assert required in names


def test_library_exports_every_declared_symbol(S):
    lib = ctypes.CDLL(S.LIB_PATH)
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert set(declared_symbols()) == set(S.EXPORTED)


def test_library_has_no_libcuda_dependency(S):
    # cudart is static and the driver is reached through the runtime, so the
    # library also loads on a machine without a driver (this CPU container).
    ctypes.CDLL(S.LIB_PATH)


def test_status_strings(S):
    for s in range(8):
        assert S._status_string(s)
    assert S.stragglar_version() >= 100


@pytest.mark.parametrize("world", [2, 4, 8, 16, 32, 64])
def test_cpp_schedule_equals_oracle(S, world):
    """The library's C++ Algorithm 1 vs the oracle: same rounds, same transfers."""
    o = OS.generate_stragglar(world)
    assert S.stragglar_schedule_rounds(world) == o.num_rounds
    for r in range(o.num_rounds):
        got = {(a, b, c, "reduce" if k == 0 else "replace") for a, b, c, k in S.stragglar_schedule_round(world, r)}
        want = {(t.src, t.dst, t.chunk, t.kind) for t in o.rounds[r]}
        assert got == want, (world, r)


@pytest.mark.parametrize("world", [2, 4, 8, 16, 64])
def test_cpp_schedule_verifies(S, world):
    """Independently of the oracle's generator: the C++ schedule passes the
    contributor-set verifier (postcondition P:202, single port P:149-150)."""
    s = OS.Schedule("stragglar", world, world - 1, world - 1)
    for r in range(S.stragglar_schedule_rounds(world)):
        s.rounds.append([OS.Transfer(a, b, c, OS.REDUCE if k == 0 else OS.REPLACE)
                         for a, b, c, k in S.stragglar_schedule_round(world, r)])
    rep = OS.verify_schedule(s)
    assert rep.valid, rep.violations[:3]


@pytest.mark.parametrize("world", [3, 5, 0, 128, 16 + 2])
def test_cpp_schedule_rejects(S, world):
    with pytest.raises(S.StragglarError):
        S.stragglar_schedule_rounds(world)


def test_calls_before_init_fail_cleanly(S):
    """No communicator: collective calls return NOT_INITIALIZED, never crash."""
    with pytest.raises(S.StragglarError) as e:
        S.stragglar_export_handle()
    assert e.value.status == 3
    lib = S._lib
    assert lib.stragglar_allreduce(None, 0, 0, 0, None) == 3
    assert lib.stragglar_team_allreduce(None, 0, 0, 0, None) == 3
    assert lib.stragglar_team_allreduce_ring(None, 16, 1, 0, None) == 3


def test_init_without_gpu_reports_error(S):
    """On this CPU box the runtime finds no device: CUDA error, not a crash.
    Unsupported worlds are rejected before touching CUDA."""
    assert S._lib.stragglar_team_init(3, 0) == 2
    assert S._lib.stragglar_init(0, 5, 0) == 2
    assert S._lib.stragglar_init(0, 16, 0) == 2
    assert S._lib.stragglar_init(5, 4, 0) == 1
    assert S._lib.stragglar_team_init(4, 9) == 1
    st = S._lib.stragglar_team_init(4, 0)
    assert st in (0, 5)
    if st == 0:
        S.stragglar_team_finalize()


@pytest.mark.parametrize("world", [6, 10, 12])
def test_cpp_appendix_b_equals_oracle(S, world):
    """Even non-power-of-2 n: the library's C++ Appendix-B generator vs the oracle."""
    o = OS.generate_stragglar_even(world)
    assert S.stragglar_schedule_rounds(world) == o.num_rounds
    for r in range(o.num_rounds):
        got = {(a, b, c, "reduce" if k == 0 else "replace") for a, b, c, k in S.stragglar_schedule_round(world, r)}
        want = {(t.src, t.dst, t.chunk, t.kind) for t in o.rounds[r]}
        assert got == want, (world, r)


@pytest.mark.parametrize("world", [2, 4, 6, 8, 10, 16, 64])
def test_cpp_broadcast_tree_equals_oracle(S, world):
    """NEXT N3 Broadcast baseline: the library's doubling tree (C++) vs the
    oracle's generate_broadcast, copy by copy and round by round."""
    sender, rnd = S.stragglar_broadcast_tree(world)
    o = OS.generate_broadcast(world)
    want_sender, want_round = [-1] * world, [0] * world
    for r, transfers in enumerate(o.rounds[1:], start=1):
        for t in transfers:
            want_sender[t.dst], want_round[t.dst] = t.src, r
    assert sender == want_sender and rnd == want_round
