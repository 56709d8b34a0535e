"""Host-side layout logic of libstragglar.so (no GPU): the slices, sub-slices
and Phase-B op lanes a StragglAR call uses (api.cu base_plan / lane_slices /
set_op_lanes).  Co-residency and flag-index safety rest on these
invariants; the named configurations pin the measured choices."""
import math

import pytest

from oracle import schedule as OS


@pytest.fixture(scope="module")
def S():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2505_23523_b200 import stragglar

    return stragglar


ESZ = {0: 4, 1: 4, 2: 2}


def chunk_bytes(count, world, esz):
    v = 16 // esz
    per = -(-count // (world - 1))
    return -(-per // v) * v * esz


def max_ops(world):
    """Most transfers any rank acts in (an exchange counts for both ends) — at most one per round."""
    sched = OS.generate(world)
    acts = {}
    for rnd in sched.rounds:
        for t in rnd:
            acts[t.src] = acts.get(t.src, 0) + 1
            if t.kind == OS.REDUCE:
                acts[t.dst] = acts.get(t.dst, 0) + 1
    return max(acts.values())


@pytest.mark.parametrize("world", [2, 4, 6, 8])
@pytest.mark.parametrize("budget", [1, 8, 37, 74, 148, 296])
@pytest.mark.parametrize("sys_scope", [False, True])
def test_layout_invariants(S, world, budget, sys_scope):
    rounds = S.stragglar_schedule_rounds(world)
    for dtype in (0, 1, 2):
        for count in [1, 7, 1000, 65_536, 524_288, 1 << 20, 13_107_200, 1 << 26]:
            G, sub, lanes = S.stragglar_plan_layout(world, world - 1, count, dtype, budget, sys_scope)
            cb = chunk_bytes(count, world, ESZ[dtype])
            assert 1 <= G <= budget
            assert 1 <= sub <= 16
            assert 1 <= lanes <= rounds                      # at most one op per rank per round (Thm 1 rounds)
            assert G * lanes <= budget                        # co-resident within the CTA budget
            if lanes > 1:
                assert sub == 1
                assert G >= math.ceil(cb / 32768) or G == budget // lanes   # slices stay <= 32 KB
            if sub > 1:
                assert G == budget and lanes == 1
            if lanes == 1 and sub == 1:                       # slices never shrink without buying lanes
                assert G == min(budget, max(1, math.ceil(cb / 16384)))


@pytest.mark.parametrize("world", [4, 6, 8])
def test_lanes_never_exceed_the_busiest_ranks_ops(S, world):
    m = max_ops(world)
    for count in [1, 1000, 65_536, 524_288]:
        _, _, lanes = S.stragglar_plan_layout(world, 0, count, 2, 296)
        assert lanes <= m


def test_named_configurations(S):
    # config 5 (n 8, straggler 3, 1 MiB bf16), team budget 74: 8 slices x 9 lanes (measured best)
    assert S.stragglar_plan_layout(8, 3, 524_288, 2, 74) == (8, 1, 9)
    # config 2 (256 MiB fp32), team budget 74: all CTAs, ~128 KB sub-slices, no lanes
    assert S.stragglar_plan_layout(8, 0, 1 << 26, 1, 74) == (74, 4, 1)
    # the same per process (2 x 148 SMs, system scope): one ~130 KB slice per CTA
    assert S.stragglar_plan_layout(8, 0, 1 << 26, 1, 296, True) == (296, 1, 1)
    # 1 GiB bf16 per process: ~128 KB sub-slices, 4 per CTA
    assert S.stragglar_plan_layout(8, 0, 1 << 29, 2, 296, True) == (296, 4, 1)
    # 2 MiB bf16: 32 KB slices make room for 7 lanes
    assert S.stragglar_plan_layout(8, 0, 1 << 20, 2, 74) == (10, 1, 7)
    # config 1 (n 4, 4 MiB fp32): 43 slices would buy no second lane, so all 74 CTAs keep 1 slice each
    assert S.stragglar_plan_layout(4, 0, 1 << 20, 1, 74) == (74, 1, 1)


def test_layout_rejects_bad_arguments(S):
    with pytest.raises(S.StragglarError):
        S.stragglar_plan_layout(3, 0, 100, 1, 74)
    with pytest.raises(S.StragglarError):
        S.stragglar_plan_layout(8, 8, 100, 1, 74)
    with pytest.raises(S.StragglarError):
        S.stragglar_plan_layout(8, 0, 100, 7, 74)



@pytest.mark.parametrize("dtype", [0, 1, 2])
@pytest.mark.parametrize("piece", [1, 16, 4096, 100_000, 8 << 20])
@pytest.mark.parametrize("count", [0, 1, 7, 8, 1000, 65_539, 1 << 20, (1 << 26) + 3])
def test_e2e_pieces(S, dtype, piece, count):
    """The host-buffer pipeline's pieces (one collective call each, so every
    rank must cut the same ones): they tile [0, count) in order, every piece
    but the last has the piece size rounded down to the kernels' 16-byte
    vector (at least one vector), the last takes the rest."""
    esz = ESZ[dtype]
    v = 16 // esz
    lens = S.stragglar_plan_e2e_pieces(count, dtype, piece)
    steady = max(v, piece // esz // v * v)
    assert sum(lens) == count and all(n > 0 for n in lens)
    assert lens[:-1] == [steady] * (len(lens) - 1)
    assert len(lens) == -(-count // steady)


def test_e2e_pieces_config2(S):
    """Config 2's host pipeline: 256 MiB fp32 per rank in 32 pieces of 8 MiB."""
    assert S.stragglar_plan_e2e_pieces(1 << 26, 1, 8 << 20) == [(8 << 20) // 4] * 32
