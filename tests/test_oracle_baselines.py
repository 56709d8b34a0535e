"""Pins for the oracle's NEXT-N3 baselines: recursive
halving/doubling (RHD) and the straggler-aware Broadcast
(P:368-373).  CPU only.  Pinned against Table 1 / P:366 / P:373 closed forms
(via oracle.cost, which is pinned to the paper's worked numbers in
test_oracle_cost.py), the contributor-set verifier (pinned to SPEC's examples
in test_oracle_schedule.py), integer brute force, exactness of integer-valued
floats, torch's own add at n = 2, the recursive-summation error bound, and the
plain definition of the StragglAR result (itself pinned in
test_oracle_numerics.py)."""
from fractions import Fraction
import math

import numpy as np
import pytest
import torch

from oracle import cost as C
from oracle import numerics as N
from oracle import schedule as S
from paper_2505_23523_b200.inputs import make_inputs

DT = ("int32", "float32", "bfloat16")


def _bits(a):
    return np.asarray(a).view(np.uint8)


def _wrap_sum(xs):
    exact = np.zeros(xs[0].size, dtype=np.int64)
    for x in xs:
        exact += x.astype(np.int64)
    return ((exact + 2 ** 31) % 2 ** 32 - 2 ** 31).astype(np.int32)


# ---------------------------------------------------------------- RHD schedule
@pytest.mark.parametrize("n", [2, 4, 8, 16, 32, 64])
def test_rhd_rounds_beta_table1(n):
    """T_RHD = 2 log n alpha + 2 (n-1)/n s beta — the schedule's round
    count is the alpha coefficient and its per-port volume the beta one."""
    s = S.generate_rhd(n)
    rep = S.verify_schedule(s)
    assert rep.valid, rep.violations[:3]
    assert s.num_rounds == 2 * int(math.log2(n)) == C.t_rhd(n, 0.0, 1.0, 0.0)
    assert rep.beta_coefficient == Fraction(2 * (n - 1), n)
    assert float(rep.beta_coefficient) == pytest.approx(C.t_rhd(n, 1.0, 0.0, 1.0))


@pytest.mark.parametrize("n", [4, 8, 16])
def test_rhd_halving_structure(n):
    """round t of the ReduceScatter pairs every rank with one
    partner and moves 1/2^(t+1) of the buffer; the AllGather mirrors it."""
    s = S.generate_rhd(n)
    L = int(math.log2(n))
    sizes = []
    for rnd in s.rounds:
        per_dst = {}
        for t in rnd:
            per_dst.setdefault(t.dst, set()).add(t.src)
            assert t.src ^ t.dst == (t.src ^ t.dst) & -(t.src ^ t.dst)   # partners differ in one bit
        assert sorted(per_dst) == list(range(n)) and all(len(v) == 1 for v in per_dst.values())
        sizes.append(len(rnd) // n)
    assert sizes[:L] == [n >> (t + 1) for t in range(L)]
    assert sizes[L:] == sizes[:L][::-1]
    assert all(t.kind == S.REDUCE for r in s.rounds[:L] for t in r)
    assert all(t.kind == S.REPLACE for r in s.rounds[L:] for t in r)
    # round k of the ReduceScatter pairs ranks differing in bit k
    for k in range(L):
        assert all(t.src ^ t.dst == 1 << k for t in s.rounds[k])
        assert all(t.src ^ t.dst == 1 << (L - 1 - k) for t in s.rounds[L + k])
    # after the ReduceScatter every rank holds exactly one chunk fully reduced, all different
    st = S.initial_state_uniform(n, n)
    for rnd in s.rounds[:L]:
        st = S.apply_round(st, rnd, n, one_chunk=False)
    full = frozenset(range(n))
    owned = [[c for c in range(n) if st[(i, c)] == full] for i in range(n)]
    assert all(len(o) == 1 for o in owned) and sorted(o[0] for o in owned) == list(range(n))


def test_rhd_spec_examples():
    """n=8 -> 6 rounds; n=2 -> 2 rounds of one chunk each; n=4 ->
    beta = 1/2 + 1/4 + 1/4 + 1/2 = 3/2."""
    assert S.generate_rhd(8).num_rounds == 6
    s2 = S.generate_rhd(2)
    assert s2.num_rounds == 2 and all(len(r) == 2 for r in s2.rounds)
    assert S.verify_schedule(S.generate_rhd(4)).beta_coefficient == Fraction(3, 2)


def test_broadcast_spec_examples():
    """n=8 -> 3 rounds, beta 3; n=2 -> 1 round; n=16 -> 4 rounds,
    verifier-valid from the AllReduce-precondition state.  S:289: in round k
    the holders send to the lowest-index non-holders, pairing in index order."""
    r8 = S.verify_schedule(S.generate_broadcast(8))
    assert S.generate_broadcast(8).num_rounds == 3 and r8.beta_coefficient == 3
    assert S.generate_broadcast(2).num_rounds == 1
    assert S.generate_broadcast(16).num_rounds == 4 and S.verify_schedule(S.generate_broadcast(16)).valid
    for rnd in S.generate_broadcast(16).rounds[1:]:
        pairs = sorted({(t.src, t.dst) for t in rnd})
        srcs, dsts = [p[0] for p in pairs], [p[1] for p in pairs]
        assert srcs == sorted(srcs) and dsts == sorted(dsts)


def test_rhd_rejects_non_power_of_two():
    with pytest.raises(S.ScheduleError):
        S.generate_rhd(6)


# ---------------------------------------------------------------- RHD numerics
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("count", [0, 1, 5, 31, 333])
def test_rhd_int32_brute_force(n, count):
    xs = make_inputs(n, count, "int32", config=95)
    want = _wrap_sum(xs)
    assert all(np.array_equal(o, want) for o in N.rhd_allreduce(xs, "int32"))
    assert np.array_equal(N.plain_rhd_allreduce(xs, "int32"), want)


@pytest.mark.parametrize("dtype", ("float32", "bfloat16"))
@pytest.mark.parametrize("n", [2, 4, 8])
def test_rhd_integer_valued_exact(dtype, n):
    xs = make_inputs(n, 517, dtype, pattern="intval")
    want = np.sum(np.stack(make_inputs(n, 517, "int32", pattern="intval")).astype(np.int64), axis=0)
    for o in N.rhd_allreduce(xs, dtype) + [N.plain_rhd_allreduce(xs, dtype)]:
        v = N.bf16_to_f32(o) if dtype == "bfloat16" else o
        assert np.array_equal(v.astype(np.int64), want)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("n", [2, 4, 8])
def test_rhd_bitmask(dtype, n):
    for o in N.rhd_allreduce(make_inputs(n, 203, dtype, pattern="bitmask"), dtype):
        v = N.bf16_to_f32(o) if dtype == "bfloat16" else o
        assert np.all(v == 2 ** n - 1)


@pytest.mark.parametrize("dtype", DT)
def test_rhd_n2_textbook(dtype):
    """n = 2: one exchange of halves + one copy = x0 + x1 by torch's own add."""
    xs = make_inputs(2, 1001, dtype, config=96)
    if dtype == "bfloat16":
        t = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16) for x in xs]
        want = (t[0] + t[1]).view(torch.int16).numpy().view(np.uint16)
    else:
        want = (torch.from_numpy(xs[0]) + torch.from_numpy(xs[1])).numpy()
    for o in N.rhd_allreduce(xs, dtype):
        assert np.array_equal(_bits(o), _bits(want))


@pytest.mark.parametrize("dtype", ("float32", "bfloat16"))
@pytest.mark.parametrize("n", [4, 8])
@pytest.mark.parametrize("count", [4099, 10 ** 5 + 3])
def test_rhd_replay_equals_butterfly_definition(dtype, n, count):
    """The chunked round replay equals the elementwise butterfly, bit for bit,
    on every rank, and stays within the pairwise-summation bound: each element
    passes log n adds, so |err| <= (log n) u sum|x| (+ the bf16 rounding)."""
    xs = make_inputs(n, count, dtype, config=97)
    want = N.plain_rhd_allreduce(xs, dtype)
    outs = N.rhd_allreduce(xs, dtype)
    assert all(np.array_equal(_bits(o), _bits(want)) for o in outs)
    exact, absum = N.exact_sum_f64(xs, dtype)
    got = N.bf16_to_f32(want).astype(np.float64) if dtype == "bfloat16" else want.astype(np.float64)
    u = 2.0 ** -24 if dtype == "float32" else 2.0 ** -8
    L = int(math.log2(n))
    assert np.all(np.abs(got - exact) <= L * u * absum * (1 + 1e-6) + 1e-30)
    # the tree order differs from the Ring's rotation order on some elements
    if dtype == "float32":
        ring = N.plain_ring_allreduce(xs, dtype)
        assert not np.array_equal(_bits(ring), _bits(want))


# ---------------------------------------------------------------- Broadcast schedule
@pytest.mark.parametrize("n", [2, 4, 6, 8, 10, 16, 32])
def test_broadcast_rounds_beta(n):
    """log n rounds of s bytes each (T_Bcast = log n alpha + log n s
    beta); ceil(log2 n) for even n that is not a power of two."""
    s = S.generate_broadcast(n)
    rep = S.verify_schedule(s)
    assert rep.valid, rep.violations[:3]
    L = math.ceil(math.log2(n))
    assert s.num_rounds == L
    assert rep.beta_coefficient == L
    if n & (n - 1) == 0:
        assert C.t_broadcast(n, 0.0, 1.0, 0.0) == s.num_rounds
        assert C.t_broadcast(n, 1.0, 0.0, 1.0) == float(rep.beta_coefficient)


@pytest.mark.parametrize("n", [2, 4, 8])
def test_broadcast_structure(n):
    """Round 0: the straggler exchanges its entire buffer with one rank
    (both Reduce); afterwards only copies, and the holders of the full sum
    double every round."""
    s = S.generate_broadcast(n)
    sigma = n - 1
    r0 = s.rounds[0]
    assert {(t.src, t.dst) for t in r0} == {(sigma, 0), (0, sigma)}
    assert all(t.kind == S.REDUCE for t in r0) and len(r0) == 2 * (n - 1)
    holders = {0, sigma}
    for rnd in s.rounds[1:]:
        assert all(t.kind == S.REPLACE and t.src in holders and t.dst not in holders for t in rnd)
        new = {t.dst for t in rnd}
        assert len(new) == min(len(holders), n - len(holders))
        holders |= new
    assert holders == set(range(n))


def test_broadcast_golden_n8():
    """Tie-break of the reading (holders ascending zipped with non-holders)."""
    s = S.generate_broadcast(8)
    pairs = [sorted({(t.src, t.dst) for t in r}) for r in s.rounds[1:]]
    assert pairs == [[(0, 1), (7, 2)], [(0, 3), (1, 4), (2, 5), (7, 6)]]


# ---------------------------------------------------------------- Broadcast numerics
@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_broadcast_equals_plain_definition(dtype, n):
    """Every chunk is fully reduced once (partial + x_sigma) and only copied
    afterwards: the result is the plain definition of c.1, on every rank."""
    xs = make_inputs(n, 1000 + 7 * n, dtype, config=98)
    for sig in range(n):
        want = N.plain_allreduce(xs, sig, dtype)
        for o in N.broadcast_allreduce(xs, sig, dtype):
            assert np.array_equal(_bits(o), _bits(want))


@pytest.mark.parametrize("n", [2, 4, 8])
def test_broadcast_int32_brute_force(n):
    xs = make_inputs(n, 257, "int32", config=99)
    want = _wrap_sum(xs)
    for sig in range(n):
        assert all(np.array_equal(o, want) for o in N.broadcast_allreduce(xs, sig, "int32"))
