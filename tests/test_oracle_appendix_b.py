"""Pins for the Appendix-B generator (even, non-power-of-2 n)."""
import itertools
import math
import random
from fractions import Fraction

import numpy as np
import pytest

from oracle import numerics as N
from oracle import schedule as S
from paper_2505_23523_b200.inputs import make_inputs


def dp_max_weight(vertices, weight):
    """Independent formulation: DP over vertex subsets (max weight of a
    matching inside `mask`), not the generator's search."""
    vs = sorted(vertices)
    k = len(vs)
    best = {0: 0}
    for mask in range(1, 1 << k):
        i = (mask & -mask).bit_length() - 1
        rest = mask & ~(1 << i)
        b = best[rest]                        # vertex i unmatched
        for j in range(i + 1, k):
            if rest >> j & 1:
                w = weight(vs[i], vs[j])
                if w > 0:
                    b = max(b, w + best[rest & ~(1 << j)])
        best[mask] = b
    return best[(1 << k) - 1]


def test_matching_spec_examples():
    """empty graph -> weight 0; triangle (a-b:2, b-c:2, a-c:1) -> 2."""
    assert S.max_weight_matching([], lambda u, v: 1)[0] == 0
    w = {(0, 1): 2, (1, 2): 2, (0, 2): 1}
    tot, m = S.max_weight_matching([0, 1, 2], lambda u, v: w.get((min(u, v), max(u, v)), 0))
    assert tot == 2 and len(m) == 1


def test_matching_equals_dp_on_random_graphs():
    """equals an exhaustive optimum on >= 500 random graphs of <= 10
    vertices with weights in {0, 1, 2} (here: the subset DP)."""
    rnd = random.Random(2505_23523)
    for _ in range(500):
        k = rnd.randint(0, 9)
        w = {(i, j): rnd.choice([0, 1, 2]) for i in range(k) for j in range(i + 1, k)}
        f = lambda u, v: w[(min(u, v), max(u, v))]  # noqa: E731
        tot, m = S.max_weight_matching(list(range(k)), f)
        assert tot == dp_max_weight(list(range(k)), f)
        used = [x for e in m for x in e]
        assert len(used) == len(set(used)) and sum(f(u, v) for u, v in m) == tot


@pytest.mark.parametrize("n", [6, 10, 12])
def test_even_schedule_valid_and_beats_ring(n):
    """verifier-valid; rounds/(n-1) < 2(n-1)/n (beats Ring's beta,
    the paper's claim P:689); hard bound rounds < 2(n-1); straggler pairing
    (r, sigma) exchanges c_r in every round r < n-1."""
    s = S.generate_stragglar_even(n)
    rep = S.verify_schedule(s)
    assert rep.valid, rep.violations[:3]
    assert rep.beta_coefficient == Fraction(s.num_rounds, n - 1)
    assert rep.beta_coefficient < Fraction(2 * (n - 1), n)
    assert s.num_rounds < 2 * (n - 1)
    for r in range(n - 1):
        red = {(t.src, t.dst, t.chunk) for t in s.rounds[r] if t.kind == S.REDUCE}
        assert red == {(r, n - 1, r), (n - 1, r, r)}


def test_even_round_count_recorded():
    """'~ n + 2 log n - 2 rounds in practice' (recorded, not a bound)."""
    s = S.generate_stragglar_even(6)
    assert s.num_rounds <= math.ceil(6 + 2 * math.log2(6) - 2)


@pytest.mark.parametrize("n", [3, 5, 4, 8])
def test_even_rejects(n):
    with pytest.raises(S.ScheduleError):
        S.generate_stragglar_even(n)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_even_numerics(dtype):
    """n = 6: the replay equals the plain definition bitwise on every rank, and
    int32 equals the integer brute force, for every straggler rank."""
    n = 6
    xs = make_inputs(n, 3001, dtype, config=98)
    for sig in range(n):
        want = N.plain_allreduce(xs, sig, dtype)
        for o in N.stragglar_allreduce(xs, sig, dtype):
            assert np.array_equal(o.view(np.uint8), want.view(np.uint8))
    if dtype == "int32":
        exact = sum(x.astype(np.int64) for x in xs)
        assert np.array_equal(want, ((exact + 2 ** 31) % 2 ** 32 - 2 ** 31).astype(np.int32))
