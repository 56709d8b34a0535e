"""Pins for oracle/schedule.py against what PAPER.md fixes (CPU only).

The holder-set bookkeeping below is re-derived in this file from the transfer
list, independently of the generator's internal dictionary A.
"""
import math
import os
import time
from fractions import Fraction

import pytest

from oracle import schedule as S

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
POW2 = [2, 4, 8, 16, 32, 64, 128, 256]


def _load_golden(name):
    rounds = {}
    for line in open(os.path.join(GOLDEN, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        r, src, dst, c, kind = line.split()
        rounds.setdefault(int(r), set()).add((int(src), int(dst), int(c), kind))
    return [rounds[r] for r in sorted(rounds)]


def _as_sets(s):
    return [{(t.src, t.dst, t.chunk, t.kind) for t in rnd} for rnd in s.rounds]


# ---------------------------------------------------------------- Theorem 1
@pytest.mark.parametrize("n", POW2)
def test_theorem1_round_count(n):
    """P:290 Theorem 1: n + log n - 2 rounds."""
    s = S.generate_stragglar(n)
    assert s.num_rounds == n + int(math.log2(n)) - 2


@pytest.mark.parametrize("n", POW2)
def test_verifier_valid_and_table1_beta(n):
    """P:202 postcondition (all ranks hold the full sum) and Table 1:
    beta coefficient (n + log n - 2)/(n - 1)."""
    rep = S.verify_schedule(S.generate_stragglar(n))
    assert rep.valid, rep.violations[:5]
    assert rep.beta_coefficient == Fraction(n + int(math.log2(n)) - 2, n - 1)


def test_generation_time_n256():
    """256 GPUs in 1.04 s (paper's machine).  Bound loosely."""
    t = time.perf_counter()
    S.generate_stragglar(256)
    assert time.perf_counter() - t < 10.0


@pytest.mark.parametrize("n", [3, 6, 12, 1, 0])
def test_non_power_of_two_rejected(n):
    """P:156 input n = 2^k; P:461-462 odd n unsupported."""
    with pytest.raises(S.ScheduleError):
        S.generate_stragglar(n)


# ---------------------------------------------------------------- structure
@pytest.mark.parametrize("n", POW2[:6])
def test_round_structure(n):
    """round r < n-1 pairs rank r with sigma, exchanging c_r, both
    reducing.  P:149-150 single port: each rank sends <= 1 and
    receives <= 1 chunk per round and has one partner.  Every transfer
    is one chunk.  No other transfer is a Reduce (the rest only
    propagate fully reduced chunks)."""
    s = S.generate_stragglar(n)
    sigma = n - 1
    for r, rnd in enumerate(s.rounds):
        red = sorted((t.src, t.dst, t.chunk) for t in rnd if t.kind == S.REDUCE)
        if r < n - 1:
            assert red == sorted([(r, sigma, r), (sigma, r, r)])
        else:
            assert red == []
        partner = {}
        for t in rnd:
            assert partner.setdefault(t.src, t.dst) == t.dst
            assert partner.setdefault(t.dst, t.src) == t.src
        srcs = [t.src for t in rnd]
        dsts = [t.dst for t in rnd]
        assert len(srcs) == len(set(srcs)) and len(dsts) == len(set(dsts))


def _holders_trace(s):
    """Re-derive, from the transfer list alone, which ranks hold each chunk
    fully reduced before every round.  Returns list over r of dict c -> set."""
    n = s.n
    sigma = n - 1
    full = {c: set() for c in range(n - 1)}
    out = [{c: set(v) for c, v in full.items()}]
    for r, rnd in enumerate(s.rounds):
        new = {c: set(v) for c, v in full.items()}
        for t in rnd:
            if t.kind == S.REDUCE:
                # the sigma pairing fully reduces c_r on both ends
                assert t.chunk == r and {t.src, t.dst} == {r, sigma}
                new[t.chunk] |= {r, sigma}
            else:
                # only fully reduced chunks propagate; snapshot: held before the round
                assert t.src in full[t.chunk], f"round {r}: {t} sends a chunk it does not hold fully reduced"
                assert t.dst not in full[t.chunk], f"round {r}: {t} is redundant"
                new[t.chunk].add(t.dst)
        full = new
        out.append({c: set(v) for c, v in full.items()})
    return out


@pytest.mark.parametrize("n", POW2[:7])
def test_lemma1_phase1_counts(n):
    """P:537 Lemma 1: before round log n every non-straggler holds exactly one
    active chunk and |A[c_j]| = 2^(log n - 1 - j), j = 0..log n - 1."""
    L = int(math.log2(n))
    if n == 2:
        pytest.skip("log n = 1: the claim is about round 1, after the last round")
    s = S.generate_stragglar(n)
    before_L = _holders_trace(s)[L]
    ns = set(range(n - 1))
    counts = {}
    for j in range(L):
        A_j = before_L[j] & ns
        assert len(A_j) == 2 ** (L - 1 - j)
        for g in A_j:
            counts[g] = counts.get(g, 0) + 1
    assert set(counts) == ns and all(v == 1 for v in counts.values())


@pytest.mark.parametrize("n", POW2[1:7])
def test_invariant_I_r(n):
    """P:589-595 I(r) before each round r in [log n, n-2]: |A[c_j]| = 2^(r-j-1)
    for j = r-log n .. r-1; P_r = A[c_{r-log n}], |P_r| = n/2, r in P_r;
    |Q_r| = n/2 - 1; active holder sets pairwise disjoint."""
    L = int(math.log2(n))
    s = S.generate_stragglar(n)
    trace = _holders_trace(s)
    ns = set(range(n - 1))
    for r in range(L, n - 1):
        before = trace[r]
        A = {j: before[j] & ns for j in range(r - L, r)}
        for j, hs in A.items():
            assert len(hs) == 2 ** (r - j - 1), (r, j, hs)
        P = A[r - L]
        Q = set().union(*(A[r - j] for j in range(1, L)))
        assert len(P) == n // 2 and r in P
        assert len(Q) == n // 2 - 1
        assert sum(len(h) for h in A.values()) == len(set().union(*A.values()))


@pytest.mark.parametrize("n", POW2[:7])
def test_lemma2_and_remark1_expiry(n):
    """P:577 Lemma 2: c_r (r < n-2) is held by every rank right after round
    r + log n and not before (it doubles from one holder); P:658 Remark
    1 / Thm 1 proof P:672-673: the final chunk c_{n-2} after round n-3+log n."""
    L = int(math.log2(n))
    s = S.generate_stragglar(n)
    trace = _holders_trace(s)
    everyone = set(range(n))
    for c in range(n - 1):
        due = c + L if c < n - 2 else n - 3 + L
        due = min(due, s.num_rounds - 1)
        assert trace[due + 1][c] == everyone, (c, due)
        if c < n - 2 and n > 2:
            assert trace[due][c] != everyone


# ---------------------------------------------------------------- goldens
def test_golden_n2():
    assert _as_sets(S.generate_stragglar(2)) == _load_golden("stragglar_n2.txt")


def test_golden_n4():
    assert _as_sets(S.generate_stragglar(4)) == _load_golden("stragglar_n4.txt")


def test_golden_n8_printed_facts():
    s = S.generate_stragglar(8)
    sets = _as_sets(s)
    for line in open(os.path.join(GOLDEN, "stragglar_n8_partial.txt")):
        f = line.split()
        if not f or f[0].startswith("#"):
            continue
        if f[0] == "transfer":
            r, a, b, c, kind = int(f[1]), int(f[2]), int(f[3]), int(f[4]), f[5]
            assert (a, b, c, kind) in sets[r]
        elif f[0] == "round_size":
            assert len(sets[int(f[1])]) == int(f[2])
        elif f[0] == "not_paired":
            r, a, b = int(f[1]), int(f[2]), int(f[3])
            assert not any({t[0], t[1]} == {a, b} for t in sets[r])


# ---------------------------------------------------------------- verifier pins
def test_verifier_double_count():
    """Reduce of {0,1} into {1,2} is a double count."""
    st = {(0, 0): frozenset({0, 1}), (1, 0): frozenset({1, 2})}
    v = []
    S.apply_round(st, [S.Transfer(0, 1, 0, S.REDUCE)], 3, 0, v)
    assert any("double count" in m for _, m in v)


def test_verifier_port_violation():
    """a rank in two matchings is a port violation."""
    st = S.initial_state_uniform(4, 4)
    v = []
    S.apply_round(st, [S.Transfer(0, 2, 0, S.REPLACE), S.Transfer(2, 1, 1, S.REPLACE)], 4, 0, v)
    assert any("port violation" in m for _, m in v)


def test_verifier_regression():
    """Replace with a non-superset is a regression."""
    st = {(0, 0): frozenset({0}), (1, 0): frozenset({1, 2})}
    v = []
    S.apply_round(st, [S.Transfer(0, 1, 0, S.REPLACE)], 3, 0, v)
    assert any("regression" in m for _, m in v)


def test_verifier_round0_n4():
    """after round 0 at n=4, ranks 0 and 3 hold c_0 with contributors {0,1,2,3}."""
    st = S.apply_round(S.initial_state_stragglar(4), S.generate_stragglar(4).rounds[0], 4)
    assert st[(0, 0)] == frozenset(range(4)) == st[(3, 0)]


def test_initial_state_examples():
    """S:68-70 precondition examples."""
    st4 = S.initial_state_stragglar(4)
    assert st4[(0, 0)] == {0, 1, 2} and all(st4[(3, c)] == {3} for c in range(3))
    st2 = S.initial_state_stragglar(2)
    assert st2[(0, 0)] == {0} and st2[(1, 0)] == {1}
    st8 = S.initial_state_stragglar(8)
    assert st8[(5, 5)] == set(range(7)) and st8[(5, 2)] == {5}


def test_verifier_truncated_invalid():
    """the n=4 schedule with round 3 deleted is invalid (postcondition)."""
    s = S.generate_stragglar(4)
    s.rounds = s.rounds[:3]
    rep = S.verify_schedule(s)
    assert not rep.valid and any("postcondition" in m for _, m in rep.violations)


# ---------------------------------------------------------------- ring baseline
@pytest.mark.parametrize("n", [2, 3, 4, 6, 8, 16])
def test_ring_rounds_and_beta(n):
    """P:360-361 / Table 1: 2(n-1) rounds, beta 2(n-1)/n; S:257 pattern."""
    s = S.generate_ring(n)
    rep = S.verify_schedule(s)
    assert rep.valid, rep.violations[:3]
    assert s.num_rounds == 2 * (n - 1)
    assert rep.beta_coefficient == Fraction(2 * (n - 1), n)
    for t in range(n - 1):
        assert {(x.src, x.dst, x.chunk) for x in s.rounds[t]} == {(i, (i + 1) % n, (i - t) % n) for i in range(n)}
