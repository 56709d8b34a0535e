"""Schedules and the contributor-set verifier — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Everything here is written in *logical* ranks: the straggler is sigma = n-1
("Without loss of generality, we assume rank n-1 is the persistent straggler",
P:200 §3.1).  Mapping to physical ranks is done in ``numerics.py``.

Algorithm 1 is garbled in several places.  The readings taken here
are SURVEY.md §8(c).3 rows 1-11 and are listed again in DESIGN.md:

  (1) loop bound: r in [0, n+L-3], i.e. exactly n+L-2 rounds (Thm 1).
  (2) the P/Q matching of line 182 runs only for r >= L.
  (3) Phase 1 "any rank g > 2(log n - 1) without a chunk": the
      mandated send first, then the other holders in ascending order each send
      to the lowest-index available chunk-free non-straggler g > 2(L-1).
  (4) critical window = [r+1, r+L] (text).
  (5) window partner rule from the text: g in Q pairs with
      the lowest-index available P rank outside the window, which sends
      c_{r-L}; g in P pairs with a Q rank outside the window holding the oldest
      active chunk c_j that g lacks with j <= g-L.
  (6) line 178 roles: the partner sends g the chunk g lacks, g sends its own.
  (7) Remark 1: for r >= n-1 sigma is appended to Q
      (sorted last) and zipped with P; it sends only c_{n-2}; the send *to*
      sigma is redundant and skipped.
  (8) "c_{n-1}" at P:294 is a typo for c_{n-2}.
  (9) "exactly one matching per round" is read as "at most one".
  (10) the sigma pairing is a bidirectional exchange, both sides Reduce (P:164,
      P:206).
  (11) snapshot rounds: a chunk received in round r is sendable from r+1 on
      ("c_r can only be sent ... from round r+1 onwards").
"""
from __future__ import annotations

from dataclasses import dataclass, field
from fractions import Fraction
from typing import Dict, FrozenSet, List, Optional, Tuple

REDUCE = "reduce"
REPLACE = "replace"


@dataclass(frozen=True)
class Transfer:
    """One directed chunk transfer inside a round.

    kind == "reduce": the receiver adds the payload into its copy
    kind == "replace": the receiver overwrites its copy with the payload
    """

    src: int
    dst: int
    chunk: int
    kind: str


@dataclass
class Schedule:
    """Ordered rounds of transfers; ranks are logical."""

    algorithm: str
    n: int
    straggler: int
    num_chunks: int
    rounds: List[List[Transfer]] = field(default_factory=list)

    @property
    def num_rounds(self) -> int:
        return len(self.rounds)


class ScheduleError(Exception):
    pass


def log2_exact(n: int) -> int:
    if n < 2 or n & (n - 1):
        raise ScheduleError(f"n={n} is not a power of two >= 2 (Alg. 1 input, P:156)")
    return n.bit_length() - 1


# --------------------------------------------------------------------------
# Algorithm 1 — StragglAR schedule generator (§3.1)
# --------------------------------------------------------------------------
def generate_stragglar(n: int) -> Schedule:
    """Algorithm 1 for power-of-2 n with sigma = n-1.

    Returns a schedule of n + log2(n) - 2 rounds (Thm 1).  The
    straggler pairing of round r < n-1 is a two-way Reduce of c_r.
    """
    L = log2_exact(n)
    sigma = n - 1
    R = n + L - 2                                    # reading (1)
    # A: active chunk -> set of non-straggler holders
    A: Dict[int, set] = {}
    sched = Schedule("stragglar", n, sigma, n - 1)

    for r in range(R):
        avail = set(range(n - 1))                    # non-stragglers not yet matched
        sigma_free = True
        round_tx: List[Transfer] = []

        def active_of(h: int) -> Optional[int]:
            for c, hs in A.items():
                if h in hs:
                    return c
            return None

        # rank r <-> sigma exchange c_r, both fully reduce it
        if r < n - 1:
            round_tx.append(Transfer(r, sigma, r, REDUCE))
            round_tx.append(Transfer(sigma, r, r, REDUCE))
            avail.discard(r)
            sigma_free = False

        if 0 < r < L:
            # Phase 1
            src, dst, c = r - 1, r - 1 + L, r - 1
            round_tx.append(Transfer(src, dst, c, REPLACE))
            avail.discard(src)
            avail.discard(dst)
            receivers = {dst}
            # reading (3): other holders, ascending, to the lowest chunk-free g > 2(L-1)
            for h in sorted(avail):
                ch = active_of(h)
                if ch is None:
                    continue
                cands = [g for g in sorted(avail)
                         if g > 2 * (L - 1) and active_of(g) is None and g not in receivers and g != h]
                if not cands:
                    raise ScheduleError(f"round {r}: no chunk-free receiver for rank {h} (contradicts Lemma 1)")
                g = cands[0]
                round_tx.append(Transfer(h, g, ch, REPLACE))
                avail.discard(h)
                avail.discard(g)
                receivers.add(g)
        elif r >= L:
            # Phase 2
            old = r - L                              # c_{r-log n}, the oldest active chunk
            P = sorted(h for h in A.get(old, ()) if h in avail)
            Q = sorted(h for c, hs in A.items() if c != old for h in hs if h in avail)
            sigma_in_Q = r >= n - 1 and sigma_free   # reading (7), Remark 1
            window = set(range(r + 1, r + L + 1))    # reading (4)
            matched: set = set()

            def exchange(p: int, q: int) -> None:
                """p in P sends c_old to q; q sends its active chunk to p."""
                round_tx.append(Transfer(p, q, old, REPLACE))
                round_tx.append(Transfer(q, p, active_of(q), REPLACE))
                matched.add(p)
                matched.add(q)

            # critical window first, reading (5)/(6)
            for g in range(r + 1, r + L + 1):
                if g >= n - 1 or g in matched or g not in avail:
                    continue
                if g in Q:
                    partners = [p for p in P if p not in matched and p not in window]
                    if not partners:
                        raise ScheduleError(f"round {r}: no partner for window rank {g} in Q")
                    exchange(partners[0], g)
                elif g in P:
                    found = None
                    for j in sorted(c for c in A if c != old and c <= g - L):
                        if g in A[j]:
                            continue
                        hs = [h for h in sorted(A[j]) if h in Q and h not in matched and h not in window]
                        if hs:
                            found = hs[0]
                            break
                    if found is None:
                        raise ScheduleError(f"round {r}: no admissible partner for window rank {g} in P")
                    exchange(g, found)
            # line 182: zip remaining P with remaining Q (sigma last)
            Pr = [p for p in P if p not in matched]
            Qr = [q for q in Q if q not in matched]
            if sigma_in_Q:
                Qr.append(sigma)
            if len(Pr) != len(Qr):
                raise ScheduleError(f"round {r}: |P|={len(Pr)} != |Q|={len(Qr)} after the window")
            for p, q in zip(Pr, Qr):
                if q == sigma:
                    # Remark 1: sigma sends only c_{n-2}; p -> sigma would be redundant
                    round_tx.append(Transfer(sigma, p, n - 2, REPLACE))
                    matched.add(p)
                else:
                    exchange(p, q)

        sched.rounds.append(round_tx)

        # bookkeeping, snapshot semantics (reading 11)
        for t in round_tx:
            if t.kind == REPLACE and t.chunk in A and t.dst != sigma:
                A[t.chunk].add(t.dst)
        if r >= L:
            A.pop(r - L, None)                       # P:187 c_{r-log n} fully propagated
        if r < n - 1:
            A[r] = {r}                               # P:191 newly active chunk
    return sched


# --------------------------------------------------------------------------
# Appendix B: even, non-power-of-2 n
# --------------------------------------------------------------------------
def max_weight_matching(vertices: List[int], weight) -> Tuple[int, List[Tuple[int, int]]]:
    """Maximum-weight matching by exhaustive search (exact; n <= 8 here).

    P:684 names Edmonds' algorithm; for a handful of vertices enumerating every
    matching is the same optimum with no room for error.  Enumeration order
    (the tie-break between equal-weight optima): take the lowest unmatched
    vertex u, try partners v > u in ascending order, then u unmatched; the
    first maximum found wins.
    """
    best = [-1, []]

    def rec(rest: List[int], cur: List[Tuple[int, int]], w: int) -> None:
        if not rest:
            if w > best[0]:
                best[0], best[1] = w, list(cur)
            return
        u, tail = rest[0], rest[1:]
        for i, v in enumerate(tail):
            wt = weight(u, v)
            if wt > 0:
                cur.append((u, v))
                rec(tail[:i] + tail[i + 1:], cur, w + wt)
                cur.pop()
        rec(tail, cur, w)

    rec(sorted(vertices), [], 0)
    return best[0], best[1]


def generate_stragglar_even(n: int, max_rounds: Optional[int] = None) -> Schedule:
    """Appendix B for even n that is not a power of two.

    Readings (DESIGN.md "Readings" 18-21, after SPEC S:216-243):
    * Phase A and the straggler pairing are kept: round r < n-1 exchanges c_r
      between rank r and sigma, both reducing (P:163-164 carries over).
    * Every other rank (and sigma once it is free, r >= n-1) is a vertex; u
      "needs" chunk c from v iff v holds c fully reduced and u does not (only
      fully reduced chunks propagate).  Edge weight 2 if each needs
      something from the other, 1 if only one direction.
    * A maximum-weight matching is taken per round; each matched rank sends the
      oldest (lowest-index) chunk its partner needs.
    * Rounds continue until every rank holds every chunk.
    """
    if n < 4 or n % 2 or not (n & (n - 1)):
        raise ScheduleError(f"n={n}: Appendix B covers even n that are not powers of two")
    sigma = n - 1
    full = {h: set() for h in range(n)}          # fully reduced chunks held
    sched = Schedule("stragglar", n, sigma, n - 1)
    limit = max_rounds if max_rounds is not None else 4 * n
    r = 0
    while any(len(full[h]) < n - 1 for h in range(n)):
        if r >= limit:
            raise ScheduleError(f"n={n}: no completion within {limit} rounds")
        tx: List[Transfer] = []
        busy = set()
        if r < n - 1:
            tx += [Transfer(r, sigma, r, REDUCE), Transfer(sigma, r, r, REDUCE)]
            busy = {r, sigma}
        verts = [h for h in range(n) if h not in busy]

        def needs(u: int, v: int) -> List[int]:
            return sorted(full[v] - full[u])

        def weight(u: int, v: int) -> int:
            return (1 if needs(u, v) else 0) + (1 if needs(v, u) else 0)

        _, matching = max_weight_matching(verts, weight)
        for u, v in matching:
            for a, b in ((u, v), (v, u)):
                nd = needs(b, a)                  # what b needs from a
                if nd:
                    tx.append(Transfer(a, b, nd[0], REPLACE))
        sched.rounds.append(tx)
        new = {h: set(c) for h, c in full.items()}
        for t in tx:
            new[t.dst].add(t.chunk)
        if r < n - 1:
            new[r].add(r)
            new[sigma].add(r)
        full = new
        r += 1
    return sched


def generate(n: int) -> Schedule:
    """Algorithm 1 for powers of two, Appendix B for other even n."""
    if n >= 2 and not (n & (n - 1)):
        return generate_stragglar(n)
    return generate_stragglar_even(n)


# --------------------------------------------------------------------------
# Baseline: Ring; S:257 fixes the transfer pattern
# --------------------------------------------------------------------------
def generate_ring(n: int) -> Schedule:
    """Ring AllReduce: n chunks, 2(n-1) rounds.

    Rounds 0..n-2: rank i sends chunk (i - t) mod n to rank i+1, which adds
    its own (Reduce).  Rounds n-1..2n-3: all-gather copies (Replace).  Ring
    direction ascending.
    """
    if n < 2:
        raise ScheduleError("ring needs n >= 2")
    s = Schedule("ring", n, n - 1, n)
    for t in range(n - 1):
        s.rounds.append([Transfer(i, (i + 1) % n, (i - t) % n, REDUCE) for i in range(n)])
    for u in range(n - 1):
        # after RS, rank i holds the full chunk (i+1) mod n; forward what you hold
        s.rounds.append([Transfer(i, (i + 1) % n, (i + 1 - u) % n, REPLACE) for i in range(n)])
    return s


# --------------------------------------------------------------------------
# Baseline: recursive halving/doubling ("Butterfly")
# --------------------------------------------------------------------------
def generate_rhd(n: int) -> Schedule:
    """RHD AllReduce on n chunks (one per rank), 2 log n rounds.

    P:364-365: "the buffer is first divided in 1/2 with one partner, then in
    1/4 with another partner, etc. to achieve a ReduceScatter.  Then, a
    mirror-image AllGather completes."  The partner order is not stated; the
    reading is SPEC's ("round k of phase 1 pairs ranks differing in
    bit k"): in ReduceScatter round t (t = 0..L-1) rank i pairs with
    i XOR 2^t; both hold the same block of n/2^t chunks; i keeps the lower half
    if bit t of i is 0, else the upper half, and receives the partner's copy of
    the half it keeps (Reduce).  After L rounds rank i holds one chunk fully
    reduced (chunk bitreverse(i)).  AllGather round L+u (u = 0..L-1) mirrors
    ReduceScatter round L-1-u: partners exchange their fully reduced blocks of
    2^u chunks (Replace).
    """
    L = log2_exact(n)
    s = Schedule("rhd", n, -1, n)
    blocks = {i: (0, n) for i in range(n)}            # (first chunk, #chunks) each rank works on
    for t in range(L):
        d = 1 << t
        rnd = []
        new = {}
        for i in range(n):
            lo, m = blocks[i]
            keep = lo if (i & d) == 0 else lo + m // 2
            new[i] = (keep, m // 2)
            rnd += [Transfer(i ^ d, i, c, REDUCE) for c in range(keep, keep + m // 2)]
        blocks = new
        s.rounds.append(rnd)
    for u in range(L):
        d = 1 << (L - 1 - u)
        rnd = []
        new = {}
        for i in range(n):
            lo, m = blocks[i]                         # i's fully reduced block
            p = i ^ d
            plo, _ = blocks[p]
            rnd += [Transfer(p, i, c, REPLACE) for c in range(plo, plo + m)]
            new[i] = (min(lo, plo), 2 * m)
        blocks = new
        s.rounds.append(rnd)
    return s


# --------------------------------------------------------------------------
# Baseline: straggler-aware Broadcast
# --------------------------------------------------------------------------
def generate_broadcast(n: int) -> Schedule:
    """Broadcast AllReduce, logical ranks (straggler sigma = n-1), n-1 chunks.

    P:369-372: the non-stragglers complete an AllReduce during the delay
    (the precondition, ``initial_state_broadcast``); "the straggler ...
    exchanges its entire buffer with any other rank to fully reduce the
    entire buffer and then initiates a broadcast with log n rounds and s bytes
    per round".  Readings: the exchange partner is logical rank 0, and the
    exchange is round 0 of the log n (T_Bcast = log n alpha + log n s beta,
    P:373, counts log n messages of s bytes).  Round r >= 1: the ranks holding
    the full sum, ascending, are zipped with the ranks that do not, ascending;
    each pair copies the whole buffer (every chunk, Replace).  Holders double
    per round: 2, 4, ..., n after ceil(log2 n) rounds.
    """
    if n < 2:
        raise ScheduleError("broadcast needs n >= 2")
    sigma = n - 1
    s = Schedule("broadcast", n, sigma, n - 1)
    s.rounds.append([Transfer(sigma, 0, c, REDUCE) for c in range(n - 1)] +
                    [Transfer(0, sigma, c, REDUCE) for c in range(n - 1)])
    holders = {0, sigma}
    while len(holders) < n:
        H = sorted(holders)
        Q = [q for q in range(n) if q not in holders]
        pairs = list(zip(H, Q))
        s.rounds.append([Transfer(h, q, c, REPLACE) for h, q in pairs for c in range(n - 1)])
        holders |= {q for _, q in pairs}
    return s


# --------------------------------------------------------------------------
# Contributor-set verifier
# --------------------------------------------------------------------------
State = Dict[Tuple[int, int], FrozenSet[int]]


def initial_state_stragglar(n: int) -> State:
    """Precondition: NS rank g holds c_g reduced over
    all non-stragglers; every other cell holds only its own rank."""
    sigma = n - 1
    ns = frozenset(range(n - 1))
    st: State = {}
    for h in range(n):
        for c in range(n - 1):
            st[(h, c)] = ns if (h == c and h != sigma) else frozenset([h])
    return st


def initial_state_uniform(n: int, num_chunks: int) -> State:
    """every cell holds its own rank only."""
    return {(h, c): frozenset([h]) for h in range(n) for c in range(num_chunks)}


def initial_state_broadcast(n: int) -> State:
    """Broadcast precondition: the non-stragglers completed an
    AllReduce among themselves; the straggler holds only its own data."""
    sigma = n - 1
    ns = frozenset(range(n - 1))
    return {(h, c): (frozenset([h]) if h == sigma else ns) for h in range(n) for c in range(n - 1)}


@dataclass
class Report:
    valid: bool
    rounds_executed: int
    violations: List[Tuple[int, str]]
    beta_coefficient: Fraction
    final_state: State


def apply_round(state: State, rnd: List[Transfer], n: int, r: int = 0,
                violations: Optional[list] = None, matching: bool = True,
                one_chunk: bool = True) -> State:
    """snapshot semantics; Reduce = disjoint union; Replace = superset copy.

    Single port: every rank sends <= 1 and receives <= 1 chunk per
    round.  With ``matching`` (StragglAR, P:204 / S:46) every rank also talks to
    a single partner; Ring sends to i+1 while receiving from i-1, so it is
    checked with ``matching=False``.  RHD and Broadcast send a block of several
    chunks to their single partner per round: ``one_chunk=False``
    keeps the one-partner rule and lifts the one-chunk rule.
    """
    viol = violations if violations is not None else []
    partner: Dict[int, int] = {}
    sends: Dict[int, int] = {}
    recvs: Dict[int, int] = {}
    for t in rnd:
        if t.src == t.dst:
            viol.append((r, f"self transfer at rank {t.src}"))
        for a, b in ((t.src, t.dst), (t.dst, t.src)):
            if matching and partner.setdefault(a, b) != b:
                viol.append((r, f"port violation: rank {a} in two matchings"))
        sends[t.src] = sends.get(t.src, 0) + 1
        recvs[t.dst] = recvs.get(t.dst, 0) + 1
    for k, v in list(sends.items()) + list(recvs.items()):
        if v > 1 and one_chunk:
            viol.append((r, f"port violation: rank {k} moves {v} chunks one way"))
    payload = [(t, state[(t.src, t.chunk)]) for t in rnd]   # snapshot first
    new = dict(state)
    for t, p in payload:
        if not p:
            viol.append((r, f"phantom send {t}"))
        cur = new[(t.dst, t.chunk)]
        if t.kind == REDUCE:
            if cur & p:
                viol.append((r, f"double count: {sorted(cur)} + {sorted(p)} at {t}"))
            new[(t.dst, t.chunk)] = cur | p
        elif t.kind == REPLACE:
            if not p >= cur:
                viol.append((r, f"regression: replace {sorted(cur)} by {sorted(p)} at {t}"))
            new[(t.dst, t.chunk)] = p
        else:
            viol.append((r, f"unknown kind {t.kind}"))
    return new


def verify_schedule(s: Schedule) -> Report:
    """replay from the algorithm's initial state; valid iff no
    violations and every cell ends with contributors {0..n-1}."""
    if s.algorithm == "stragglar":
        st = initial_state_stragglar(s.n)
    elif s.algorithm == "broadcast":
        st = initial_state_broadcast(s.n)
    else:
        st = initial_state_uniform(s.n, s.num_chunks)
    viol: List[Tuple[int, str]] = []
    beta = Fraction(0)
    blocks = s.algorithm in ("rhd", "broadcast")
    for r, rnd in enumerate(s.rounds):
        st = apply_round(st, rnd, s.n, r, viol, matching=(s.algorithm != "ring"), one_chunk=not blocks)
        per_port: Dict[Tuple[int, str], int] = {}
        for t in rnd:
            per_port[(t.src, "out")] = per_port.get((t.src, "out"), 0) + 1
            per_port[(t.dst, "in")] = per_port.get((t.dst, "in"), 0) + 1
        beta += Fraction(max(per_port.values()) if per_port else 0, s.num_chunks)
    full = frozenset(range(s.n))
    for (h, c), v in st.items():
        if v != full:
            viol.append((len(s.rounds), f"postcondition: rank {h} chunk {c} has {sorted(v)}"))
    return Report(not viol, len(s.rounds), viol, beta, st)
