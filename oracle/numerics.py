"""Numeric oracle for the StragglAR AllReduce — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

What the method computes (§3.1 "postcondition, where all ranks, including
the straggler, possess a fully reduced buffer") is the elementwise SUM of the n
ranks' buffers, identical on every rank.  Two oracles are given:

* ``plain_allreduce``: the result written out as a definition.  The paper does
  not fix the ReduceScatter summation order nor the bf16 accumulation
  precision (it called ``ncclReduceScatter``).  Reading (SURVEY.md
  §8(c).1 / §8(c).3 row 12): non-stragglers are summed in
  ascending *physical* rank order with fp32 accumulation, bf16 is rounded once
  after the ReduceScatter, and the straggler's data is added last with one
  more rounding ("exchange chunk c_r" to "fully reduce" it).
* ``stragglar_allreduce``: the method step by step — Phase A (ReduceScatter
  among the n-1 non-stragglers) then the round-by-round replay
  of Algorithm 1's schedule with snapshot semantics (reading 11).

dtypes: "int32" wraps modulo 2**32; "float32" adds in fp32 (IEEE RNE);
"bfloat16" (numpy uint16 bit patterns) widens to fp32, adds, and rounds to
nearest-even.
"""
from __future__ import annotations

from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import schedule as S

DTYPES = ("int32", "float32", "bfloat16")
ESIZE = {"int32": 4, "float32": 4, "bfloat16": 2}
NPTYPE = {"int32": np.int32, "float32": np.float32, "bfloat16": np.uint16}


# --------------------------------------------------------------------------
# bf16 <-> fp32 (the bf16 format is the top 16 bits of an IEEE binary32)
# --------------------------------------------------------------------------
def bf16_to_f32(b: np.ndarray) -> np.ndarray:
    """Widen: the bf16 bits become the high half of the binary32 word (exact)."""
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_rne(x: np.ndarray) -> np.ndarray:
    """Round binary32 to bf16, round-to-nearest, ties-to-even.

    Dropping the low 16 bits after adding 0x7FFF + (bit 16) rounds the
    magnitude to nearest with ties to the even kept LSB; a carry out of the
    mantissa correctly bumps the exponent (and saturates to inf).  NaNs keep
    a quiet-NaN payload.
    """
    u = np.asarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    r = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    if nan.any():
        r = r.copy()
        r[nan] = ((u[nan] >> np.uint64(16)).astype(np.uint16) | np.uint16(0x0040))
    return r


# --------------------------------------------------------------------------
# elementwise SUM of two operands, per dtype
# --------------------------------------------------------------------------
def add(a: np.ndarray, b: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "int32":
        return (a.astype(np.int32).view(np.uint32) + b.astype(np.int32).view(np.uint32)).view(np.int32)
    if dtype == "float32":
        return (a.astype(np.float32) + b.astype(np.float32)).astype(np.float32)
    if dtype == "bfloat16":
        return f32_to_bf16_rne(bf16_to_f32(a) + bf16_to_f32(b))
    raise ValueError(dtype)


# --------------------------------------------------------------------------
# buffer partition ("evenly divided into n-1 chunks"; reading 13)
# --------------------------------------------------------------------------
def chunk_elems(count: int, parts: int, dtype: str) -> int:
    """Ce = roundup(ceil(count/parts), 16/esz): chunks start on 16-byte boundaries.
    The paper pads to 1 KiB for NCCL; results do not depend on it."""
    v = 16 // ESIZE[dtype]
    per = -(-count // parts) if count else 0
    return -(-per // v) * v


def chunk_bounds(count: int, parts: int, dtype: str) -> List[Tuple[int, int]]:
    ce = chunk_elems(count, parts, dtype)
    return [(min(j * ce, count), min((j + 1) * ce, count)) for j in range(parts)]


def logical_to_physical(n: int, sigma_phys: int) -> List[int]:
    """the persistent straggler is swapped with logical rank n-1."""
    if not 0 <= sigma_phys < n:
        raise ValueError("straggler rank out of range")
    m = list(range(n))
    m[n - 1], m[sigma_phys] = sigma_phys, n - 1
    return m


# --------------------------------------------------------------------------
# plain definition
# --------------------------------------------------------------------------
def _canonical_partial(inputs: Sequence[np.ndarray], ns_phys: Sequence[int], dtype: str,
                       sl: slice = slice(None)) -> np.ndarray:
    """Sum over non-stragglers, ascending physical rank, left to right; one rounding for bf16."""
    order = sorted(ns_phys)
    if dtype == "int32":
        acc = inputs[order[0]][sl].astype(np.int32).view(np.uint32).copy()
        for p in order[1:]:
            acc = acc + inputs[p][sl].astype(np.int32).view(np.uint32)
        return acc.view(np.int32)
    if dtype == "float32":
        acc = inputs[order[0]][sl].astype(np.float32).copy()
        for p in order[1:]:
            acc = acc + inputs[p][sl].astype(np.float32)
        return acc
    acc = bf16_to_f32(inputs[order[0]][sl]).copy()
    for p in order[1:]:
        acc = acc + bf16_to_f32(inputs[p][sl])
    return f32_to_bf16_rne(acc)


def plain_allreduce(inputs: Sequence[np.ndarray], sigma_phys: int, dtype: str,
                    sl: slice = slice(None)) -> np.ndarray:
    """out[i] = (canonical non-straggler sum)[i] (+) x_sigma[i] — identical on all ranks."""
    n = len(inputs)
    ns = [p for p in range(n) if p != sigma_phys]
    if n == 1:
        return np.array(inputs[0][sl], copy=True)
    part = _canonical_partial(inputs, ns, dtype, sl)
    return add(part, inputs[sigma_phys][sl], dtype)


def exact_sum_f64(inputs: Sequence[np.ndarray], dtype: str) -> Tuple[np.ndarray, np.ndarray]:
    """Exact-ish reference for tolerances: float64 sum and sum of |x| (n <= 8
    binary32/bf16 terms are summed exactly enough in binary64 for 1e-5 checks)."""
    if dtype == "bfloat16":
        xs = [bf16_to_f32(x).astype(np.float64) for x in inputs]
    else:
        xs = [np.asarray(x).astype(np.float64) for x in inputs]
    s = np.zeros_like(xs[0])
    a = np.zeros_like(xs[0])
    for x in xs:
        s = s + x
        a = a + np.abs(x)
    return s, a


def rel_error_vs_abs_sum(got: np.ndarray, ref: np.ndarray, inputs: Sequence[np.ndarray],
                         dtype: str) -> float:
    """SURVEY.md §8(c).6 reading: max_i |got_i - ref_i| / max(sum_p |x_p[i]|, tiny)."""
    if dtype == "bfloat16":
        g = bf16_to_f32(got).astype(np.float64)
        r = bf16_to_f32(ref).astype(np.float64)
    else:
        g = np.asarray(got).astype(np.float64)
        r = np.asarray(ref).astype(np.float64)
    _, absum = exact_sum_f64(inputs, dtype)
    if g.size == 0:
        return 0.0
    return float(np.max(np.abs(g - r) / np.maximum(absum, 1e-30)))


# --------------------------------------------------------------------------
# the method, step by step
# --------------------------------------------------------------------------
def phase_a_reduce_scatter(bufs: List[np.ndarray], sigma_phys: int, dtype: str) -> None:
    """non-straggler logical rank g ends with chunk c_g reduced over
    all non-stragglers ("partially reduced").  In place; sigma untouched."""
    n = len(bufs)
    phys = logical_to_physical(n, sigma_phys)
    ns = [p for p in range(n) if p != sigma_phys]
    bounds = chunk_bounds(bufs[0].size, n - 1, dtype)
    snapshot = [b.copy() for b in bufs]
    for g in range(n - 1):
        lo, hi = bounds[g]
        bufs[phys[g]][lo:hi] = _canonical_partial(snapshot, ns, dtype, slice(lo, hi))


def replay_schedule(bufs: List[np.ndarray], sched: S.Schedule, phys: Sequence[int], dtype: str,
                    bounds: Sequence[Tuple[int, int]]) -> None:
    """Execute the rounds with snapshot semantics: every payload of round r is
    read before any write of round r lands (reading 11).  Reduce adds the
    payload into the receiver's copy; Replace overwrites it."""
    for rnd in sched.rounds:
        payloads = []
        for t in rnd:
            lo, hi = bounds[t.chunk]
            payloads.append((t, bufs[phys[t.src]][lo:hi].copy()))
        for t, p in payloads:
            lo, hi = bounds[t.chunk]
            dst = bufs[phys[t.dst]]
            if t.kind == S.REDUCE:
                dst[lo:hi] = add(dst[lo:hi], p, dtype)
            else:
                dst[lo:hi] = p


def stragglar_allreduce(inputs: Sequence[np.ndarray], sigma_phys: int, dtype: str,
                        sched: Optional[S.Schedule] = None) -> List[np.ndarray]:
    """Phase A + Phase B of StragglAR on n host buffers (physical rank order)."""
    n = len(inputs)
    bufs = [np.array(x, copy=True) for x in inputs]
    if n == 1:
        return bufs
    if sched is None:
        sched = S.generate(n)      # Algorithm 1 (powers of two) or Appendix B (even n)
    phys = logical_to_physical(n, sigma_phys)
    phase_a_reduce_scatter(bufs, sigma_phys, dtype)
    replay_schedule(bufs, sched, phys, dtype, chunk_bounds(bufs[0].size, n - 1, dtype))
    return bufs


def direct_completion_allreduce(inputs: Sequence[np.ndarray], sigma_phys: int, dtype: str) -> List[np.ndarray]:
    """NEXT row N1(ii): Phase A as in the paper, then one
    round in which each owner g fully reduces its chunk (partial_g + x_sigma,
    the same single add as the straggler exchange of P:164/P:206) and copies
    it to every rank.  Valid when the fabric lets a rank send to several peers
    at once (NVSwitch), which the paper's single-port model excludes
    (P:149-150).  Same result as the pairwise schedule, bit for bit."""
    n = len(inputs)
    bufs = [np.array(x, copy=True) for x in inputs]
    if n == 1:
        return bufs
    phys = logical_to_physical(n, sigma_phys)
    phase_a_reduce_scatter(bufs, sigma_phys, dtype)
    bounds = chunk_bounds(bufs[0].size, n - 1, dtype)
    snapshot = [b.copy() for b in bufs]
    for g in range(n - 1):
        lo, hi = bounds[g]
        full = add(snapshot[phys[g]][lo:hi], snapshot[sigma_phys][lo:hi], dtype)
        for q in range(n):
            bufs[q][lo:hi] = full
    return bufs


# --------------------------------------------------------------------------
# Ring baseline, ring-order oracle
# --------------------------------------------------------------------------
def ring_allreduce(inputs: Sequence[np.ndarray], dtype: str) -> List[np.ndarray]:
    """Replay of the Ring schedule (oracle.schedule.generate_ring) over physical
    ranks 0 -> 1 -> ... -> n-1 -> 0 with n chunks; partials travel in the
    buffer dtype, so bf16 is rounded at every hop."""
    n = len(inputs)
    bufs = [np.array(x, copy=True) for x in inputs]
    if n == 1:
        return bufs
    sched = S.generate_ring(n)
    replay_schedule(bufs, sched, list(range(n)), dtype, chunk_bounds(bufs[0].size, n, dtype))
    return bufs


def rhd_allreduce(inputs: Sequence[np.ndarray], dtype: str) -> List[np.ndarray]:
    """Replay of the RHD schedule (oracle.schedule.generate_rhd)
    over physical ranks with n chunks (the Ring's partition); partials travel
    in the buffer dtype, so bf16 is rounded after every pairwise add."""
    n = len(inputs)
    bufs = [np.array(x, copy=True) for x in inputs]
    if n == 1:
        return bufs
    replay_schedule(bufs, S.generate_rhd(n), list(range(n)), dtype, chunk_bounds(bufs[0].size, n, dtype))
    return bufs


def plain_rhd_allreduce(inputs: Sequence[np.ndarray], dtype: str) -> np.ndarray:
    """Definition of the RHD result, written elementwise with no chunks or
    rounds: a butterfly of pairwise sums, level k (k = 0..log n - 1) adding the
    values of ranks i and i XOR 2^k (halves with one partner, then
    quarters with the next; partner order as SPEC S:266), one rounding per
    level.  Every rank ends with the same bits (each add is commutative)."""
    n = len(inputs)
    v = [np.array(x, copy=True) for x in inputs]
    d = 1
    while d < n:
        v = [add(v[i], v[i ^ d], dtype) for i in range(n)]
        d *= 2
    return v[0]


def broadcast_allreduce(inputs: Sequence[np.ndarray], sigma_phys: int, dtype: str) -> List[np.ndarray]:
    """Straggler-aware Broadcast baseline, step by step.

    Precondition: the non-stragglers complete an AllReduce during
    the delay.  Its summation order is unstated; reading: the canonical order
    of StragglAR's Phase A (ascending physical rank, fp32 accumulation, bf16
    rounded once), applied to the whole buffer.  Then the schedule of
    ``schedule.generate_broadcast`` is replayed (the straggler's exchange adds
    x_sigma once, the log n - 1 doubling rounds copy)."""
    n = len(inputs)
    bufs = [np.array(x, copy=True) for x in inputs]
    if n == 1:
        return bufs
    ns = [p for p in range(n) if p != sigma_phys]
    part = _canonical_partial(inputs, ns, dtype)
    for p in ns:
        bufs[p][:] = part
    phys = logical_to_physical(n, sigma_phys)
    replay_schedule(bufs, S.generate_broadcast(n), phys, dtype, chunk_bounds(bufs[0].size, n - 1, dtype))
    return bufs


def plain_ring_allreduce(inputs: Sequence[np.ndarray], dtype: str) -> np.ndarray:
    """Definition of the Ring result: chunk k is accumulated in rotation order
    x_k, x_{k+1}, ..., x_{k+n-1} (mod n) with one rounding per hop."""
    n = len(inputs)
    count = inputs[0].size
    out = np.empty_like(inputs[0])
    for k, (lo, hi) in enumerate(chunk_bounds(count, n, dtype)):
        acc = np.array(inputs[k][lo:hi], copy=True)
        for j in range(1, n):
            acc = add(acc, inputs[(k + j) % n][lo:hi], dtype)
        out[lo:hi] = acc
    return out
