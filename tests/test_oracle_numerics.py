"""Pins for oracle/numerics.py (CPU only): brute force, closed forms, library
routines for rounding, error bounds — never the oracle against itself alone."""
import numpy as np
import pytest
import torch

from oracle import numerics as N
from oracle import schedule as S
from paper_2505_23523_b200.inputs import make_inputs

DT = ("int32", "float32", "bfloat16")


def _bits(a):
    return np.asarray(a).view(np.uint8)


# ---------------------------------------------------------------- bf16 rounding vs torch
def test_bf16_rne_matches_torch():
    rng = np.random.default_rng(1)
    x = np.concatenate([
        rng.standard_normal(200000).astype(np.float32),
        np.clip(rng.standard_normal(20000) * 1e38, -3.4e38, 3.4e38).astype(np.float32),  # rounds up to inf
        (rng.standard_normal(20000) * 1e-39).astype(np.float32),     # subnormals
        np.array([0.0, -0.0, np.inf, -np.inf, 3.3895314e38, 1.0 + 2 ** -8, 1.0 + 3 * 2 ** -8,
                  1.0 + 2 ** -9], dtype=np.float32),
        # exact ties: low 16 bits == 0x8000 with even and odd kept LSB
        (rng.integers(0, 2 ** 15, 5000, dtype=np.uint32) << 17 | 0x8000).view(np.float32),
        (rng.integers(0, 2 ** 15, 5000, dtype=np.uint32) << 17 | 0x18000).view(np.float32),
    ])
    nan = np.isnan(x)
    got = N.f32_to_bf16_rne(x)
    # NaN payloads are implementation-defined: only require NaN -> NaN
    assert np.all((got[nan] & 0x7F80) == 0x7F80) and np.all((got[nan] & 0x7F) != 0)
    x = x[~nan]
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(N.f32_to_bf16_rne(x), ref)


def test_bf16_widen_matches_torch():
    b = np.arange(0, 2 ** 16, dtype=np.uint32).astype(np.uint16)
    b = b[(b & 0x7F80) != 0x7F80]  # skip inf/nan encodings
    ref = torch.from_numpy(b.view(np.int16)).view(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(N.bf16_to_f32(b), ref)


# ---------------------------------------------------------------- chunking / mapping
@pytest.mark.parametrize("count", [0, 1, 2, 3, 7, 8, 17, 1000, 2 ** 20, 10 ** 6 + 3])
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("dtype", DT)
def test_chunk_bounds_partition(count, n, dtype):
    """the buffer is divided into n-1 chunks c_0..c_{n-2} (reading 13:
    16-byte aligned starts, ceil split, shorter/empty tail)."""
    b = N.chunk_bounds(count, n - 1, dtype)
    assert len(b) == n - 1
    assert b[0][0] == 0 and b[-1][1] == count
    for (lo, hi), (lo2, _) in zip(b, b[1:]):
        assert hi == lo2 and lo <= hi
    v = 16 // N.ESIZE[dtype]
    assert all(lo % v == 0 for lo, _ in b if lo < count)
    assert max(hi - lo for lo, hi in b) <= -(-count // (n - 1)) + v - 1


@pytest.mark.parametrize("n", [2, 4, 8])
def test_logical_physical_swap(n):
    """P:200 / P:345: the straggler is swapped with rank n-1."""
    for sig in range(n):
        m = N.logical_to_physical(n, sig)
        assert sorted(m) == list(range(n)) and m[n - 1] == sig
        assert all(m[q] == q for q in range(n - 1) if q not in (sig,))


# ---------------------------------------------------------------- brute force
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("count", [0, 1, 5, 31, 64, 333])
def test_int32_brute_force(n, count):
    """P:202 postcondition with exact integer arithmetic: sum in int64, wrap."""
    xs = make_inputs(n, count, "int32", config=91, pattern="normal")
    exact = np.zeros(count, dtype=np.int64)
    for x in xs:
        exact += x.astype(np.int64)
    want = ((exact + 2 ** 31) % 2 ** 32 - 2 ** 31).astype(np.int32)
    for sig in range(n):
        outs = N.stragglar_allreduce(xs, sig, "int32")
        assert all(np.array_equal(o, want) for o in outs)
        assert np.array_equal(N.plain_allreduce(xs, sig, "int32"), want)
        assert all(np.array_equal(o, want) for o in N.ring_allreduce(xs, "int32"))


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("n", [2, 4, 8])
def test_bitmask_sum(dtype, n):
    """x_p = 1 << p must sum to 2^n - 1 everywhere (exact in all dtypes, n <= 8)."""
    xs = make_inputs(n, 203, dtype, pattern="bitmask")
    for sig in range(n):
        for o in N.stragglar_allreduce(xs, sig, dtype):
            v = N.bf16_to_f32(o) if dtype == "bfloat16" else o
            assert np.all(v == 2 ** n - 1)


@pytest.mark.parametrize("dtype", ("float32", "bfloat16"))
@pytest.mark.parametrize("n", [2, 4, 8])
def test_integer_valued_exact(dtype, n):
    """|x| <= 16, n <= 8: every partial sum is an integer <= 128 in magnitude,
    exact in bf16/fp32 in any order -> equals the integer brute force."""
    xs = make_inputs(n, 517, dtype, pattern="intval")
    ints = make_inputs(n, 517, "int32", pattern="intval")
    want = np.sum(np.stack(ints).astype(np.int64), axis=0)
    for sig in range(n):
        for o in N.stragglar_allreduce(xs, sig, dtype) + N.ring_allreduce(xs, dtype):
            v = N.bf16_to_f32(o) if dtype == "bfloat16" else o
            assert np.array_equal(v.astype(np.int64), want)


# ---------------------------------------------------------------- n = 2 textbook case
@pytest.mark.parametrize("dtype", DT)
def test_n2_is_textbook_sum(dtype):
    """n = 2: one exchange of the whole buffer = x0 + x1 elementwise,
    computed here by torch's own add in the buffer dtype."""
    xs = make_inputs(2, 1001, dtype, config=92)
    if dtype == "bfloat16":
        t = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16) for x in xs]
        want = (t[0] + t[1]).view(torch.int16).numpy().view(np.uint16)
    elif dtype == "float32":
        want = (torch.from_numpy(xs[0]) + torch.from_numpy(xs[1])).numpy()
    else:
        want = (torch.from_numpy(xs[0]) + torch.from_numpy(xs[1])).numpy()  # torch int32 wraps
    for sig in range(2):
        for o in N.stragglar_allreduce(xs, sig, dtype):
            assert np.array_equal(_bits(o), _bits(want))


# ---------------------------------------------------------------- fp32 order and error bound
@pytest.mark.parametrize("n", [4, 8])
def test_fp32_canonical_order_library(n):
    """Reading 12 (canonical order): the non-straggler sum is numpy's axis-0
    reduction of the ascending-physical stack (a sequential row fold), then
    x_sigma is added."""
    xs = make_inputs(n, 4099, "float32", config=93)
    for sig in range(n):
        ns = np.stack([xs[p] for p in range(n) if p != sig])
        want = np.add.reduce(ns, axis=0) + xs[sig]
        assert np.array_equal(N.plain_allreduce(xs, sig, "float32"), want)


@pytest.mark.parametrize("dtype,bound", [("float32", lambda n: (n - 1) * 2.0 ** -24),
                                         ("bfloat16", lambda n: 2 * 2.0 ** -8 + (n - 2) * 2.0 ** -24)])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_error_bound_vs_exact(dtype, bound, n):
    """Recursive summation bound |fl(sum) - sum| <= (k-1) u sum|x| (u = 2^-24
    for fp32; bf16 adds two roundings of u = 2^-8).  Both are
    far inside north_star's 1e-5 / 1e-2 tolerances."""
    xs = make_inputs(n, 20011, dtype, config=94)
    exact, absum = N.exact_sum_f64(xs, dtype)
    for sig in range(n):
        got = N.plain_allreduce(xs, sig, dtype)
        g = N.bf16_to_f32(got) if dtype == "bfloat16" else got
        err = np.max(np.abs(g.astype(np.float64) - exact) / np.maximum(absum, 1e-30))
        assert err <= bound(n) * 1.0001
        assert err <= (1e-5 if dtype == "float32" else 1e-2)


# ---------------------------------------------------------------- schedule independence
@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("n", [2, 4, 8])
@pytest.mark.parametrize("count", [0, 1, 6, 97, 4096 + 5])
def test_replay_equals_definition(dtype, n, count):
    """P:202 + P:206: every chunk is fully reduced exactly once (partial +
    x_sigma) and only copied afterwards, so the replay of Algorithm 1 equals
    the plain definition bitwise on every rank, for every straggler rank."""
    xs = make_inputs(n, count, dtype, config=95)
    for sig in range(n):
        want = N.plain_allreduce(xs, sig, dtype)
        for o in N.stragglar_allreduce(xs, sig, dtype):
            assert np.array_equal(_bits(o), _bits(want))


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_ring_replay_equals_rotation_definition(dtype, n):
    xs = make_inputs(n, 1237, dtype, config=96)
    want = N.plain_ring_allreduce(xs, dtype)
    for o in N.ring_allreduce(xs, dtype):
        assert np.array_equal(_bits(o), _bits(want))


def test_phase_a_precondition_values():
    """P:158 / P:202: after Phase A, logical rank g holds c_g summed over the
    non-stragglers; everything else is untouched (checked against the integer
    brute force)."""
    n, sig, count = 8, 3, 1000
    xs = make_inputs(n, count, "int32", config=97, pattern="intval")
    bufs = [x.copy() for x in xs]
    N.phase_a_reduce_scatter(bufs, sig, "int32")
    phys = N.logical_to_physical(n, sig)
    bounds = N.chunk_bounds(count, n - 1, "int32")
    ns_sum = sum(xs[p].astype(np.int64) for p in range(n) if p != sig)
    for g in range(n - 1):
        lo, hi = bounds[g]
        for q in range(n):
            want = ns_sum[lo:hi] if q == phys[g] else xs[q][lo:hi]
            assert np.array_equal(bufs[q][lo:hi].astype(np.int64), want)


def test_tolerance_function():
    xs = [np.array([1.0, -2.0], np.float32), np.array([3.0, 2.0], np.float32)]
    ref = np.array([4.0, 0.0], np.float32)
    got = np.array([4.0, 4e-6], np.float32)
    assert N.rel_error_vs_abs_sum(got, ref, xs, "float32") == pytest.approx(1e-6, rel=1e-3)


@pytest.mark.parametrize("dtype", DT)
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_direct_completion_equals_definition(dtype, n):
    """N1(ii): Phase A + one direct completion round reaches the plain
    definition bitwise (and therefore the pairwise schedule's result)."""
    xs = make_inputs(n, 2049, dtype, config=99)
    for sig in range(n):
        want = N.plain_allreduce(xs, sig, dtype)
        for o in N.direct_completion_allreduce(xs, sig, dtype):
            assert np.array_equal(_bits(o), _bits(want))
