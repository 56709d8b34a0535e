"""GPU parity of the StragglAR kernels against the CPU oracle, through the C ABI.

Single-device team mode: all n logical ranks on cuda:0, same kernels, flags
and schedule as the per-process NVLink mode.  Every output element of every
rank is compared with the oracle's replay (bit-exact for every dtype: the
canonical summation order makes fp32/bf16 reproducible); the north_star
tolerances (1e-5 fp32, 1e-2 bf16 relative to sum|x|) are asserted
too, as the acceptance bar.
"""
import os

import numpy as np
import pytest
import torch

from oracle import numerics as N
from paper_2505_23523_b200.inputs import make_inputs

pytestmark = pytest.mark.gpu

TOL = {"int32": 0.0, "float32": 1e-5, "bfloat16": 1e-2}


@pytest.fixture(scope="module", params=["lsu", "tma"])
def S(request):
    """Every test runs with both Phase-B data movers (SM 16-byte vectors, TMA bulk)."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    os.environ["STRAGGLAR_MOVER"] = request.param
    import __graft_entry__

    __graft_entry__.build()
    from paper_2505_23523_b200 import stragglar

    torch.cuda.set_device(0)
    return stragglar


def to_dev(x, dtype):
    if dtype == "bfloat16":
        return torch.from_numpy(x.view(np.int16)).cuda().view(torch.bfloat16)
    return torch.from_numpy(x).cuda()


def to_host(t, dtype):
    if dtype == "bfloat16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def check_equal(outs, want, xs, dtype, what=""):
    for p, (o, w) in enumerate(zip(outs, want)):
        ob, wb = o.view(np.uint8), w.view(np.uint8)
        if not np.array_equal(ob, wb):
            diff = np.nonzero(o.view(np.uint16 if dtype == "bfloat16" else np.uint32)
                              != w.view(np.uint16 if dtype == "bfloat16" else np.uint32))[0]
            err = N.rel_error_vs_abs_sum(o, w, xs, dtype)
            pytest.fail(f"{what} rank {p}: {diff.size} elements differ (first {diff[:8]}), rel err {err:.3g}")
        assert N.rel_error_vs_abs_sum(o, w, xs, dtype) <= TOL[dtype]


def run_team(S, n, sigma, dtype, count, pattern="normal", config=1, algo="stragglar"):
    xs = make_inputs(n, count, dtype, config=config, pattern=pattern)
    bufs = [to_dev(x, dtype) for x in xs]
    S.stragglar_team_init(n, sigma)
    if algo == "stragglar":
        S.stragglar_team_allreduce(bufs)
    elif algo == "direct":
        S.stragglar_team_allreduce_direct(bufs)
    elif algo == "rhd":
        S.stragglar_team_allreduce_rhd(bufs)
    elif algo == "bcast":
        S.stragglar_team_allreduce_bcast(bufs)
    else:
        S.stragglar_team_allreduce_ring(bufs)
    torch.cuda.synchronize()
    code, where = S.stragglar_check_error_where(True)
    assert code == 0, f"{algo}: device error {code} at 0x{where:x}"

    outs = [to_host(b, dtype) for b in bufs]
    return xs, outs


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_every_straggler_small(S, dtype, n):
    """Every straggler rank; ragged counts (tails, fewer elements than chunks)."""
    for sigma in range(n):
        for count in [1, 5, 8 * (n - 1) + 3, 1000, 4099]:
            xs, outs = run_team(S, n, sigma, dtype, count)
            check_equal(outs, N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, f"n={n} sigma={sigma} count={count}")


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n,sigma", [(2, 1), (4, 0), (6, 2), (8, 0), (8, 3), (8, 7)])
def test_medium_spans_many_slices(S, dtype, n, sigma):
    """Sizes spanning every slice of every chunk plus a ragged tail."""
    for count in [(1 << 20) + 5, 10 ** 6 + 3]:
        xs, outs = run_team(S, n, sigma, dtype, count, config=2)
        check_equal(outs, N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, f"n={n} count={count}")


@pytest.mark.parametrize("pattern", ["bitmask", "intval"])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_patterns(S, pattern, dtype):
    """x_p = 1 << p: every element must be 2^n - 1 (a missed or doubled
    contribution names the rank); integer-valued inputs are exact."""
    n = 8
    xs, outs = run_team(S, n, 5, dtype, 77777, pattern=pattern)
    want = N.stragglar_allreduce(xs, 5, dtype)
    check_equal(outs, want, xs, dtype, pattern)
    if pattern == "bitmask":
        v = N.bf16_to_f32(outs[0]) if dtype == "bfloat16" else outs[0]
        assert np.all(v == 255)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_ring_baseline(S, dtype, n):
    """The hand-written Ring against the ring-order oracle (per-hop rounding)."""
    for count in [3, 1001, (1 << 18) + 7]:
        xs, outs = run_team(S, n, 0, dtype, count, algo="ring")
        check_equal(outs, N.ring_allreduce(xs, dtype), xs, dtype, f"ring n={n} count={count}")


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_direct_completion(S, dtype, n):
    """NEXT row N1(ii): Phase A + one-round direct completion; same bits as
    the paper's schedule (oracle.numerics.direct_completion_allreduce =
    plain definition), every straggler rank, ragged counts."""
    for sigma in range(n):
        for count in [3, 8 * (n - 1) + 5, 70001]:
            xs, outs = run_team(S, n, sigma, dtype, count, algo="direct")
            check_equal(outs, N.direct_completion_allreduce(xs, sigma, dtype), xs, dtype, f"direct n={n} s={sigma}")
    xs, outs = run_team(S, n, n - 1, dtype, (1 << 20) + 3, algo="direct")
    check_equal(outs, N.direct_completion_allreduce(xs, n - 1, dtype), xs, dtype, "direct large")


def test_repeated_calls_and_phases(S):
    """Epoch flags across back-to-back calls (no reset, no cross-call hazard);
    Phase A + injected delay + Phase B as separate calls equals the one-call
    allreduce; ring calls interleaved."""
    n, sigma, dtype, count = 8, 2, "float32", 300001
    S.stragglar_team_init(n, sigma)
    for it in range(6):
        xs = make_inputs(n, count, dtype, config=10 + it)
        bufs = [to_dev(x, dtype) for x in xs]
        if it % 3 == 0:
            S.stragglar_team_allreduce(bufs)
        elif it % 3 == 1:
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(20_000)
            S.stragglar_team_complete(bufs)
        else:
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(20_000)
            S.stragglar_team_complete_direct(bufs)
        ring = [to_dev(x, dtype) for x in xs]
        S.stragglar_team_allreduce_ring(ring)
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        check_equal([to_host(b, dtype) for b in bufs], N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, f"it {it}")
        check_equal([to_host(b, dtype) for b in ring], N.ring_allreduce(xs, dtype), xs, dtype, f"ring it {it}")


def test_all_ranks_identical_full_size(S):
    """BASELINE config 2 (n=8, straggler 0, 256 MiB fp32 per rank) in the
    launch configuration bench.py times: every element of every rank against
    the plain definition, and the ranks bitwise identical."""
    n, sigma, dtype, count = 8, 0, "float32", 1 << 26
    xs = make_inputs(n, count, dtype, config=2)
    bufs = [to_dev(x, dtype) for x in xs]
    S.stragglar_team_init(n, sigma)
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_inject_delay(1_000_000)
    S.stragglar_team_complete(bufs)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    for p in range(1, n):
        assert torch.equal(bufs[p].view(torch.int32), bufs[0].view(torch.int32))
    got = to_host(bufs[0], dtype)
    want = N.plain_allreduce(xs, sigma, dtype)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("piece_bytes", [None, "4096", "100000"])
def test_host_entry_point(S, piece_bytes):
    """End-to-end C-ABI call from pinned host buffers; with small pieces the
    H2D / AllReduce / D2H pipeline runs many overlapped pieces (ragged last
    piece included) and must give the same bits."""
    n, sigma, dtype, count = 4, 1, "bfloat16", 123457
    xs = make_inputs(n, count, dtype, config=3)
    host = [torch.from_numpy(x.view(np.int16)).view(torch.bfloat16).pin_memory() for x in xs]
    out = [torch.empty_like(h).pin_memory() for h in host]
    dev = [torch.empty(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    old = os.environ.pop("STRAGGLAR_E2E_PIECE_BYTES", None)
    if piece_bytes:
        os.environ["STRAGGLAR_E2E_PIECE_BYTES"] = piece_bytes
    try:
        S.stragglar_team_init(n, sigma)          # knobs are read at init
        S.stragglar_team_allreduce_host(host, out, dev)
    finally:
        os.environ.pop("STRAGGLAR_E2E_PIECE_BYTES", None)
        if old is not None:
            os.environ["STRAGGLAR_E2E_PIECE_BYTES"] = old
    outs = [o.view(torch.int16).numpy().view(np.uint16) for o in out]
    check_equal(outs, N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, "host")
    S.stragglar_team_allreduce_host(host, host, dev)          # in place on the host
    check_equal([h.view(torch.int16).numpy().view(np.uint16) for h in host],
                N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, "host in place")


def test_cuda_graph_replay(S):
    """The call epoch lives in device memory, so a captured CUDA graph of the
    whole AllReduce (Phase A, delay, Phase B) replays correctly; inputs are
    refreshed in the static buffers between replays."""
    n, sigma, dtype, count = 8, 6, "bfloat16", 200003
    S.stragglar_team_init(n, sigma)
    bufs = [torch.empty(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    ring = [torch.empty_like(b) for b in bufs]
    for b in bufs + ring:
        b.zero_()
    S.stragglar_team_allreduce(bufs)          # warm up outside capture
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            S.stragglar_team_reduce_scatter(bufs, side)
            S.stragglar_team_inject_delay(5_000, side)
            S.stragglar_team_complete(bufs, side)
            S.stragglar_team_allreduce_ring(ring, side)
    for it in range(3):
        xs = make_inputs(n, count, dtype, config=30 + it)
        for b, r, x in zip(bufs, ring, xs):
            b.copy_(to_dev(x, dtype))
            r.copy_(to_dev(x, dtype))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        check_equal([to_host(b, dtype) for b in bufs], N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, f"graph {it}")
        check_equal([to_host(b, dtype) for b in ring], N.ring_allreduce(xs, dtype), xs, dtype, f"graph ring {it}")
    # eager calls still work after the replays (shared device epoch)
    xs = make_inputs(n, count, dtype, config=40)
    for b, x in zip(bufs, xs):
        b.copy_(to_dev(x, dtype))
    S.stragglar_team_allreduce(bufs)
    torch.cuda.synchronize()
    check_equal([to_host(b, dtype) for b in bufs], N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, "eager after graph")


def test_argument_errors(S):
    S.stragglar_team_init(4, 0)
    bufs = [torch.zeros(64, device="cuda") for _ in range(4)]
    with pytest.raises(S.StragglarError) as e:
        S.stragglar_team_complete(bufs)       # Phase B without Phase A
    assert e.value.status == 1
    S.stragglar_team_reduce_scatter(bufs)
    with pytest.raises(S.StragglarError):
        S.stragglar_team_allreduce(bufs)      # Phase A pending: complete it first
    S.stragglar_team_complete(bufs)
    mis = [torch.zeros(65, device="cuda")[1:] for _ in range(4)]
    with pytest.raises(S.StragglarError) as e:
        S.stragglar_team_allreduce(mis)       # not 16-byte aligned
    assert e.value.status == 1
    with pytest.raises(TypeError):
        S.stragglar_team_allreduce([torch.zeros(64, device="cuda", dtype=torch.float64) for _ in range(4)])
    S.stragglar_team_allreduce([torch.zeros(0, device="cuda") for _ in range(4)])  # count 0: no-op
    with pytest.raises(S.StragglarError):
        S.stragglar_team_init(3, 0)
    with pytest.raises(S.StragglarError):
        S.stragglar_team_init(10, 0)


@pytest.mark.parametrize("n,sigma,count,dtype", [
    (8, 0, 13_107_200, "bfloat16"),   # BASELINE configs[3]: 25 MiB bf16 DP bucket
    (8, 3, 524_288, "bfloat16"),      # BASELINE configs[4]: [64 x 8192] bf16 TP activation, straggler 3
    (4, 0, 1 << 20, "float32"),       # BASELINE configs[0]
])
def test_baseline_configs_exact(S, n, sigma, count, dtype):
    """The BASELINE workloads at their exact sizes, split phases + delay as
    bench.py/sweep.py time them, every element vs the oracle's replay."""
    xs = make_inputs(n, count, dtype, config=4)
    bufs = [to_dev(x, dtype) for x in xs]
    S.stragglar_team_init(n, sigma)
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_inject_delay(50_000)
    S.stragglar_team_complete(bufs)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    check_equal([to_host(b, dtype) for b in bufs], N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, "config")


def test_huge_buffers_sampled(S):
    """Maximum sizes: 3 GiB per rank (> 2^31 bytes, 24 GiB over the 8 ranks),
    inputs drawn on the device from seeded generators; the plain definition
    is evaluated by the oracle on 200k sampled indices (chunk and slice
    boundaries included) and every rank must be bitwise identical."""
    n, sigma = 8, 2
    count = (3 << 30) // 4 + 7
    S.stragglar_team_init(n, sigma)
    bufs = []
    for p in range(n):
        g = torch.Generator(device="cuda").manual_seed(2505_23523 + p)
        bufs.append(torch.randn(count, device="cuda", generator=g))
    ce = N.chunk_elems(count, n - 1, "float32")
    edges = [0, 1, count - 1, count - 2, (1 << 29) - 1, 1 << 29, (1 << 31) // 4, ((1 << 31) // 4) + 1]
    edges += [j * ce + d for j in range(1, n - 1) for d in (-1, 0, 1)]
    rng = np.random.default_rng(7)
    idx = np.unique(np.concatenate([np.array(edges), rng.integers(0, count, 200_000)]))
    tidx = torch.from_numpy(idx).cuda()
    xs = [b[tidx].cpu().numpy() for b in bufs]
    S.stragglar_team_reduce_scatter(bufs)
    S.stragglar_team_inject_delay(100_000)
    S.stragglar_team_complete(bufs)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    want = N.plain_allreduce(xs, sigma, "float32")
    for p in range(n):
        got = bufs[p][tidx].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), p
    for p in range(1, n):
        assert torch.equal(bufs[p].view(torch.int32), bufs[0].view(torch.int32))
    del bufs
    torch.cuda.empty_cache()


def test_randomized_cases(S):
    """Seeded random sweep: world, straggler, dtype, count, pattern, algorithm."""
    rng = np.random.default_rng(2505)
    for case in range(40):
        n = int(rng.choice([2, 4, 6, 8]))
        sigma = int(rng.integers(0, n))
        dtype = str(rng.choice(["int32", "float32", "bfloat16"]))
        count = int(rng.choice([rng.integers(1, 64), rng.integers(64, 5000), rng.integers(5000, 600_000)]))
        pattern = str(rng.choice(["normal", "intval", "bitmask"]))
        algo = str(rng.choice(["stragglar", "direct", "ring"]))
        xs, outs = run_team(S, n, sigma, dtype, count, pattern=pattern, config=60 + case, algo=algo)
        want = N.ring_allreduce(xs, dtype) if algo == "ring" else N.stragglar_allreduce(xs, sigma, dtype)
        check_equal(outs, want, xs, dtype, f"case {case}: n={n} s={sigma} {dtype} {count} {pattern} {algo}")


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_system_scope_flags(S, dtype):
    """The per-process (NVLink) mode's memory-model scope — ld.acquire.sys /
    fence.acq_rel.sys flags — exercised in team mode on every Phase-B path
    (schedule, direct completion) and the Ring, with one and several slices
    per CTA."""
    old = {k: os.environ.get(k) for k in ("STRAGGLAR_SYS_SCOPE", "STRAGGLAR_SUBSLICES", "STRAGGLAR_SUBSLICE_BYTES")}
    try:
        os.environ["STRAGGLAR_SYS_SCOPE"] = "1"
        for sub in ("1", "16"):
            os.environ["STRAGGLAR_SUBSLICES"] = sub
            os.environ["STRAGGLAR_SUBSLICE_BYTES"] = "4096"
            for n, sigma in [(4, 2), (8, 0), (6, 5)]:
                for count in [9999, 300001, 3_000_017]:
                    for algo in ("stragglar", "direct", "ring"):
                        xs, outs = run_team(S, n, sigma, dtype, count, config=80, algo=algo)
                        want = N.ring_allreduce(xs, dtype) if algo == "ring" else N.stragglar_allreduce(xs, sigma, dtype)
                        check_equal(outs, want, xs, dtype, f"sys n={n} {algo} sub={sub}")
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_delayed_single_launch(S):
    """The measurement entry point with the straggler delayed inside the
    kernel (Phase B overlapping the Phase-A tail) gives the same bits."""
    n, sigma, dtype = 8, 4, "float32"
    S.stragglar_team_init(n, sigma)
    for count, d in [(123457, 0), (123457, 30_000), (2_000_003, 100_000)]:
        xs = make_inputs(n, count, dtype, config=90)
        bufs = [to_dev(x, dtype) for x in xs]
        S.stragglar_team_allreduce_delayed(bufs, d)
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        check_equal([to_host(b, dtype) for b in bufs], N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, f"d={d}")


def test_trace_stamps(S):
    """Tracing: every Phase-B op of every rank and slice gets ordered stamps
    (wait <= data <= done), and the result is still exact."""
    n, sigma, dtype, count = 4, 1, "float32", 200003
    xs = make_inputs(n, count, dtype, config=95)
    bufs = [to_dev(x, dtype) for x in xs]
    S.stragglar_team_init(n, sigma)
    S.stragglar_team_set_trace(True)
    S.stragglar_team_allreduce(bufs)
    torch.cuda.synchronize()
    tr, G = S.stragglar_team_read_trace()
    S.stragglar_team_set_trace(False)
    check_equal([to_host(b, dtype) for b in bufs], N.stragglar_allreduce(xs, sigma, dtype), xs, dtype, "trace")
    nops = [4, 2, 2, 4]          # sends per logical rank at n = 4 (Appendix A of SURVEY)
    seen = 0
    for p in range(n):
        logical = {1: 3, 3: 1}.get(p, p)     # straggler 1 <-> logical 3
        for s in range(G):
            for k in range(nops[logical]):
                w, d, e = tr[((p * G + s) * 16 + k) * 3:((p * G + s) * 16 + k) * 3 + 3]
                assert 0 < w <= d <= e, (p, s, k, w, d, e)
                seen += 1
    assert seen == G * sum(nops)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_subslices(S, dtype):
    """Several slices per CTA (LaunchPlan::sub, each handed over with its own
    flag): forced at moderate sizes with small slice targets, on the fused
    call, the split phases, direct completion and the Ring (sub = 1 there),
    with the Phase-B trace laid out per slice."""
    keys = ("STRAGGLAR_SLICE_BYTES", "STRAGGLAR_SUBSLICE_BYTES")
    old = {k: os.environ.get(k) for k in keys}
    try:
        os.environ["STRAGGLAR_SLICE_BYTES"] = "1024"
        os.environ["STRAGGLAR_SUBSLICE_BYTES"] = "1024"     # 3-16 slices per CTA below
        for n, sigma, count in [(8, 0, 2_000_003), (4, 2, 900_001), (6, 1, 777_777), (2, 1, 500_001)]:
            for algo in ("stragglar", "direct", "ring"):
                xs, outs = run_team(S, n, sigma, dtype, count, config=97, algo=algo)
                want = N.ring_allreduce(xs, dtype) if algo == "ring" else N.stragglar_allreduce(xs, sigma, dtype)
                check_equal(outs, want, xs, dtype, f"sub n={n} {algo}")
            # split phases with tracing: G * sub slices per chunk in the trace
            xs = make_inputs(n, count, dtype, config=98)
            bufs = [to_dev(x, dtype) for x in xs]
            S.stragglar_team_init(n, sigma)
            S.stragglar_team_set_trace(True)
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(20_000)
            S.stragglar_team_complete(bufs)
            torch.cuda.synchronize()
            assert S.stragglar_team_check_error() == 0
            tr, nslices = S.stragglar_team_read_trace()
            S.stragglar_team_set_trace(False)
            assert nslices > S.stragglar_team_slices(), (nslices, S.stragglar_team_slices())
            check_equal([to_host(b, dtype) for b in bufs], N.stragglar_allreduce(xs, sigma, dtype), xs, dtype,
                        f"sub split n={n}")
            stamps = np.asarray(tr).reshape(n, nslices, 16, 3)
            assert (stamps[:, :, 0, 2] > 0).all()       # every rank's first op ran on every slice
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


# ---------------------------------------------------------------- NEXT N3 baselines
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 4, 8])
def test_rhd_baseline(S, dtype, n):
    """Recursive halving/doubling against the oracle's RHD replay (butterfly
    order, bf16 rounded per step), ragged counts incl. fewer elements than ranks."""
    for count in [1, 3, 8 * n + 5, 1001, (1 << 18) + 7, (1 << 20) + 3]:
        xs, outs = run_team(S, n, 0, dtype, count, algo="rhd", config=80)
        check_equal(outs, N.rhd_allreduce(xs, dtype), xs, dtype, f"rhd n={n} count={count}")


def test_rhd_needs_power_of_two(S):
    S.stragglar_team_init(6, 0)
    bufs = [torch.zeros(64, device="cuda") for _ in range(6)]
    with pytest.raises(S.StragglarError) as e:
        S.stragglar_team_allreduce_rhd(bufs)
    assert e.value.status == 2


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 4, 6, 8])
def test_bcast_baseline(S, dtype, n):
    """Straggler-aware Broadcast (one launch): every straggler rank, ragged
    counts; equals the oracle's step-by-step replay (= the plain definition)."""
    for sigma in range(n):
        for count in [3, 8 * (n - 1) + 5, 70001]:
            xs, outs = run_team(S, n, sigma, dtype, count, algo="bcast", config=81)
            check_equal(outs, N.broadcast_allreduce(xs, sigma, dtype), xs, dtype, f"bcast n={n} s={sigma} c={count}")
    xs, outs = run_team(S, n, n // 2, dtype, (1 << 20) + 3, algo="bcast", config=82)
    check_equal(outs, N.broadcast_allreduce(xs, n // 2, dtype), xs, dtype, "bcast large")


@pytest.mark.parametrize("n,sigma", [(8, 0), (4, 3), (2, 1)])
def test_bcast_split_with_delay(S, n, sigma):
    """Precondition -> injected delay -> completion (how the bench times the
    Broadcast baseline's post-arrival part) gives the same bits; a completion
    without its precondition is rejected."""
    dtype, count = "bfloat16", 250007
    S.stragglar_team_init(n, sigma)
    bufs = [torch.zeros(64, device="cuda") for _ in range(n)]
    with pytest.raises(S.StragglarError):
        S.stragglar_team_bcast_complete(bufs)
    xs = make_inputs(n, count, dtype, config=83)
    bufs = [to_dev(x, dtype) for x in xs]
    S.stragglar_team_bcast_precondition(bufs)
    with pytest.raises(S.StragglarError):
        S.stragglar_team_allreduce(bufs)          # a precondition is pending
    S.stragglar_team_inject_delay(30_000)
    S.stragglar_team_bcast_complete(bufs)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    check_equal([to_host(b, dtype) for b in bufs], N.broadcast_allreduce(xs, sigma, dtype), xs, dtype, "bcast split")


def test_all_algorithms_back_to_back(S):
    """Every algorithm of the library on the same communicator, queued back to
    back with no host synchronisation: the flag slots of one algorithm never
    satisfy a wait of another (epochs), and each result equals its oracle."""
    n, sigma, dtype, count = 8, 5, "float32", 180001
    S.stragglar_team_init(n, sigma)
    algos = ["stragglar", "rhd", "bcast", "ring", "direct", "bcast", "rhd", "stragglar"]
    runs = []
    for it, algo in enumerate(algos):
        xs = make_inputs(n, count, dtype, config=84 + it)
        bufs = [to_dev(x, dtype) for x in xs]
        runs.append((algo, xs, bufs))
    torch.cuda.synchronize()
    for algo, xs, bufs in runs:
        {"stragglar": S.stragglar_team_allreduce, "rhd": S.stragglar_team_allreduce_rhd,
         "bcast": S.stragglar_team_allreduce_bcast, "ring": S.stragglar_team_allreduce_ring,
         "direct": S.stragglar_team_allreduce_direct}[algo](bufs)
    torch.cuda.synchronize()
    assert S.stragglar_team_check_error() == 0
    for algo, xs, bufs in runs:
        want = {"rhd": lambda: N.rhd_allreduce(xs, dtype), "ring": lambda: N.ring_allreduce(xs, dtype),
                "bcast": lambda: N.broadcast_allreduce(xs, sigma, dtype)}.get(
                    algo, lambda: N.stragglar_allreduce(xs, sigma, dtype))()
        check_equal([to_host(b, dtype) for b in bufs], want, xs, dtype, algo)


def test_baselines_full_size(S):
    """BASELINE config 2 size (n=8, 256 MiB fp32 per rank) in the bench's
    launch configuration: RHD vs its butterfly definition and Broadcast vs the
    plain definition on 300k sampled indices; all ranks bitwise identical."""
    n, sigma, dtype, count = 8, 0, "float32", 1 << 26
    xs_full = make_inputs(n, count, dtype, config=2)
    rng = np.random.default_rng(11)
    idx = np.unique(np.concatenate([rng.integers(0, count, 300_000), [0, count - 1]]))
    xs = [x[idx] for x in xs_full]
    S.stragglar_team_init(n, sigma)
    for algo in ("rhd", "bcast"):
        bufs = [to_dev(x, dtype) for x in xs_full]
        if algo == "rhd":
            S.stragglar_team_allreduce_rhd(bufs)
            want = N.plain_rhd_allreduce(xs, dtype)
        else:
            S.stragglar_team_bcast_precondition(bufs)
            S.stragglar_team_inject_delay(1_000_000)
            S.stragglar_team_bcast_complete(bufs)
            want = N.plain_allreduce(xs, sigma, dtype)
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        for p in range(1, n):
            assert torch.equal(bufs[p].view(torch.int32), bufs[0].view(torch.int32)), (algo, p)
        got = bufs[0][torch.from_numpy(idx).cuda()].cpu().numpy()
        assert np.array_equal(got.view(np.uint32), want.view(np.uint32)), algo
        del bufs
        torch.cuda.empty_cache()


@pytest.mark.parametrize("algo", ["rhd", "bcast", "stragglar", "ring"])
def test_baselines_many_subslices(S, algo):
    """8 CTAs per rank and ~4 KB slices: every CTA walks up to 16 sub-slices,
    one flag each (the hand-off granularity of large messages, exercised at a
    size the oracle replays in full)."""
    keys = ("STRAGGLAR_TEAM_SLICES", "STRAGGLAR_SLICE_BYTES", "STRAGGLAR_SUBSLICE_BYTES")
    old = {k: os.environ.get(k) for k in keys}
    os.environ.update({"STRAGGLAR_TEAM_SLICES": "8", "STRAGGLAR_SLICE_BYTES": "1024", "STRAGGLAR_SUBSLICE_BYTES": "4096"})
    try:
        n, sigma, dtype, count = 4, 3, "float32", 400003
        xs, outs = run_team(S, n, sigma, dtype, count, algo=algo, config=85)
    finally:
        for k, v in old.items():
            os.environ.pop(k, None)
            if v is not None:
                os.environ[k] = v
    want = {"rhd": lambda: N.rhd_allreduce(xs, dtype), "ring": lambda: N.ring_allreduce(xs, dtype),
            "bcast": lambda: N.broadcast_allreduce(xs, sigma, dtype)}.get(
                algo, lambda: N.stragglar_allreduce(xs, sigma, dtype))()
    check_equal(outs, want, xs, dtype, algo)


def test_baselines_randomized_and_graph(S):
    """Seeded random sweep over the NEXT-N3 baselines (world, straggler, dtype,
    count, pattern), then RHD + Broadcast (split, with the delay) captured in
    one CUDA graph and replayed on fresh inputs."""
    rng = np.random.default_rng(2506)
    for case in range(24):
        algo = str(rng.choice(["rhd", "bcast"]))
        n = int(rng.choice([2, 4, 8] if algo == "rhd" else [2, 4, 6, 8]))
        sigma = int(rng.integers(0, n))
        dtype = str(rng.choice(["int32", "float32", "bfloat16"]))
        count = int(rng.choice([rng.integers(1, 64), rng.integers(64, 5000), rng.integers(5000, 600_000)]))
        pattern = str(rng.choice(["normal", "intval", "bitmask"]))
        xs, outs = run_team(S, n, sigma, dtype, count, pattern=pattern, config=120 + case, algo=algo)
        want = N.rhd_allreduce(xs, dtype) if algo == "rhd" else N.broadcast_allreduce(xs, sigma, dtype)
        check_equal(outs, want, xs, dtype, f"case {case}: {algo} n={n} s={sigma} {dtype} {count} {pattern}")
    n, sigma, dtype, count = 8, 4, "bfloat16", 150001
    S.stragglar_team_init(n, sigma)
    rb = [torch.zeros(count, dtype=torch.bfloat16, device="cuda") for _ in range(n)]
    bb = [torch.zeros_like(b) for b in rb]
    S.stragglar_team_allreduce_rhd(rb)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    with torch.cuda.stream(side):
        with torch.cuda.graph(g, stream=side):
            S.stragglar_team_allreduce_rhd(rb, side)
            S.stragglar_team_bcast_precondition(bb, side)
            S.stragglar_team_inject_delay(5_000, side)
            S.stragglar_team_bcast_complete(bb, side)
    for it in range(2):
        xs = make_inputs(n, count, dtype, config=150 + it)
        for r, b, x in zip(rb, bb, xs):
            r.copy_(to_dev(x, dtype))
            b.copy_(to_dev(x, dtype))
        torch.cuda.synchronize()
        g.replay()
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        check_equal([to_host(b, dtype) for b in rb], N.rhd_allreduce(xs, dtype), xs, dtype, f"graph rhd {it}")
        check_equal([to_host(b, dtype) for b in bb], N.broadcast_allreduce(xs, sigma, dtype), xs, dtype, f"graph bcast {it}")


def test_sweep_max_size_bf16_sampled(S):
    """BASELINE config 3's largest point (1 GiB bf16 per rank, n = 8, straggler 0)
    through StragglAR (split, with delay), RHD and the Broadcast baseline:
    inputs drawn on the device, each result checked on 200k sampled indices
    (chunk edges included) against its plain definition, and all ranks bitwise
    identical."""
    n, sigma, count = 8, 0, 1 << 29
    S.stragglar_team_init(n, sigma)
    ce = N.chunk_elems(count, n - 1, "bfloat16")
    ce_r = N.chunk_elems(count, n, "bfloat16")
    edges = [0, 1, count - 1] + [j * c + d for c in (ce, ce_r) for j in range(1, n) for d in (-1, 0, 1) if j * c + d < count]
    rng = np.random.default_rng(17)
    idx = np.unique(np.concatenate([np.array(edges), rng.integers(0, count, 200_000)]))
    tidx = torch.from_numpy(idx).cuda()
    for algo in ("stragglar", "rhd", "bcast"):
        bufs = []
        for p in range(n):
            g = torch.Generator(device="cuda").manual_seed(2505_23523 + 10 * p)
            bufs.append(torch.randn(count, device="cuda", generator=g).to(torch.bfloat16))
        xs = [b[tidx].view(torch.int16).cpu().numpy().view(np.uint16) for b in bufs]
        if algo == "stragglar":
            S.stragglar_team_reduce_scatter(bufs)
            S.stragglar_team_inject_delay(200_000)
            S.stragglar_team_complete(bufs)
            want = N.plain_allreduce(xs, sigma, "bfloat16")
        elif algo == "rhd":
            S.stragglar_team_allreduce_rhd(bufs)
            want = N.plain_rhd_allreduce(xs, "bfloat16")
        else:
            S.stragglar_team_bcast_precondition(bufs)
            S.stragglar_team_inject_delay(200_000)
            S.stragglar_team_bcast_complete(bufs)
            want = N.plain_allreduce(xs, sigma, "bfloat16")
        torch.cuda.synchronize()
        assert S.stragglar_team_check_error() == 0
        for p in range(1, n):
            assert torch.equal(bufs[p].view(torch.int16), bufs[0].view(torch.int16)), (algo, p)
        got = bufs[0][tidx].view(torch.int16).cpu().numpy().view(np.uint16)
        assert np.array_equal(got, want), algo
        del bufs
        torch.cuda.empty_cache()


@pytest.mark.parametrize("knobs", [
    {"STRAGGLAR_OP_LANES": "1"},                                   # one CTA walks a slice's ops in round order
    {"STRAGGLAR_OP_LANES": "16", "STRAGGLAR_LANE_SLICE_MAX": "0"},  # lanes, plain 16 KB slices
    {"STRAGGLAR_LANE_SLICE_MAX": "65536"},                         # lanes with up to 64 KB slices
    {"STRAGGLAR_RS_WHOLE": "1", "STRAGGLAR_SUBSLICES": "16", "STRAGGLAR_SUBSLICE_BYTES": "4096"},
    {"STRAGGLAR_SYS_SCOPE": "1", "STRAGGLAR_OP_LANES": "16"},
])
def test_layout_knobs_same_bits(S, knobs):
    """Round-2 layout choices (op lanes, lane-aware slices, whole-range Phase A
    with batched flags) change who moves which bytes when, never the result:
    split and fused calls stay bit-exact vs the oracle."""
    old = {k: os.environ.get(k) for k in knobs}
    try:
        os.environ.update(knobs)
        for n, sigma in [(4, 1), (6, 5), (8, 3)]:
            for dtype in ("float32", "bfloat16"):
                for count in [5003, 200_003, 1_500_001]:
                    xs = make_inputs(n, count, dtype, config=33)
                    want = N.stragglar_allreduce(xs, sigma, dtype)
                    for split in (False, True):
                        bufs = [to_dev(x, dtype) for x in xs]
                        S.stragglar_team_init(n, sigma)
                        if split:
                            S.stragglar_team_reduce_scatter(bufs)
                            S.stragglar_team_inject_delay(20_000)
                            S.stragglar_team_complete(bufs)
                        else:
                            S.stragglar_team_allreduce(bufs)
                        torch.cuda.synchronize()
                        assert S.stragglar_team_check_error() == 0
                        check_equal([to_host(b, dtype) for b in bufs], want, xs, dtype,
                                    f"{knobs} n={n} {dtype} count={count} split={split}")
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
