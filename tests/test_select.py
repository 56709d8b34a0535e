"""Algorithm selection for an expected delay (NEXT row N2) against the
paper's §4.2 condition as the oracle states it (CPU only)."""
import math

import pytest

from oracle import cost as C


@pytest.fixture(scope="module")
def S():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2505_23523_b200 import stragglar

    return stragglar


@pytest.mark.parametrize("n", [2, 4, 8, 16, 64])
@pytest.mark.parametrize("nbytes", [2 ** 20, 25 * 2 ** 20, 2 ** 28, 2 ** 30, 4 * 2 ** 30])
def test_critical_delay_matches_paper_beta_terms(S, n, nbytes):
    """alpha = 0: the library's critical delay equals P:423-424 evaluated with
    the oracle's Table-1 costs (the ReduceScatter moves (m-1)/m of the buffer
    among m = n-1 ranks in both)."""
    beta = 1 / 770e9
    _, crit = S.stragglar_select(n, nbytes, 0.0, 0.0, beta)
    want = C.critical_delay(n, nbytes, 0.0, beta, C.t_ring(n, nbytes, 0.0, beta))
    assert crit == pytest.approx(want, rel=1e-12, abs=1e-15)


@pytest.mark.parametrize("n", [4, 8])
def test_choice_flips_at_the_critical_delay(S, n):
    """StragglAR is chosen iff delay >= critical; the end-to-end model times
    (P:417 measured from the non-stragglers' start) tie at the critical delay."""
    alpha, beta, s = 3e-6, 1 / 770e9, 2 ** 30
    _, crit = S.stragglar_select(n, s, 0.0, alpha, beta)
    assert S.stragglar_select(n, s, crit * 1.001 + 1e-9, alpha, beta)[0]
    if crit > 0:
        assert not S.stragglar_select(n, s, crit * 0.999, alpha, beta)[0]
        L = int(math.log2(n))
        R = n + L - 2
        t_rs = alpha + (n - 2) / (n - 1) * s * beta
        t_sar = R * alpha + R / (n - 1) * s * beta
        t_ring = 2 * (n - 1) * alpha + 2 * (n - 1) / n * s * beta
        assert max(crit, t_rs) + t_sar == pytest.approx(crit + t_ring, rel=1e-9)


def test_large_buffers_without_delay_prefer_ring_at_n8(S):
    """with no delay StragglAR pays the whole ReduceScatter (15/7 vs
    7/4 s*beta at n=8) and loses; with a delay that masks the ReduceScatter it
    wins (Table 1)."""
    use0, crit = S.stragglar_select(8, 2 ** 30, 0.0, 3e-6, 1 / 770e9)
    assert not use0 and crit > 0
    use1, _ = S.stragglar_select(8, 2 ** 30, 0.0015, 3e-6, 1 / 770e9)
    assert use1


def test_select_rejects_bad_world(S):
    with pytest.raises(S.StragglarError):
        S.stragglar_select(5, 1.0, 0.0, 0.0, 1.0)


@pytest.mark.parametrize("n", [4, 8, 16])
@pytest.mark.parametrize("nbytes", [2 ** 20, 2 ** 26, 2 ** 30])
@pytest.mark.parametrize("delay", [0.0, 1e-4, 2e-3])
@pytest.mark.parametrize("alpha", [0.0, 3e-6])
def test_select_algorithm_is_the_model_argmin(S, n, nbytes, delay, alpha):
    """N2 + N3: the library picks the fastest of StragglAR / Ring / RHD by
    completion from the non-stragglers' start.  The baselines' costs
    are the oracle's Table-1 forms; StragglAR's ReduceScatter is
    this implementation's one direct-pull step (alpha + (n-2)/(n-1) s beta),
    which equals the oracle's ReduceScatter at alpha = 0."""
    beta = 1 / 770e9
    algo, t = S.stragglar_select_algorithm(n, nbytes, delay, alpha, beta)
    t_rs = alpha + (n - 2) / (n - 1) * nbytes * beta
    if alpha == 0.0:
        assert t_rs == pytest.approx(C.t_reduce_scatter(n - 1, nbytes, 0.0, beta), rel=1e-12)
    cand = {"stragglar": max(delay, t_rs) + C.t_stragglar(n, nbytes, alpha, beta),
            "ring": delay + C.t_ring(n, nbytes, alpha, beta),
            "rhd": delay + C.t_rhd(n, nbytes, alpha, beta)}
    best = min(cand.values())
    assert t == pytest.approx(best, rel=1e-12)
    assert cand[algo] == pytest.approx(best, rel=1e-12)
    order = ["stragglar", "ring", "rhd"]     # tie-break
    assert algo == next(a for a in order if cand[a] <= best * (1 + 1e-12))


def test_small_buffers_pick_rhd_large_delayed_pick_stragglar(S):
    """at small sizes the latency-optimal RHD wins; with a delay
    that masks the ReduceScatter and a large buffer StragglAR wins."""
    beta = 1 / 770e9
    assert S.stragglar_select_algorithm(8, 2 ** 20, 0.0, 3e-6, beta)[0] == "rhd"
    assert S.stragglar_select_algorithm(8, 2 ** 30, 2e-3, 3e-6, beta)[0] == "stragglar"
    assert S.stragglar_select_algorithm(6, 2 ** 20, 0.0, 3e-6, beta)[0] != "rhd"   # RHD needs a power of two
