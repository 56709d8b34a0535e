"""Pins for oracle/cost.py: Table 1 closed forms and §4.2's critical delay."""
import math

import pytest

from oracle import cost as C
from oracle import schedule as S

A, B = 3e-6, 1 / 450e9          # alpha = 3 us, beta = 1/(450 GB/s)
GiB = 2 ** 30


def test_spec_worked_numbers():
    """T_SAR(256, 1 GiB) ~ 3.24 ms, T_Ring ~ 6.28 ms, ratio ~ 1.94
    ('nearly 2x')."""
    sar = C.t_stragglar(256, GiB, A, B)
    ring = C.t_ring(256, GiB, A, B)
    assert sar == pytest.approx(3.24e-3, rel=5e-3)
    assert ring == pytest.approx(6.28e-3, rel=5e-3)
    assert ring / sar == pytest.approx(1.94, abs=0.02)


def test_spec_reduce_scatter_number():
    """ring RS among 7 ranks of 4 GiB ~ 8.20 ms; m = 1 costs 0."""
    assert C.t_reduce_scatter(7, 4 * GiB, A, B) == pytest.approx(8.20e-3, rel=5e-3)
    assert C.t_reduce_scatter(1, GiB, A, B) == 0.0


@pytest.mark.parametrize("n", [2, 4, 8, 16, 64, 256])
def test_schedule_cost_equals_table1(n):
    """rounds*alpha + beta_coef*s*beta of the generated schedule equals
    Table 1's closed form."""
    rep = S.verify_schedule(S.generate_stragglar(n))
    s = 123456789.0
    assert rep.rounds_executed * A + float(rep.beta_coefficient) * s * B == pytest.approx(C.t_stragglar(n, s, A, B), rel=1e-12)
    rr = S.verify_schedule(S.generate_ring(n))
    assert rr.rounds_executed * A + float(rr.beta_coefficient) * s * B == pytest.approx(C.t_ring(n, s, A, B), rel=1e-12)


def test_beta_limits_and_monotone_speedup():
    """StragglAR's beta coefficient -> 1, Ring's -> 2; the (alpha=0)
    speedup grows with n."""
    sp = [C.t_ring(n, 1.0, 0, 1) / C.t_stragglar(n, 1.0, 0, 1) for n in [4, 8, 16, 32, 64, 128, 256]]
    assert all(b > a for a, b in zip(sp, sp[1:]))
    assert C.t_stragglar(2 ** 20, 1.0, 0, 1) == pytest.approx(1.0, abs=1e-4)
    assert C.t_ring(2 ** 20, 1.0, 0, 1) == pytest.approx(2.0, abs=1e-5)
    assert sp[1] == pytest.approx(1.75 / (9 / 7))       # n = 8: 1.361 ideal gain


def test_critical_delay_identity_and_bound():
    """at the critical delay the end-to-end times tie;
    it is below T_RS (P:421-422 'almost 2x less than the RS runtime')."""
    n, s = 8, 4 * GiB
    tb = C.t_ring(n, s, A, B)
    d = C.critical_delay(n, s, A, B, tb)
    assert 0 < d < C.t_reduce_scatter(n - 1, s, A, B)
    assert C.end_to_end_stragglar(n, s, d, A, B) == pytest.approx(C.end_to_end_ring(n, s, d, A, B), rel=1e-12)
    lo, hi = 0.0, 1.0
    for _ in range(200):
        mid = (lo + hi) / 2
        if C.end_to_end_stragglar(n, s, mid, A, B) > C.end_to_end_ring(n, s, mid, A, B):
            lo = mid
        else:
            hi = mid
    assert hi == pytest.approx(d, rel=1e-9)


def test_zero_delay_stragglar_loses():
    """with no delay StragglAR pays the whole RS: at n=8 its beta is
    6/7 + 9/7 = 15/7 > Ring's 7/4."""
    s = GiB
    assert C.end_to_end_stragglar(8, s, 0.0, 0.0, 1.0) == pytest.approx((6 / 7 + 9 / 7) * s)
    assert C.end_to_end_stragglar(8, s, 0.0, 0.0, 1.0) > C.end_to_end_ring(8, s, 0.0, 0.0, 1.0)
