"""alpha-beta cost model — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:114-121 (§3): a message of s bytes costs alpha + s*beta; alpha counts rounds,
beta counts sequential bytes.  Table 1 gives the closed forms;
§4.2 gives the critical-delay condition.
"""
from __future__ import annotations

import math


def _log2(n: int) -> int:
    L = int(round(math.log2(n)))
    if 2 ** L != n:
        raise ValueError("power-of-2 n required")
    return L


def t_stragglar(n: int, s: float, alpha: float, beta: float) -> float:
    """T_SAR = (n + log n - 2) alpha + (n + log n - 2)/(n-1) s beta."""
    R = n + _log2(n) - 2
    return R * alpha + R / (n - 1) * s * beta


def t_ring(n: int, s: float, alpha: float, beta: float) -> float:
    """P:361 / Table 1: 2(n-1) alpha + 2(n-1)/n s beta."""
    return 2 * (n - 1) * alpha + 2 * (n - 1) / n * s * beta


def t_rhd(n: int, s: float, alpha: float, beta: float) -> float:
    """P:366 / Table 1: 2 log n alpha + 2(n-1)/n s beta."""
    return 2 * _log2(n) * alpha + 2 * (n - 1) / n * s * beta


def t_broadcast(n: int, s: float, alpha: float, beta: float) -> float:
    """log n alpha + log n s beta."""
    L = _log2(n)
    return L * alpha + L * s * beta


def t_reduce_scatter(m: int, s: float, alpha: float, beta: float) -> float:
    """Ring ReduceScatter among m ranks (the Ring's first half):
    (m-1) alpha + (m-1)/m s beta; m = 1 costs nothing."""
    if m <= 1:
        return 0.0
    return (m - 1) * alpha + (m - 1) / m * s * beta


def critical_delay(n: int, s: float, alpha: float, beta: float, t_baseline: float) -> float:
    """StragglAR beats baseline B iff T_delay >= T_RS - max{T_B - T_SAR, 0}."""
    t_rs = t_reduce_scatter(n - 1, s, alpha, beta)
    return max(t_rs - max(t_baseline - t_stragglar(n, s, alpha, beta), 0.0), 0.0)


def end_to_end_stragglar(n: int, s: float, delay: float, alpha: float, beta: float) -> float:
    """Measured from the non-stragglers' start: max(delay, T_RS) + T_SAR."""
    return max(delay, t_reduce_scatter(n - 1, s, alpha, beta)) + t_stragglar(n, s, alpha, beta)


def end_to_end_ring(n: int, s: float, delay: float, alpha: float, beta: float) -> float:
    """Bulk-synchronous Ring waits for the straggler: delay + T_Ring."""
    return delay + t_ring(n, s, alpha, beta)
