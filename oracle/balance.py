"""R²CCL-Balance: proportional redistribution over healthy channels.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:73 (§5.1): "when a NIC or link on server i fails, it redistributes the
portion of D_i that would have used the failed NIC across the remaining
healthy NICs in proportion to their available bandwidth."  P:80: "allowing
their combined throughput to approach B_i^rem".
(redistribute), S:472 (conservation: remainder to the highest-bandwidth NIC),
S:473 (monotonicity).

Reading C-15: split R units (16-byte vectors) as share_c = floor(R*w_c/Σw)
over the healthy channels, remainder to the highest weight (ties -> lowest id).
"""
from __future__ import annotations


class AllFailed(Exception):
    """S:456 'errors: all NICs failed'."""


def redistribute(R: int, weights: dict[int, int], failed: set[int] | frozenset = frozenset()) -> dict[int, int]:
    """Integer shares of R units over healthy channels, proportional to weight."""
    healthy = sorted(c for c in weights if c not in failed and weights[c] > 0)
    if not healthy:
        raise AllFailed("all channels failed")
    total = sum(weights[c] for c in healthy)
    shares = {c: (R * weights[c]) // total for c in healthy}
    rem = R - sum(shares.values())
    top = min(healthy, key=lambda c: (-weights[c], c))
    shares[top] += rem
    return shares


def part_ranges(R: int, weights: dict[int, int], failed=frozenset()) -> list[tuple[int, int, int]]:
    """Contiguous parts [lo, hi) of an R-vector item, laid out in channel-id
    order; channels with a zero share get no part.  -> [(channel, lo, hi)]."""
    shares = redistribute(R, weights, failed)
    out, lo = [], 0
    for c in sorted(shares):
        if shares[c] > 0:
            out.append((c, lo, lo + shares[c]))
            lo += shares[c]
    assert lo == R
    return out


def completion_ratio(weights: dict[int, int], failed: set[int]) -> float:
    """Ideal healthy/degraded makespan ratio for one server losing `failed`
    (P:80 'completion time is dictated primarily by the reduced capacity of
    the slowest server'): Σw / Σ_healthy w  (8/7 for one of 8 equal)."""
    tot = sum(weights.values())
    rem = sum(w for c, w in weights.items() if c not in failed)
    return tot / rem
