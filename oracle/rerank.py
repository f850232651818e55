"""Topology-aware logical re-ranking: R²CCL's bridge-based repair of a ring
order (Algorithm 1, App. D; §6).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:726: "pairs of neighbors whose rail overlap falls below a bandwidth
threshold are separated by inserting 'bridge' nodes with broader rail
connectivity.  This targeted repair modifies only the problematic edges".

On the box (SURVEY C-1) a rail is a channel: S_u = the channels whose
endpoint on rank u is alive.  The capacity of the ring edge (u, v) is
|S_u ∩ S_v| exactly as in Algorithm 1; reading R-13 adds one
case: a neighbour pair with no live link left on any common channel has
capacity 0 (no direct path), so it is bridged like an empty rail
intersection -- the 2-hop relay through a proxy GPU at ring level.
Partly dead links leave the capacity |S_u ∩ S_v| (Balance handles them, as
for a single NIC failure); with no dead link the two are identical.

Readings (SURVEY C-19, SPEC S:643 vs S:632): the bridge scan visits
w ∈ R' \\ {u, v} in R' index order from position 0 (this reproduces SPEC's
hand trace S:632; "starting after v" would pick n3 there); PrevNode /
NextNode are evaluated in the current, already mutated R';
candidates are sorted by gap = B_global − cap descending, ties by ring
position ascending; a candidate pair that an earlier relocation has
already separated is skipped (Algorithm 1 leaves "between u, v" undefined
once they are not neighbours).
"""
from __future__ import annotations

from typing import Callable, Sequence


def global_floor(order: Sequence[int], rails: dict[int, frozenset]) -> int:
    """Algorithm 1 line 2: B_global <- min_{n in R} |S_n|."""
    if not order:
        raise ValueError("empty ring")
    return min(len(rails[u]) for u in order)


def intersect_cap(rails: dict[int, frozenset]) -> Callable[[int, int], int]:
    """|S_u ∩ S_v| (Algorithm 1 lines 5, 13, 14)."""
    return lambda u, v: len(rails[u] & rails[v])


def link_cap(rails: dict[int, frozenset], dead_links: set) -> Callable[[int, int], int]:
    """Reading R-13: |S_u ∩ S_v|, or 0 when the link u -> v is dead on every
    common channel; dead_links holds (u, v, c)."""
    def cap(u, v):
        common = rails[u] & rails[v]
        return len(common) if any((u, v, c) not in dead_links for c in common) else 0
    return cap


def find_candidates(order: Sequence[int], cap: Callable[[int, int], int], B: int) -> list[tuple[int, int]]:
    """Algorithm 1 lines 3-9: adjacent pairs (u, v) (wrapping) with
    cap(u, v) < B_global, sorted by severity (gap) descending, ties by ring
    position ascending."""
    n = len(order)
    cands = []
    for i in range(n):
        u, v = order[i], order[(i + 1) % n]
        c = cap(u, v)
        if c < B:
            cands.append((B - c, i, u, v))
    cands.sort(key=lambda e: (-e[0], e[1]))
    return [(u, v) for _, _, u, v in cands]


def rerank(order: Sequence[int], rails: dict[int, frozenset], cap: Callable[[int, int], int] | None = None) -> list[int]:
    """Algorithm 1, step by step.  Returns R'."""
    if cap is None:
        cap = intersect_cap(rails)
    R = list(order)                                   # line 1: R' <- R
    if len(R) < 3:
        return R
    B = global_floor(R, rails)                        # line 2
    for u, v in find_candidates(order, cap, B):       # lines 3-11 (candidates from R), line 11
        if not adjacent(R, u, v):
            continue                                  # an earlier relocation already separated u and v
        best = None                                   # line 12
        for w in list(R):                             # line 13: w in R' \ {u, v}, index order (C-19)
            if w in (u, v):
                continue
            i = R.index(w)
            x, y = R[i - 1], R[(i + 1) % len(R)]      # line 14: PrevNode / NextNode in R'
            new_cap = min(cap(u, w), cap(w, v))       # line 15
            removal_cap = cap(x, y)                   # line 16
            if new_cap >= B and removal_cap >= B:     # line 17
                best = w                              # line 18
                break                                 # line 19
        if best is not None:                          # line 22
            R.remove(best)                            # Relocate(best, between u, v): u, v stay adjacent
            j = R.index(u)
            R.insert(j + 1 if R[(j + 1) % len(R)] == v else j, best)
    return R


def adjacent(R: Sequence[int], u: int, v: int) -> bool:
    """u and v are ring neighbours in R (either direction)."""
    j = R.index(u)
    return R[(j + 1) % len(R)] == v or R[j - 1] == v


def min_adjacent_cap(order: Sequence[int], cap: Callable[[int, int], int]) -> int:
    """The ring's bottleneck edge (SPEC S:638 property)."""
    n = len(order)
    return min(cap(order[i], order[(i + 1) % n]) for i in range(n))
