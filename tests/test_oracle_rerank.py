"""Pins for oracle/rerank.py -- Algorithm 1 (PAPER App. D, §6
P:726) -- and for the re-ranked ring's Layer-1 result: SPEC's worked
examples (tests/golden/worked_examples.json, cited), the properties SPEC
S:636-640 states (permutation, bottleneck never decreases, idempotence),
each relocation re-checked against the acceptance rule of lines 15-17, and
exact integer sums for any ring order.  CPU only."""
import itertools
import json
import os
import random

import numpy as np
import pytest

import r2inputs
from oracle import rerank as RR
from oracle import semantic as OS

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def rails_of(lst):
    return {u: frozenset(s) for u, s in enumerate(lst)}


@pytest.mark.parametrize("ex", GOLD["global_floor"], ids=lambda e: e["cite"][:8])
def test_global_floor_examples(ex):
    rails = rails_of(ex["rails"])
    assert RR.global_floor(list(rails), rails) == ex["expect"]


@pytest.mark.parametrize("ex", GOLD["rerank"], ids=lambda e: e["cite"][:8])
def test_rerank_worked_examples(ex):
    rails = rails_of(ex["rails"])
    B = RR.global_floor(ex["ring"], rails)
    assert B == ex["B_global"]
    assert [list(p) for p in RR.find_candidates(ex["ring"], RR.intersect_cap(rails), B)] == ex["candidates"]
    assert RR.rerank(ex["ring"], rails) == ex["expect"]


def test_candidates_sorted_by_gap():
    """two mismatched pairs with gaps 2 and 1 -> the larger gap first."""
    rails = rails_of([[0, 1, 2], [0, 1, 2], [0], [0, 1, 2], [1, 2], [0, 1, 2]])
    # B_global = 1; no pair below 1 -> use a floor of 3 through an explicit cap
    cap = RR.intersect_cap(rails)
    c = RR.find_candidates([0, 1, 2, 3, 4, 5], cap, 3)
    gaps = [3 - cap(u, v) for u, v in c]
    assert gaps == sorted(gaps, reverse=True) and gaps[0] == 2 and 1 in gaps


def random_case(rng, n, K, p_loss):
    rails = {}
    for u in range(n):
        s = frozenset(c for c in range(K) if rng.random() > p_loss)
        rails[u] = s if s else frozenset([rng.randrange(K)])
    order = list(range(n))
    rng.shuffle(order)
    return order, rails


def check_relocations(order, rails, cap):
    """Replay: R' differs from R only by relocations each of which met lines
    15-17 when it was made -- re-derived here from the input alone by a
    brute-force search over single relocations (independent of rerank)."""
    out = RR.rerank(order, rails, cap)
    assert sorted(out) == sorted(order)                      # S:636 permutation
    assert RR.min_adjacent_cap(out, cap) >= RR.min_adjacent_cap(order, cap)
    B = RR.global_floor(order, rails)
    cands = RR.find_candidates(order, cap, B)
    if not cands:
        assert out == list(order)
    # a candidate pair for which SOME w meets both conditions in the original
    # ring cannot be left with a sub-B edge between u and v unless an earlier
    # repair separated them
    n = len(order)
    for u, v in cands:
        ok_ws = []
        for w in order:
            if w in (u, v):
                continue
            i = order.index(w)
            if min(cap(u, w), cap(w, v)) >= B and cap(order[i - 1], order[(i + 1) % n]) >= B:
                ok_ws.append(w)
        j = out.index(u)
        if ok_ws and out[(j + 1) % n] == v and len(cands) == 1:
            raise AssertionError(f"pair {(u, v)} had a valid bridge {ok_ws} but stayed adjacent: {out}")
    return out


@pytest.mark.parametrize("seed", range(500))
def test_rerank_properties_random(seed):
    """500 random rail-failure patterns on 8-16 nodes."""
    rng = random.Random(seed)
    n = rng.randint(8, 16)
    order, rails = random_case(rng, n, 8, rng.choice([0.05, 0.15, 0.3]))
    cap = RR.intersect_cap(rails)
    out = check_relocations(order, rails, cap)
    # S:640 idempotence once no candidates are left
    if not RR.find_candidates(out, cap, RR.global_floor(out, rails)):
        assert RR.rerank(out, rails) == out


def test_rerank_brute_force_small():
    """Every rail assignment of n = 4 ranks over K = 2 channels (non-empty
    sets), identity ring: properties hold; a single disjoint pair is always
    repaired when the rest is healthy (a healthy node is a valid bridge)."""
    subsets = [frozenset(s) for k in (1, 2) for s in itertools.combinations(range(2), k)]
    for combo in itertools.product(subsets, repeat=4):
        rails = dict(enumerate(combo))
        check_relocations([0, 1, 2, 3], rails, RR.intersect_cap(rails))
    for n in (4, 5, 6):
        for a in range(n):
            b = (a + 1) % n
            rails = {u: frozenset(range(3)) for u in range(n)}
            rails[a], rails[b] = frozenset({0, 2}), frozenset({1, 2})
            cap = RR.intersect_cap(rails)
            out = RR.rerank(list(range(n)), rails)
            assert RR.min_adjacent_cap(out, cap) == 2, (n, a, out)


def test_link_capacity_bridges_dead_links():
    """Reading R-13: all links 1 -> 2 dead (every channel): the pair is
    bridged like an empty rail intersection; partly dead links leave the
    ring alone (Balance's case); without dead links link_cap ==
    intersect_cap."""
    n, K = 4, 3
    rails = {u: frozenset(range(K)) for u in range(n)}
    dead = {(1, 2, c) for c in range(K)}
    cap = RR.link_cap(rails, dead)
    assert RR.find_candidates([0, 1, 2, 3], cap, 3) == [(1, 2)]
    out = RR.rerank([0, 1, 2, 3], rails, cap)
    assert RR.min_adjacent_cap(out, cap) == 3 and out == [1, 0, 2, 3]
    part = RR.link_cap(rails, {(1, 2, c) for c in range(K - 1)})
    assert part(1, 2) == K and RR.rerank([0, 1, 2, 3], rails, part) == [0, 1, 2, 3]
    assert all(RR.link_cap(rails, set())(u, v) == RR.intersect_cap(rails)(u, v)
               for u in range(n) for v in range(n))


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_allreduce_ring_order(dtype):
    """P:726 ordering-agnostic: int32 results equal the wrapped big-int sum for
    every ring order; float results for the identity order equal the standard
    ring; every rank of a re-ranked fold holds one shard folded along R'."""
    n, N = 4, 4 * 8 * 3
    xs = r2inputs.inputs(n, N, dtype, seed=31)
    shard = N // n
    for order in itertools.permutations(range(n)):
        y = OS.allreduce_ring(xs, list(order), shard, dtype)
        if dtype == "int32":
            want = (sum(x.astype(np.int64) for x in xs) % (1 << 32)).astype(np.uint32).view(np.int32)
            assert np.array_equal(y, want)
    assert np.array_equal(OS.allreduce_ring(xs, list(range(n)), shard, dtype).view(np.uint8),
                          OS.allreduce(xs, shard, dtype).view(np.uint8))
    if dtype == "float32":
        # hand case, n = 3, shard 0 owned by position 0: fold x_{p1}, x_{p2}, x_{p0}
        a, b, c = np.float32(1e8), np.float32(-1e8), np.float32(1.0)
        xs3 = [np.array([v], np.float32) for v in (c, a, b)]     # rank 0: 1, rank 1: 1e8, rank 2: -1e8
        y_std = OS.allreduce_ring(xs3, [0, 1, 2], 1, dtype)       # (1e8 + -1e8) + 1 = 1
        y_rr = OS.allreduce_ring(xs3, [1, 0, 2], 1, dtype)        # shard 0 at rank 1: (1 + -1e8) + 1e8 = 0
        assert y_std[0] == np.float32(1.0) and y_rr[0] == np.float32(0.0)
