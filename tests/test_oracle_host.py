"""Pins for the oracle's host-logic pieces (rollback, chain, Balance,
triangulation, cost) against the worked examples SPEC/PAPER print
(tests/golden/worked_examples.json, each entry cited), exhaustive tables and
brute force.  CPU only."""
import itertools
import json
import os

import numpy as np

import r2inputs
import pytest

from oracle import balance as B
from oracle import cost as C
from oracle.geometry import Geometry
from oracle import ledger as L
from oracle import triangulation as T

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


# ------------------------------------------------------------ rollback / chain

@pytest.mark.parametrize("ex", GOLD["rollback"], ids=lambda e: e["cite"][:8])
def test_rollback_worked_examples(ex):
    done = [q in ex["completed"] for q in range(ex["chunks"])]
    assert L.rollback(done) == (ex["resume"], ex["floor"])
    assert L.residual(done) == ex["retransmit"]


def test_rollback_without_failure_raises():
    with pytest.raises(L.NoFailurePending):
        L.rollback([True, False], failure_pending=False)


def test_rollback_brute_force_invariants():
    """resume = floor + 1; every q < resume is complete; q = resume is not."""
    for k in range(0, 9):
        for mask in itertools.product([False, True], repeat=k):
            resume, floor = L.rollback(list(mask))
            assert resume == floor + 1
            assert all(mask[:resume])
            assert resume == k or not mask[resume]


@pytest.mark.parametrize("ex", GOLD["failover_chain"], ids=lambda e: e["cite"][:5])
def test_failover_chain_examples(ex):
    d = {int(k): v for k, v in ex["distances"].items()}
    assert L.failover_chain_by_distance(d) == ex["chain"]


@pytest.mark.parametrize("ex", GOLD["migrate"], ids=lambda e: e["cite"][:5])
def test_migrate_examples(ex):
    healthy = set(ex["chain"]) - set(ex["failed"])
    if ex["active"] is None:
        with pytest.raises(L.NoBackup):
            L.migrate(ex["chain"], healthy)
    else:
        assert L.migrate(ex["chain"], healthy)[0] == ex["active"]


def test_cyclic_chain_is_a_permutation_of_the_others():
    for K in range(1, 9):
        for c in range(K):
            ch = L.failover_chain(c, K)
            assert sorted(ch) == sorted(set(range(K)) - {c})
            assert ch[:1] == ([(c + 1) % K] if K > 1 else [])


# ------------------------------------------------------------ Balance

@pytest.mark.parametrize("ex", GOLD["redistribute"], ids=lambda e: e["cite"][:5])
def test_redistribute_examples(ex):
    w = dict(enumerate(ex["weights"]))
    got = B.redistribute(ex["R"], w, set(ex["failed"]))
    assert got == {int(k): v for k, v in ex["shares"].items()}
    if "ratio" in ex:
        assert B.completion_ratio(w, set(ex["failed"])) == pytest.approx(ex["ratio"])


def test_redistribute_all_failed():
    with pytest.raises(B.AllFailed):
        B.redistribute(10, {0: 1, 1: 1}, {0, 1})


def test_redistribute_conservation_and_proportionality():
    rng = np.random.default_rng(1)
    for _ in range(2000):
        K = int(rng.integers(1, 9))
        w = {c: int(rng.integers(1, 300)) for c in range(K)}
        failed = {c for c in range(K) if rng.random() < 0.3}
        if len(failed) == K:
            continue
        R = int(rng.integers(0, 100000))
        sh = B.redistribute(R, w, failed)
        assert sum(sh.values()) == R
        assert set(sh) == set(range(K)) - failed
        tot = sum(w[c] for c in sh)
        top = min(sh, key=lambda c: (-w[c], c))
        for c, s in sh.items():
            ideal = R * w[c] / tot
            assert ideal - 1 < s <= ideal + (len(sh) if c == top else 0)


def test_monotonic_in_the_real_valued_share():
    """failing another channel never decreases a remaining channel's
    proportional share (exactly true for R*w/Σw; the integer remainder rule of
    S:472 can move < K units, reading C-15 in DESIGN.md)."""
    rng = np.random.default_rng(2)
    for _ in range(500):
        K = int(rng.integers(2, 9))
        w = {c: int(rng.integers(1, 50)) for c in range(K)}
        R = int(rng.integers(1, 10 ** 6))
        f1 = {int(rng.integers(K))}
        f2 = f1 | {int(rng.integers(K))}
        if len(f2) == K or f2 == f1:
            continue
        s1 = B.redistribute(R, w, f1)
        s2 = B.redistribute(R, w, f2)
        for c in s2:
            assert s2[c] >= s1[c] - (K - 1)


def test_part_ranges_tile_the_item():
    for R in (1, 2, 7, 8, 100, 32768):
        parts = B.part_ranges(R, {c: 1 for c in range(8)}, {5})
        assert parts[0][1] == 0 and parts[-1][2] == R
        for a, b in zip(parts, parts[1:]):
            assert a[2] == b[1] and a[0] < b[0]


# ------------------------------------------------------------ triangulation

@pytest.mark.parametrize("ex", GOLD["triangulation"], ids=lambda e: e["cite"][:5])
def test_triangulation_named_rows(ex):
    assert T.triangulate(*ex["outcomes"]) == ex["verdict"]


def test_triangulation_total():
    """S:349 / S:744: every outcome combination maps to exactly one verdict."""
    seen = {}
    for ab, ba in itertools.product(T.OUTCOMES, repeat=2):
        seen[(ab, ba)] = T.triangulate(ab, ba)
    for ab, ba, xa, xb in itertools.product(T.OUTCOMES, repeat=4):
        seen[(ab, ba, xa, xb)] = T.triangulate(ab, ba, xa, xb)
    assert len(seen) == 9 + 81
    assert all(v in T.VERDICTS for v in seen.values())
    # aux rows never change a decision already taken by the endpoints
    for ab, ba in itertools.product(T.OUTCOMES, repeat=2):
        if (ab, ba) != ("T", "T"):
            for xa, xb in itertools.product(T.OUTCOMES, repeat=2):
                assert seen[(ab, ba, xa, xb)] == seen[(ab, ba)]


def test_triangulation_missing_aux_outcome():
    with pytest.raises(ValueError):
        T.triangulate("T", "T", "S", None)


@pytest.mark.parametrize("ex", GOLD["probe"], ids=lambda e: e["cite"][:5])
def test_probe_examples(ex):
    n, c = 3, 0
    ep = [[False], [False], [False]]
    link = [[False], [False], [False]]
    ep[0][0] = ex["prober_dead"]
    ep[1][0] = ex["target_dead"]
    link[0][0] = ex["link_dead"]
    assert T.probe(0, 1, c, n, ep, link) == ex["outcome"]


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_emulated_faults_localize(n):
    """Round for connection (A -> A+1) after each emulated fault kind gives the
    P:19 verdict (with aux for n >= 3; INCONCLUSIVE on a 2-ring link)."""
    K = 2
    for A in range(n):
        Bn = (A + 1) % n
        for kind in ("LOCAL", "REMOTE", "LINK"):
            ep = [[False] * K for _ in range(n)]
            link = [[False] * K for _ in range(n)]
            if kind == "LOCAL":
                ep[A][1] = True
            elif kind == "REMOTE":
                ep[Bn][1] = True
            else:
                link[A][1] = True
            rnd = T.run_round(A, Bn, 1, n, ep, link)
            want = {"LOCAL": T.LOCAL_ENDPOINT, "REMOTE": T.REMOTE_ENDPOINT,
                    "LINK": T.LINK if n >= 3 else T.INCONCLUSIVE}[kind]
            assert rnd["verdict"] == want
            assert rnd["aux"] == (None if n == 2 else min(set(range(n)) - {A, Bn}))


# ------------------------------------------------------------ cost / App. A

@pytest.mark.parametrize("ex", GOLD["cost"], ids=lambda e: e["cite"][:5])
def test_cost_examples(ex):
    got = getattr(C, ex["fn"])(*ex["args"])
    tol = ex.get("tol", 1e-12)
    if isinstance(ex["value"], list):
        assert got == pytest.approx(tuple(ex["value"]), abs=tol)
    else:
        assert got == pytest.approx(ex["value"], abs=tol)


def test_ystar_solves_t1_eq_t2_and_grid_argmin():
    """App. A Step 1 (T1(Y*) = T2(Y*)) and Step 3 (argmin) by brute force."""
    rng = np.random.default_rng(3)
    Y = np.linspace(0, 1, 10001)
    for _ in range(200):
        n, g = int(rng.integers(2, 65)), int(rng.integers(2, 9))
        th = C.threshold(n, g)
        X = float(rng.uniform(th + 1e-3, 0.99))
        ys = C.y_star(n, g, X)
        T1, T2, _ = C.stage_times(ys, n, g, X)
        assert T1 == pytest.approx(T2, rel=1e-9)
        tt = np.array([C.total_time(y, n, g, X) for y in Y])
        assert abs(Y[int(np.argmin(tt))] - C.optimal_partition(n, g, X)) <= 2e-3
        Xl = float(rng.uniform(1e-3, th))
        tl = np.array([C.total_time(y, n, g, Xl) for y in Y])
        assert np.all(tl[0] <= tl + 1e-12)


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_traffic_formulas_against_executed_schedule(n):
    """SURVEY §8(d) per-GPU traffic of the push ring ("must send
    (n-1)/n D_total ... must receive the same amount"): the closed forms
    2(n-1)/n S (NVLink) and (5n-4)/n S (HBM) equal the bytes the Layer-2
    simulator actually moves when it executes the schedule -- per rank, for
    every rank, with no padding (N a multiple of n*K*V)."""
    from oracle import protocol as OP
    K, E = 2, 4
    N = n * K * 4 * 16
    xs = r2inputs.inputs(n, N, "int32", seed=n)
    res = OP.simulate(xs, Geometry(n, K, N, E, 64), "int32", seed=1)
    S = N * E
    for r in range(n):
        assert res.bytes_sent[r].sum() == C.nvlink_bytes_per_gpu(S, n)
        assert res.hbm_bytes[r] == C.hbm_bytes_per_gpu(S, n)


def test_traffic_formulas_against_survey_table():
    """SURVEY §8(d)'s printed table at S = 256 MiB: NVLink per direction
    256 / 384 / 448 MiB and HBM total 768 / 1024 / 1152 MiB at n = 2 / 4 / 8."""
    S = 256 * 2 ** 20
    table = {2: (256, 768), 4: (384, 1024), 8: (448, 1152)}
    for n, (nv, hbm) in table.items():
        assert C.nvlink_bytes_per_gpu(S, n) == nv * 2 ** 20
        assert C.hbm_bytes_per_gpu(S, n) == hbm * 2 ** 20


@pytest.mark.parametrize("n", [2, 3, 5])
def test_reprobe_readmits_exactly_when_connection_healthy(n):
    """f4 (P:19 re-probe): for every emulated fabric state of one channel
    (each endpoint and each ring link alive or dead, brute force), the
    re-probe of (A -> A+1) re-admits iff both endpoints and the link A -> A+1
    are alive -- faults elsewhere (other ranks' endpoints, other links) never
    block re-admission and never fake it."""
    import itertools
    from oracle import triangulation as OT2
    K = 1
    for bits in itertools.product((False, True), repeat=2 * n):
        ep = [[bits[r]] for r in range(n)]
        ln = [[bits[n + r]] for r in range(n)]
        for a in range(n):
            b = (a + 1) % n
            want = not ep[a][0] and not ep[b][0] and not ln[a][0]
            if n == 2:   # the two ring links of a 2-ring join the same pair in opposite directions
                want = want and not ln[b][0]
            assert OT2.reprobe_readmits(a, b, 0, n, ep, ln) == want, (bits, a)
    assert K == 1
