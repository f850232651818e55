"""Pins for oracle Layer 2 (oracle/protocol.py): the simulated fault-tolerant
ring allreduce must reproduce Layer 1 exactly under every fault point
(brute force on tiny inputs, S:740-741 / SURVEY §8(c)), the config-1 event
record, traffic accounting and the degraded-bandwidth model
(S:742-743).  CPU only."""
import itertools
import json
import os

import numpy as np
import pytest

import r2inputs
from oracle import semantic as S
from oracle.geometry import Geometry
from tests.scenario import effective_chunk_bytes
from oracle.protocol import BALANCE, HOT_REPAIR, Fault, simulate

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


def layer1(xs, g, dtype):
    return S.allreduce(xs, g.shard, dtype)


# ------------------------------------------------------------ fault-free

@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n,K,N", [(2, 1, 100), (3, 2, 1000), (4, 2, 4096), (5, 3, 777), (8, 8, 5000)])
def test_fault_free_equals_layer1(dtype, n, K, N):
    E = r2inputs.elem_bytes(dtype)
    g = Geometry(n, K, N, E, effective_chunk_bytes(N, n, K, E, 256, 2))
    xs = r2inputs.inputs(n, N, dtype, seed=n * 10 + K)
    y = layer1(xs, g, dtype)
    for seed in range(3):
        res = simulate(xs, g, dtype, seed=seed)
        assert res.error is None and not res.events
        for r in range(n):
            assert same(res.y[r], y)


@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
def test_inplace_fault_free(dtype):
    n, K, N = 4, 2, 999
    E = r2inputs.elem_bytes(dtype)
    g = Geometry(n, K, N, E, 64)
    xs = r2inputs.inputs(n, N, dtype, seed=4)
    res = simulate(xs, g, dtype, seed=1, inplace=True)
    y = layer1(xs, g, dtype)
    assert all(same(res.y[r], y) for r in range(n))


def test_traffic_accounting_fault_free():
    """each rank sends 2(n-1)/n of the (padded) buffer, split evenly over
    the K channels."""
    for n, K in [(2, 2), (3, 3), (4, 2), (8, 8)]:
        N = 3000
        g = Geometry(n, K, N, 4, 64)
        xs = r2inputs.inputs(n, N, "int32", seed=1)
        res = simulate(xs, g, "int32", seed=0)
        per_rank = res.bytes_sent.sum(axis=1)
        assert np.all(per_rank == 2 * (n - 1) * g.Np * 4 // n)
        assert np.all(res.bytes_sent == res.bytes_sent[0, 0])


# ------------------------------------------------------------ config 1

@pytest.mark.parametrize("dtype", ["int32", "float32"])
@pytest.mark.parametrize("strategy", [BALANCE, HOT_REPAIR])
def test_config1_event_record(dtype, strategy):
    c1 = GOLD["config1"]
    g = Geometry(c1["n"], c1["K"], c1["N"], 4, c1["chunk_bytes"])
    assert g.m == 8
    xs = r2inputs.inputs(c1["n"], c1["N"], dtype)
    f = Fault(**c1["fault"])
    res = simulate(xs, g, dtype, faults=[f], strategy=strategy, seed=5)
    y = layer1(xs, g, dtype)
    assert res.error is None
    assert all(same(res.y[r], y) for r in range(c1["n"]))
    (ev,) = res.events
    assert (ev["verdict"], ev["a"], ev["b"], ev["aux"]) == (c1["verdict"], c1["a"], c1["b"], c1["aux"])
    assert (ev["resume"], ev["floor"], ev["retransmit"]) == (c1["resume"], c1["floor"], c1["retransmit"])
    if strategy == HOT_REPAIR:
        assert (ev["assignee"], ev["chain_pos"]) == (c1["assignee"], 0)
    else:
        assert set(ev["shares"]) == {c1["assignee"]}       # K=2: Balance == HotRepair
    # traffic: fault-free bytes + the partial b bytes of the faulted chunk
    free = simulate(xs, g, dtype, seed=5)
    assert res.bytes_sent.sum() == free.bytes_sent.sum() + c1["fault"]["b"]


# ------------------------------------------------------------ brute force

def brute_cases(n, K, m, vec_per_chunk):
    steps = 2 * n - 2
    bs = sorted({0, (vec_per_chunk // 2) * 16, vec_per_chunk * 16 - 16})
    for r, c, t, j, b, kind in itertools.product(range(n), range(K), range(steps), range(m), bs,
                                                 ("LOCAL", "REMOTE", "LINK")):
        yield Fault(kind, r, c, t, j, b)


@pytest.mark.parametrize("n,K,m", [(2, 1, 1), (2, 2, 2), (3, 2, 1), (3, 3, 2), (4, 2, 2), (4, 3, 1)])
@pytest.mark.parametrize("strategy", [BALANCE, HOT_REPAIR])
def test_brute_force_single_fault(n, K, m, strategy):
    """Every (rank, channel, q, b, kind) at depth 1: buffers == fault-free, or
    NO_BACKUP exactly when the chain is exhausted (K = 1)."""
    dtype = "int32"
    vpc = 2
    N = n * K * m * vpc * 4
    g = Geometry(n, K, N, 4, vpc * 16)
    assert g.m == m
    xs = r2inputs.inputs(n, N, dtype, seed=n + 7 * K + m)
    y = layer1(xs, g, dtype)
    cnt = 0
    for i, f in enumerate(brute_cases(n, K, m, vpc)):
        res = simulate(xs, g, dtype, faults=[f], strategy=strategy, seed=i)
        cnt += 1
        if K == 1:
            assert res.error == "NO_BACKUP"
            continue
        assert res.error is None, f
        for r in range(n):
            assert same(res.y[r], y), (f, r)
        assert len(res.fired) == 1
    assert cnt > 0


@pytest.mark.parametrize("strategy", [BALANCE, HOT_REPAIR])
@pytest.mark.parametrize("n,K", [(3, 3), (4, 3), (2, 3)])
def test_brute_force_depth2_on_adopter(strategy, n, K):
    """A second fault on the adopting backup while it carries the residual
    (P:36 'If that NIC later fails ... moves to the next NIC'): buffers stay
    exact; both failovers are recorded."""
    dtype, m, vpc = "bfloat16", 2, 2
    E = 2
    N = n * K * m * vpc * 8
    g = Geometry(n, K, N, E, vpc * 16)
    xs = r2inputs.inputs(n, N, dtype, seed=3)
    y = layer1(xs, g, dtype)
    steps = 2 * n - 2
    i = 0
    for r, c, q1 in itertools.product(range(n), range(K), range(steps * m)):
        t1, j1 = divmod(q1, m)
        adopter = (c + 1) % K
        for q2 in range(q1, steps * m):
            t2, j2 = divmod(q2, m)
            f1 = Fault("LINK", r, c, t1, j1, 16)
            f2 = Fault("LINK", r, adopter, t2, j2, 0, origin=c)
            res = simulate(xs, g, dtype, faults=[f1, f2], strategy=strategy, seed=i)
            i += 1
            assert res.error is None, (f1, f2)
            assert all(same(res.y[rr], y) for rr in range(n))
            if len(res.fired) == 2:
                origins = sorted(ev["origin"] for ev in res.events)
                assert origins == sorted([c, c, adopter])
    assert i > 0


def test_no_backup_when_chain_exhausted():
    n, K, m = 3, 2, 2
    N = n * K * m * 8
    g = Geometry(n, K, N, 4, 32)
    xs = r2inputs.inputs(n, N, "int32", seed=1)
    f1 = Fault("LINK", 1, 0, 1, 0, 0)
    f2 = Fault("LINK", 1, 1, 1, 1, 0, origin=0)
    for strat in (BALANCE, HOT_REPAIR):
        res = simulate(xs, g, "int32", faults=[f1, f2], strategy=strat, seed=0)
        assert res.error == "NO_BACKUP"


@pytest.mark.parametrize("kind", ["LOCAL", "REMOTE", "LINK"])
@pytest.mark.parametrize("inplace", [False, True])
def test_random_interleavings_identical(kind, inplace):
    """Dependency-respecting interleavings never change the buffers."""
    n, K = 4, 3
    N = 5000
    g = Geometry(n, K, N, 2, 64)
    xs = r2inputs.inputs(n, N, "bfloat16", seed=8)
    y = layer1(xs, g, "bfloat16")
    for seed in range(12):
        f = Fault(kind, seed % n, seed % K, (seed * 5) % g.steps, seed % g.m, 32)
        res = simulate(xs, g, "bfloat16", faults=[f], seed=seed, inplace=inplace)
        assert res.error is None
        assert all(same(res.y[r], y) for r in range(n))


def test_local_fault_kills_both_connections_through_endpoint():
    """Reading C-14: a LOCAL verdict at (r, c) reroutes (r-1 -> r, c) too."""
    n, K = 4, 3
    N = 4000
    g = Geometry(n, K, N, 4, 64)
    xs = r2inputs.inputs(n, N, "float32", seed=2)
    res = simulate(xs, g, "float32", faults=[Fault("LOCAL", 2, 1, 0, 0, 16)], seed=3)
    assert res.error is None
    assert (2, 1) in res.health["dead_endpoints"]
    ranks = sorted({ev["rank"] for ev in res.events})
    assert 2 in ranks
    assert all(ev["verdict"] in ("LOCAL_ENDPOINT", "REMOTE_ENDPOINT") for ev in res.events)
    assert all(same(res.y[r], layer1(xs, g, "float32")) for r in range(n))


# ------------------------------------------------------------ degraded model

@pytest.mark.parametrize("strategy,ratio", [(BALANCE, 7 / 8), (HOT_REPAIR, 0.5)])
def test_degraded_plan_channel_load(strategy, ratio):
    """Plan-time placement with one dead channel of K=8 on one connection: the
    busiest channel carries 8/7 (Balance) or 2x (HotRepair) of a healthy
    channel's bytes -> ideal throughput ratio 7/8 resp. 1/2."""
    n, K = 4, 8
    N = n * K * 8 * 7 * 64
    g = Geometry(n, K, N, 4, 7 * 64 * 16)
    xs = r2inputs.inputs(n, N, "int32", seed=6)
    res = simulate(xs, g, "int32", strategy=strategy, health={"dead_links": [(1, 3)]}, seed=0)
    assert res.error is None
    assert all(same(res.y[r], layer1(xs, g, "int32")) for r in range(n))
    healthy_per_channel = res.bytes_sent[0, 0]
    assert res.bytes_sent[1, 3] == 0
    assert res.bytes_sent[1].sum() == res.bytes_sent[0].sum()
    assert healthy_per_channel / res.bytes_sent[1].max() == pytest.approx(ratio, rel=1e-3)


def test_n1_and_empty():
    g = Geometry(1, 2, 10, 4, 64)
    x = r2inputs.inputs(1, 10, "int32")
    assert same(simulate(x, g, "int32").y[0], x[0])
    g0 = Geometry(3, 2, 0, 4, 64)
    res = simulate([np.zeros(0, np.int32)] * 3, g0, "int32")
    assert res.error is None
