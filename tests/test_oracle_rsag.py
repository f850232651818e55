"""Pins for the standalone ReduceScatter / AllGather of the oracle (SURVEY
§8(f) f1; "a ReduceScatter retains only a 1/n shard ... an AllGather
must receive the same amount"; P:94 ring AllReduce = ReduceScatter then
AllGather; P:353/572 R²CCL-Balance on both).

Layer 1 (oracle/semantic.py reduce_scatter / all_gather) is pinned to things
other than itself: the exact modular integer sum (closed form, independent of
the fold order), the composition AllGather(ReduceScatter(x)) == AllReduce(x)
(the AllReduce fold is pinned in test_oracle_semantic.py), and rank-tagged
inputs whose gathered layout is known by construction.  Layer 2
(oracle/protocol.py with op = reduce_scatter / all_gather) must reproduce
Layer 1 bit for bit under every single-fault point on tiny inputs (brute
force) and under random interleavings.  CPU only."""
import itertools

import numpy as np
import pytest

import r2inputs
from oracle import semantic as S
from oracle.geometry import ALL_GATHER, REDUCE_SCATTER, Geometry
from tests.scenario import effective_chunk_bytes
from oracle.protocol import BALANCE, HOT_REPAIR, Fault, simulate


def same(a, b):
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


def geom(op, n, K, N, dtype, chunk=256, W=2):
    E = r2inputs.elem_bytes(dtype)
    return Geometry(n, K, N, E, effective_chunk_bytes(N, n, K, E, chunk, W, op), op)


# ------------------------------------------------------------ Layer 1 pins

@pytest.mark.parametrize("n,count", [(2, 5), (3, 64), (4, 1000), (5, 7), (8, 33)])
def test_rs_int32_is_exact_modular_sum(n, count):
    """Integer addition is associative: every fold order gives the wrapped sum."""
    xs = r2inputs.inputs(n, n * count, "int32", seed=11 * n + count, dist="wrap")
    out = S.reduce_scatter(xs, count, "int32")
    tot = np.zeros(n * count, dtype=np.uint64)
    for x in xs:
        tot += np.asarray(x).view(np.uint32).astype(np.uint64)
    tot = (tot & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
    for r in range(n):
        assert np.array_equal(out[r], tot[r * count:(r + 1) * count]), r


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n,K", [(2, 1), (3, 2), (4, 8), (8, 8)])
def test_allgather_of_reducescatter_is_allreduce(dtype, n, K):
    """ring AllReduce = ReduceScatter followed by AllGather.  With the
    shard a multiple of K*V the two geometries coincide, so the bits agree."""
    V = 16 // r2inputs.elem_bytes(dtype)
    count = K * V * 5
    xs = r2inputs.inputs(n, n * count, dtype, seed=n * 3 + K)
    ar = S.allreduce(xs, count, dtype)
    rs = S.reduce_scatter(xs, count, dtype)
    assert same(S.all_gather(rs), ar)


def test_allgather_layout_rank_tagged():
    """Rank r's shard holds 1000*r + i: the gathered buffer is 1000*(i // c) + i % c."""
    n, c = 5, 13
    shards = [np.arange(c, dtype=np.int32) + 1000 * r for r in range(n)]
    y = S.all_gather(shards)
    i = np.arange(n * c)
    assert np.array_equal(y, (1000 * (i // c) + i % c).astype(np.int32))


def test_rs_fp32_within_error_bound():
    """Recursive summation bound: |fl(sum) - sum| <= (n-1) u sum|x_i| (u = 2^-24)."""
    n, count = 8, 4096
    xs = r2inputs.inputs(n, n * count, "float32", seed=5)
    out = S.reduce_scatter(xs, count, "float32")
    ex = S.exact_sum_f64(xs, "float32")
    absum = np.sum([np.abs(np.asarray(x, dtype=np.float64)) for x in xs], axis=0)
    for r in range(n):
        sl = slice(r * count, (r + 1) * count)
        err = np.abs(out[r].astype(np.float64) - ex[sl])
        assert np.all(err <= (n - 1) * 2.0 ** -24 * absum[sl] * (1 + 1e-6))


# ------------------------------------------------------------ Layer 2 pins

def run(op, xs, g, dtype, **kw):
    res = simulate(xs, g, dtype, **kw)
    return res


def expected(op, xs, g, dtype):
    if op == REDUCE_SCATTER:
        return S.reduce_scatter(xs, g.N, dtype)
    y = S.all_gather(xs)
    return [y] * g.n


def op_inputs(op, n, count, dtype, seed):
    return r2inputs.inputs(n, n * count if op == REDUCE_SCATTER else count, dtype, seed=seed)


@pytest.mark.parametrize("op", [REDUCE_SCATTER, ALL_GATHER])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n,K,count", [(2, 1, 100), (3, 2, 1000), (4, 2, 4096), (5, 3, 777), (8, 8, 5000)])
def test_fault_free_equals_layer1(op, dtype, n, K, count):
    g = geom(op, n, K, count, dtype)
    xs = op_inputs(op, n, count, dtype, n * 10 + K)
    want = expected(op, xs, g, dtype)
    for seed in range(2):
        res = run(op, xs, g, dtype, seed=seed)
        assert res.error is None and not res.events
        for r in range(n):
            assert same(res.y[r], want[r]), (seed, r)


@pytest.mark.parametrize("op", [REDUCE_SCATTER, ALL_GATHER])
@pytest.mark.parametrize("inplace", [False, True])
def test_inplace_and_traffic(op, inplace):
    n, K, count, dtype = 4, 2, 1000, "bfloat16"
    g = geom(op, n, K, count, dtype)
    xs = op_inputs(op, n, count, dtype, 3)
    want = expected(op, xs, g, dtype)
    res = run(op, xs, g, dtype, seed=1, inplace=inplace)
    for r in range(n):
        assert same(res.y[r], want[r])
    # each rank sends (n-1) shards (padded to the channel split) in either op
    sent = res.bytes_sent.sum(axis=1)
    assert np.all(sent == (n - 1) * g.shard * 2), sent


def brute(op, n, K, m, vpc, kinds=("LOCAL", "REMOTE", "LINK")):
    steps = n if op == REDUCE_SCATTER else n - 1     # AllGather and Broadcast: n - 1
    bs = sorted({0, (vpc // 2) * 16, vpc * 16 - 16})
    for r, c, t, j, b, kind in itertools.product(range(n), range(K), range(steps), range(m), bs, kinds):
        yield Fault(kind, r, c, t, j, b)


@pytest.mark.parametrize("op", [REDUCE_SCATTER, ALL_GATHER])
@pytest.mark.parametrize("n,K,m", [(2, 2, 2), (3, 2, 1), (3, 3, 2), (4, 2, 2)])
@pytest.mark.parametrize("strategy", [BALANCE, HOT_REPAIR])
def test_brute_force_single_fault(op, n, K, m, strategy):
    """Every (rank, channel, step, chunk, b, kind): buffers == Layer 1.  The
    ReduceScatter's final add (a LOCAL item) is never a fault point."""
    dtype = "int32"
    vpc = 2
    count = K * m * vpc * 4
    g = Geometry(n, K, count, 4, vpc * 16, op)
    assert g.m == m
    xs = op_inputs(op, n, count, dtype, n + 7 * K + m)
    want = expected(op, xs, g, dtype)
    fired = 0
    for i, f in enumerate(brute(op, n, K, m, vpc)):
        res = run(op, xs, g, dtype, faults=[f], strategy=strategy, seed=i)
        assert res.error is None, f
        for r in range(n):
            assert same(res.y[r], want[r]), (f, r)
        if op == REDUCE_SCATTER and f.t == n - 1:
            assert not res.fired and not res.events, f        # LOCAL item: no connection
        else:
            assert len(res.fired) == 1, f
            fired += 1
    assert fired > 0


@pytest.mark.parametrize("op", [REDUCE_SCATTER, ALL_GATHER])
def test_fault_event_matches_rollback_definition(op):
    """One LINK fault mid-chunk: the record's resume is the first stream
    position without a completion, floor = resume - 1, and the residual
    count includes the stopped worker's unfinished LOCAL items (reading R-5)."""
    n, K, dtype = 4, 2, "int32"
    count = K * 4 * 4 * 4
    g = Geometry(n, K, count, 4, 4 * 16, op)
    xs = op_inputs(op, n, count, dtype, 9)
    t = 1
    f = Fault("LINK", 2, 1, t, 2, 32)
    res = run(op, xs, g, dtype, faults=[f], seed=4)
    want = expected(op, xs, g, dtype)
    for r in range(n):
        assert same(res.y[r], want[r])
    ev = [e for e in res.events if e["origin"] == 1 and e["rank"] == 2]
    assert len(ev) == 1
    e = ev[0]
    assert e["verdict"] == "LINK"
    assert e["resume"] == t * g.m + 2 and e["floor"] == e["resume"] - 1
    assert e["retransmit"] == g.steps * g.m - e["resume"]


@pytest.mark.parametrize("op", [REDUCE_SCATTER, ALL_GATHER])
@pytest.mark.parametrize("strategy", [BALANCE, HOT_REPAIR])
def test_static_degraded_plan(op, strategy):
    """A connection known dead before the call: plan-time re-placement, the
    result is unchanged and the dead channel carries nothing."""
    n, K, count, dtype = 4, 3, 3 * 8 * 6, "float32"
    g = geom(op, n, K, count, dtype, chunk=64)
    xs = op_inputs(op, n, count, dtype, 21)
    res = run(op, xs, g, dtype, strategy=strategy, seed=2, health={"dead_links": [(1, 2)]})
    want = expected(op, xs, g, dtype)
    for r in range(n):
        assert same(res.y[r], want[r])
    assert res.bytes_sent[1, 2] == 0


# ------------------------------------------------------------ LL protocol (f3)

@pytest.mark.parametrize("op", ["allreduce", REDUCE_SCATTER, ALL_GATHER])
def test_ll_geometry_adds_unpack_step(op):
    """Reading R-6: LL adds one LOCAL unpack step to AllReduce / AllGather; the
    ReduceScatter already ends in a LOCAL final add."""
    n, K, count = 4, 2, 1000
    g0 = Geometry(n, K, count, 4, 256, op)
    g1 = Geometry(n, K, count, 4, 256, op, ll=True)
    extra = 0 if op == REDUCE_SCATTER else 1
    assert g1.steps == g0.steps + extra
    assert [t for t in range(g1.steps) if g1.local(t)] == [g1.steps - 1]


@pytest.mark.parametrize("op", ["allreduce", REDUCE_SCATTER, ALL_GATHER])
@pytest.mark.parametrize("strategy", [BALANCE, HOT_REPAIR])
def test_ll_brute_force_single_fault(op, strategy):
    """The LL step list under every single fault point: buffers == Layer 1;
    unpack items are never fault points and are re-placed with the residual."""
    n, K, m, vpc = 3, 3, 2, 2
    count = (n * K if op == "allreduce" else K) * m * vpc * 4
    g = Geometry(n, K, count, 4, vpc * 16, op, ll=True)
    assert g.m == m
    xs = (r2inputs.inputs(n, count, "int32", seed=99) if op == "allreduce" else op_inputs(op, n, count, "int32", 99))
    want = [S.allreduce(xs, g.shard, "int32")] * n if op == "allreduce" else expected(op, xs, g, "int32")
    for i, (r, c, t, j) in enumerate(itertools.product(range(n), range(K), range(g.steps), range(m))):
        f = Fault("LINK", r, c, t, j, 16)
        res = run(op, xs, g, "int32", faults=[f], strategy=strategy, seed=i)
        assert res.error is None, f
        for rr in range(n):
            assert same(res.y[rr], want[rr]), (f, rr)
        assert (len(res.fired) == 0) == g.local(t), f


# ------------------------------------------------------------ Broadcast (f1)

from oracle.geometry import BROADCAST  # noqa: E402


def test_broadcast_layer1_rank_tagged():
    """Every rank receives the root's buffer: rank-tagged inputs."""
    xs = [np.arange(11, dtype=np.int32) + 100 * r for r in range(5)]
    for root in range(5):
        for r, y in enumerate(S.broadcast(xs, root)):
            assert np.array_equal(y, np.arange(11, dtype=np.int32) + 100 * root)


@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
@pytest.mark.parametrize("n,K,count,root", [(2, 1, 100, 1), (3, 2, 1000, 0), (4, 3, 4097, 2), (8, 8, 5000, 5)])
@pytest.mark.parametrize("inplace", [False, True])
def test_broadcast_fault_free(dtype, n, K, count, root, inplace):
    E = r2inputs.elem_bytes(dtype)
    g = Geometry(n, K, count, E, effective_chunk_bytes(count, n, K, E, 256, 2, BROADCAST), BROADCAST, root=root)
    xs = r2inputs.inputs(n, count, dtype, seed=n + root)
    res = simulate(xs, g, dtype, seed=3, inplace=inplace)
    assert res.error is None
    for r in range(n):
        assert same(res.y[r], xs[root]), r
    # every rank but the last of the chain sends the (padded) buffer once
    sent = res.bytes_sent.sum(axis=1)
    last = (root - 1) % n
    for r in range(n):
        assert sent[r] == (0 if r == last else g.shard * E), (r, sent)


@pytest.mark.parametrize("n,K,m", [(3, 2, 2), (4, 3, 1), (4, 2, 2)])
@pytest.mark.parametrize("strategy", [BALANCE, HOT_REPAIR])
def test_broadcast_brute_force_single_fault(n, K, m, strategy):
    """Every (rank, channel, step, chunk, kind) fault: buffers == root's; a
    fault at a step where the rank does not send never fires."""
    vpc = 2
    count = K * m * vpc * 4
    for root in (0, n - 1):
        g = Geometry(n, K, count, 4, vpc * 16, BROADCAST, root=root)
        assert g.m == m
        xs = r2inputs.inputs(n, count, "int32", seed=root + 7)
        for i, f in enumerate(brute(BROADCAST, n, K, m, vpc)):
            res = run(BROADCAST, xs, g, "int32", faults=[f], strategy=strategy, seed=i)
            assert res.error is None, f
            for r in range(n):
                assert same(res.y[r], xs[root]), (f, r)
            assert (len(res.fired) == 1) == g.active(f.rank, f.t), f
