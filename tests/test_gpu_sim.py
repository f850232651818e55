"""Parity of the CUDA path (through the C ABI) with the oracle, in simulated-
rank mode: k ranks on one B200 in one cooperative kernel (the 1-GPU
"local reduce" configuration; ranks that wait on each other must not be
separate launches on one GPU).  Bit-exact for all dtypes;
failover records compared field by field with oracle Layer 2."""
import numpy as np
import pytest
import torch

import r2inputs
from oracle import protocol as OP
from oracle import semantic as OS
from tests.gpu_util import (check_result, norm_event, oracle_faults, oracle_geom, poisoned, run, same_bits,
                            sim_comm, to_dev, to_np)
from paper_2512_25059_b200 import build as B
from paper_2512_25059_b200 import r2ccl as R
from paper_2512_25059_b200 import torch_api as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def setup(cuda_required):
    B.build()
    torch.cuda.set_device(0)


_COMMS = {}


def healthy_comm(n, K=4, W=2, chunk=64 * 1024):
    key = (n, K, W, chunk)
    if key not in _COMMS:
        _COMMS[key] = sim_comm(n, K, W, chunk)
    return _COMMS[key]


# ------------------------------------------------------------ fault-free

@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("N", [1, 1000, 12345, (1 << 20) + 7])
def test_fault_free_parity(dtype, n, N):
    comm = healthy_comm(n)
    xs = r2inputs.inputs(n, N, dtype, seed=1000 + n)
    rc, out = run(comm, xs, dtype)
    assert rc == R.SUCCESS
    check_result(out, xs, oracle_geom(comm, N, dtype), dtype)


@pytest.mark.parametrize("dtype", ["int32", "bfloat16"])
@pytest.mark.parametrize("K,W,chunk", [(1, 1, 16), (2, 3, 4096), (8, 2, 512 * 1024), (3, 1, 48)])
def test_fault_free_configs(dtype, K, W, chunk):
    n, N = 4, 200_003
    comm = healthy_comm(n, K, W, chunk)
    xs = r2inputs.inputs(n, N, dtype, seed=77)
    rc, out = run(comm, xs, dtype)
    assert rc == R.SUCCESS
    check_result(out, xs, oracle_geom(comm, N, dtype), dtype)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_inplace_parity(dtype):
    n, N = 4, 300_001
    comm = healthy_comm(n)
    xs = r2inputs.inputs(n, N, dtype, seed=5)
    rc, out = run(comm, xs, dtype, inplace=True)
    assert rc == R.SUCCESS
    check_result(out, xs, oracle_geom(comm, N, dtype), dtype)


def test_many_calls_and_wrap_inputs():
    """Consecutive collectives alternate scratch parity; flags are seq-tagged."""
    n, N = 3, 100_000
    comm = healthy_comm(n)
    for i in range(7):
        xs = r2inputs.inputs(n, N, "int32", seed=i, dist="wrap")
        rc, out = run(comm, xs, "int32")
        assert rc == R.SUCCESS
        check_result(out, xs, oracle_geom(comm, N, "int32"), "int32")


def test_invalid_args():
    comm = healthy_comm(2)
    t = torch.zeros((2, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(R.R2Error) as e:
        comm.allreduce(t.data_ptr() + 4, t.data_ptr(), 10, R.FLOAT32)
    assert e.value.code == R.ERR_INVALID_ARG
    with pytest.raises(R.R2Error):
        comm.allreduce(t.data_ptr(), t.data_ptr(), (16 << 20), R.FLOAT32)
    comm.allreduce(t.data_ptr(), t.data_ptr(), 0, R.FLOAT32)  # no-op


def test_host_buffers():
    n, N = 4, 50_000
    comm = healthy_comm(n)
    xs = r2inputs.inputs(n, N, "float32", seed=9)
    send = torch.from_numpy(np.stack(xs)).pin_memory()
    recv = torch.empty_like(send).pin_memory()
    T.allreduce_host(comm, send, recv)
    assert comm.sync() == R.SUCCESS
    check_result(recv.numpy(), xs, oracle_geom(comm, N, "float32"), "float32")


def host_segments(count, E):
    """The pipelined host path's segmentation (r2ccl.h r2_allreduce_host)."""
    if count * E < (8 << 20):
        return [(0, count)]
    V = 16 // E
    nseg = min(8, max(1, count * E // (4 << 20)))
    seg = (count + nseg - 1) // nseg // V * V + V
    return [(lo, min(count, lo + seg)) for lo in range(0, count, seg)][:nseg]


@pytest.mark.parametrize("N", [(12 << 20) // 2 + 5, (9 << 20) // 2])
def test_host_buffers_segmented(N):
    """From 8 MiB on the host path is segmented and pipelined; every segment
    is its own collective: bit-exact against the oracle fold per segment
    (ragged rows: 2-D copies into packed per-segment stage rows)."""
    n, dt = 4, "bfloat16"
    comm = sim_comm(n, 4, 2, 64 * 1024, max_bytes=16 << 20)
    xs = r2inputs.inputs(n, N, dt, seed=17)
    row = -(-N // 8) * 8
    a = np.zeros((n, row), dtype=np.uint16)
    a[:, :N] = np.stack(xs)
    send = torch.from_numpy(a.view(np.int16)).pin_memory()
    recv = torch.empty_like(send).pin_memory()
    for _ in range(2):
        recv.fill_(-1)
        comm.allreduce_host(send.data_ptr(), recv.data_ptr(), N, R.BFLOAT16, torch.cuda.current_stream().cuda_stream)
        assert comm.sync() == R.SUCCESS
        torch.cuda.synchronize()
        out = recv.numpy().view(np.uint16)
        for lo, hi in host_segments(N, 2):
            g = oracle_geom(comm, hi - lo, dt)
            y = OS.allreduce([x[lo:hi] for x in xs], g.shard, dt)
            for r in range(n):
                assert same_bits(out[r, lo:hi], y), (lo, r)
        assert np.all(out[:, N:] == 0xFFFF)      # row padding untouched


# ------------------------------------------------------------ faults

def faulted(n, K, W, N, dtype, faults, strategy="BALANCE", chunk=64 * 1024, inplace=False, seed=3):
    comm = sim_comm(n, K, W, chunk, strategy=strategy)
    for f in faults:
        comm.inject_fault(at_seq=1, **f)
    xs = r2inputs.inputs(n, N, dtype, seed=seed)
    rc, out = run(comm, xs, dtype, inplace=inplace)
    g = oracle_geom(comm, N, dtype)
    return comm, xs, rc, out, g


def oracle_of(xs, g, dtype, faults, strategy, inplace=False):
    return OP.simulate(xs, g, dtype, faults=oracle_faults(faults), strategy=strategy, seed=1, inplace=inplace)


@pytest.mark.parametrize("dtype", ["int32", "float32"])
@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_config1_link_fault(dtype, strategy):
    """BASELINE configs[0]: 4 ranks, 1 MiB, K=2, 16 KiB chunks, LINK fault on
    (1 -> 2, ch 0) at t=1, j=3, b=8 KiB."""
    f = dict(kind="LINK", src_rank=1, channel=0, step=1, chunk=3, byte_offset=8192, poison=1)
    comm, xs, rc, out, g = faulted(4, 2, 1, 262144, dtype, [f], strategy, chunk=16384)
    assert rc == R.SUCCESS
    check_result(out, xs, g, dtype)
    ev = [norm_event(e) for e in comm.events()]
    want = [norm_event(e) for e in oracle_of(xs, g, dtype, [f], strategy).events]
    assert ev == want
    assert ev[0]["resume"] == 11 and ev[0]["retransmit"] == 37 and ev[0]["verdict"] == "LINK"
    assert comm.events()[0]["failover_ms"] > 0


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
@pytest.mark.parametrize("W", [1, 3])
@pytest.mark.parametrize("dtype", ["bfloat16", "int32"])
def test_link_fault_events_exact(strategy, W, dtype):
    n, K, N = 4, 4, 400_000
    f = dict(kind="LINK", src_rank=2, channel=1, step=2, chunk=1, byte_offset=5000, poison=1)
    comm, xs, rc, out, g = faulted(n, K, W, N, dtype, [f], strategy, chunk=16384)
    assert rc == R.SUCCESS
    check_result(out, xs, g, dtype)
    res = oracle_of(xs, g, dtype, [f], strategy)
    assert [norm_event(e) for e in comm.events()] == [norm_event(e) for e in res.events]
    st = comm.status()
    assert np.array_equal(np.array(st["bytes"])[:, :K], res.bytes_sent)


@pytest.mark.parametrize("kind", ["LOCAL", "REMOTE"])
@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_endpoint_faults(kind, strategy):
    n, K, N = 4, 3, 300_000
    f = dict(kind=kind, src_rank=1, channel=2, step=1, chunk=0, byte_offset=16 * 100, poison=1)
    comm, xs, rc, out, g = faulted(n, K, 2, N, "bfloat16", [f], strategy, chunk=8192)
    assert rc == R.SUCCESS
    check_result(out, xs, g, "bfloat16")
    evs = comm.events()
    prim = [e for e in evs if e["rank"] == 1 and e["origin"] == 2]
    assert len(prim) == 1
    want = "LOCAL_ENDPOINT" if kind == "LOCAL" else "REMOTE_ENDPOINT"
    assert prim[0]["verdict"] == want and prim[0]["resume"] == 1 * g.m + 0
    st = comm.status()
    dead_rank = 1 if kind == "LOCAL" else 2
    assert (dead_rank, 2) in st["dead_endpoints"]
    # both ring connections through the dead endpoint were re-placed (C-14)
    assert {e["rank"] for e in evs} == {dead_rank - 1, dead_rank}


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_successive_failover(strategy):
    """Config 4: a second fault on the adopting backup mid-retransmit."""
    n, K, N = 4, 4, 400_000
    f1 = dict(kind="LINK", src_rank=3, channel=1, step=1, chunk=2, byte_offset=4096)
    f2 = dict(kind="LINK", src_rank=3, channel=2, step=3, chunk=1, byte_offset=0, origin_channel=1)
    comm, xs, rc, out, g = faulted(n, K, 2, N, "bfloat16", [f1, f2], strategy, chunk=8192)
    assert rc == R.SUCCESS
    check_result(out, xs, g, "bfloat16")
    res = oracle_of(xs, g, "bfloat16", [f1, f2], strategy)
    assert len(res.fired) == 2
    got = sorted((norm_event(e) for e in comm.events()), key=lambda e: (e["stopped_channel"], e["origin"]))
    want = sorted((norm_event(e) for e in res.events), key=lambda e: (e["stopped_channel"], e["origin"]))
    # the first failover is deterministic: exact record
    assert [e for e in got if e["stopped_channel"] == 1] == [e for e in want if e["stopped_channel"] == 1]
    # the second depends on how far the adopter had got with its own items
    # when the adopted chunk failed (timing): same verdict and re-placed
    # origins, a consistent rollback (resume = floor + 1, residual <= rest)
    g2 = [e for e in got if e["stopped_channel"] == 2]
    w2 = [e for e in want if e["stopped_channel"] == 2]
    assert {e["origin"] for e in g2} == {e["origin"] for e in w2} == {1, 2}
    total = g.steps * g.m
    for e in g2:
        assert e["verdict"] == "LINK" and e["floor"] == e["resume"] - 1
        assert 0 <= e["retransmit"] <= total - e["resume"]
        if e["origin"] == 1:
            assert e["resume"] >= 1 * g.m + 2     # nothing before the first fault point re-opens


def test_no_backup_releases_stream():
    n, K, N = 3, 2, 100_000
    f1 = dict(kind="LINK", src_rank=1, channel=0, step=1, chunk=0, byte_offset=0)
    f2 = dict(kind="LINK", src_rank=1, channel=1, step=2, chunk=0, byte_offset=0, origin_channel=0)
    comm, xs, rc, out, g = faulted(n, K, 1, N, "int32", [f1, f2], "HOT_REPAIR", chunk=8192)
    assert rc == R.ERR_NO_BACKUP
    assert comm.status()["last_error"] == R.ERR_NO_BACKUP


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_degraded_static_plan_and_repair(strategy):
    """Later calls run a plan-time placement around the dead channel;
    REPAIR re-admits it."""
    n, K, N = 4, 4, 500_000
    f = dict(kind="LINK", src_rank=0, channel=3, step=0, chunk=0, byte_offset=0)
    comm, xs, rc, out, g = faulted(n, K, 2, N, "float32", [f], strategy, chunk=16384)
    assert rc == R.SUCCESS
    b0 = np.array(comm.status()["bytes"])[:, :K]
    xs2 = r2inputs.inputs(n, N, "float32", seed=42)
    rc, out = run(comm, xs2, "float32")
    assert rc == R.SUCCESS
    check_result(out, xs2, g, "float32")
    b1 = np.array(comm.status()["bytes"])[:, :K] - b0
    res = OP.simulate(xs2, g, "float32", strategy=strategy, health={"dead_links": [(0, 3)]}, seed=0)
    assert np.array_equal(b1, res.bytes_sent)
    comm.inject_fault(at_seq=comm.status()["seq"] + 1, kind="REPAIR", src_rank=0, channel=3)
    rc, out = run(comm, xs2, "float32")
    assert rc == R.SUCCESS and comm.status()["dead_links"] == []
    check_result(out, xs2, g, "float32")


def test_inplace_with_fault_in_fused_step():
    """A retransmitted final-add chunk must not read an overwritten input."""
    n, K, N = 4, 2, 200_000
    f = dict(kind="LINK", src_rank=2, channel=0, step=3, chunk=0, byte_offset=2048)
    comm, xs, rc, out, g = faulted(n, K, 2, N, "bfloat16", [f], "BALANCE", chunk=8192, inplace=True)
    assert rc == R.SUCCESS
    check_result(out, xs, g, "bfloat16")


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_periodic_faults_back_to_back(strategy):
    """Config-5 pattern in miniature: collectives enqueued back to back (no
    sync), a LINK fault every 12 calls, REPAIR of every (rank, channel) re-armed
    6 calls later while earlier collectives are still in flight.  Every result
    bit-exact; health records never change under a running kernel."""
    n, K, N, calls = 4, 4, 60_000, 72
    comm = sim_comm(n, K, 2, chunk_bytes=16384, strategy=strategy)
    pool = [r2inputs.inputs(n, N, "bfloat16", seed=s) for s in range(3)]
    g = oracle_geom(comm, N, "bfloat16")
    sends = [to_dev(x, "bfloat16") for x in pool]
    recvs = [poisoned(n, N, "bfloat16") for _ in range(calls)]
    rng = np.random.default_rng(17)
    for f in range(calls // 12):
        s = 1 + 12 * f
        comm.inject_fault(at_seq=s, kind="LINK", src_rank=int(rng.integers(n)), channel=int(rng.integers(K)),
                          step=int(rng.integers(g.steps)), chunk=int(rng.integers(g.m)), byte_offset=32)
        for r in range(n):
            for c in range(K):
                comm.inject_fault(at_seq=s + 6, kind="REPAIR", src_rank=r, channel=c)
    for i in range(calls):
        T.allreduce(comm, sends[i % 3], recvs[i], count=N)
    assert comm.sync() == R.SUCCESS
    for i in range(calls):
        check_result(to_np(recvs[i], "bfloat16")[:, :N], pool[i % 3], g, "bfloat16")
    assert len({e["seq"] for e in comm.events()}) == calls // 12


def test_probe_verdicts():
    comm = sim_comm(4, 4, 1)
    v = comm.probe(peer=2, channel=1, rank_local=1)
    assert v["verdict"] == "NONE" and v["outcomes"] == ("S", "S", "S", "S") and v["aux"] == 0
    f = dict(kind="LINK", src_rank=1, channel=1, step=0, chunk=0, byte_offset=0)
    comm.inject_fault(at_seq=1, **f)
    xs = r2inputs.inputs(4, 10_000, "int32", seed=1)
    rc, out = run(comm, xs, "int32")
    assert rc == R.SUCCESS
    v = comm.probe(peer=2, channel=1, rank_local=1)
    assert v["verdict"] == "LINK" and v["outcomes"] == ("T", "T", "S", "S")
    v = comm.probe(peer=3, channel=1, rank_local=2)
    assert v["verdict"] == "NONE"


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_brute_force_small(strategy):
    """Every (rank, channel, q) x kind on n=3, K=3, m=2 (one comm, REPAIR in
    between): buffers always bit-exact, LINK records exact."""
    n, K, W = 3, 3, 2
    comm = sim_comm(n, K, W, chunk_bytes=64, strategy=strategy)
    N = n * K * 2 * 16   # int32: 4 vectors per chunk -> m = 2
    xs = r2inputs.inputs(n, N, "int32", seed=123)
    g = oracle_geom(comm, N, "int32")
    assert g.m == 2
    for r in range(n):
        for c in range(K):
            for q in range(g.steps * g.m):
                for kind in ("LINK", "LOCAL", "REMOTE"):
                    t, j = divmod(q, g.m)
                    seq = comm.status()["seq"] + 1
                    f = dict(kind=kind, src_rank=r, channel=c, step=t, chunk=j, byte_offset=16, poison=1)
                    comm.inject_fault(at_seq=seq, **f)
                    ne = len(comm.events())
                    rc, out = run(comm, xs, "int32")
                    assert rc == R.SUCCESS, f
                    check_result(out, xs, g, "int32")
                    if kind == "LINK":
                        want = [norm_event(e) for e in oracle_of(xs, g, "int32", [f], strategy).events]
                        assert [norm_event(e) for e in comm.events()[ne:]] == want, f
                    # re-admit everything before the next case
                    for rr in range(n):
                        for cc in range(K):
                            comm.inject_fault(at_seq=seq + 1, kind="REPAIR", src_rank=rr, channel=cc)
                    rc, out = run(comm, xs, "int32")
                    assert rc == R.SUCCESS


# ------------------------------------------------------------ re-probe (f4)

def test_reprobe_readmits_after_heal():
    """P:19 periodic re-probe: a LINK-dead connection is re-probed with
    back-off; after the emulated fabric heals (HEAL, which the library is not
    told about) a re-probe finds A->B and B->A healthy and the connection is
    re-admitted from the next collective; results bit-exact throughout."""
    import time
    n, K, N = 4, 3, 60_000
    comm = sim_comm(n, K, 2, 8192, reprobe_us=300, reprobe_max_us=5000)
    xs = r2inputs.inputs(n, N, "int32", seed=31)
    g = oracle_geom(comm, N, "int32")
    comm.inject_fault(at_seq=1, kind="LINK", src_rank=1, channel=2, step=1, chunk=0, byte_offset=64)
    for _ in range(2):                       # faulted, then degraded
        rc, out = run(comm, xs, "int32")
        assert rc == R.SUCCESS
        check_result(out, xs, g, "int32")
    assert (1, 2) in comm.status()["dead_links"]
    time.sleep(0.03)                         # re-probes fail: still dead, backing off
    st = comm.status()
    assert st["n_reprobes"] >= 2 and st["n_readmits"] == 0 and (1, 2) in st["dead_links"]
    seq = st["seq"] + 1
    comm.inject_fault(at_seq=seq, kind="HEAL", src_rank=1, channel=2)
    rc, out = run(comm, xs, "int32")         # the fabric heals in stream order before this call
    assert rc == R.SUCCESS
    check_result(out, xs, g, "int32")
    deadline = time.time() + 2.0
    while comm.status()["n_readmits"] == 0 and time.time() < deadline:
        time.sleep(0.005)
    assert comm.status()["n_readmits"] == 1
    b0 = comm.status()["bytes"][1][2]
    rc, out = run(comm, xs, "int32")         # re-admitted from this collective on
    assert rc == R.SUCCESS
    check_result(out, xs, g, "int32")
    st = comm.status()
    assert st["dead_links"] == [] and st["bytes"][1][2] > b0


def test_reprobe_disabled_keeps_connection_dead():
    import time
    n, K, N = 3, 2, 30_000
    comm = sim_comm(n, K, 1, 8192, reprobe_us=0)
    xs = r2inputs.inputs(n, N, "int32", seed=32)
    comm.inject_fault(at_seq=1, kind="LINK", src_rank=0, channel=1, step=0, chunk=0, byte_offset=0)
    comm.inject_fault(at_seq=2, kind="HEAL", src_rank=0, channel=1)
    for _ in range(3):
        rc, out = run(comm, xs, "int32")
        assert rc == R.SUCCESS
    time.sleep(0.02)
    st = comm.status()
    assert st["n_reprobes"] == 0 and (0, 1) in st["dead_links"]


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_channel_bandwidth_model(strategy):
    """channel_gbps (channels as bandwidth units, r2ccl.h): paced lanes give the
    same bits and the same failover records as the unpaced path."""
    n, K, W, N = 4, 3, 2, 200_003
    comm = sim_comm(n, K, W, 16384, strategy=strategy, channel_gbps=20)
    f = dict(kind="LINK", src_rank=2, channel=1, step=2, chunk=1, byte_offset=5000, poison=1)
    comm.inject_fault(at_seq=1, **f)
    xs = r2inputs.inputs(n, N, "int32", seed=51)
    rc, out = run(comm, xs, "int32")
    assert rc == R.SUCCESS
    g = oracle_geom(comm, N, "int32")
    check_result(out, xs, g, "int32")
    res = OP.simulate(xs, g, "int32", faults=oracle_faults([f]), strategy=strategy, seed=1)
    assert [norm_event(e) for e in comm.events()] == [norm_event(e) for e in res.events]
    rc, out = run(comm, xs, "int32")          # degraded steady state, paced
    assert rc == R.SUCCESS
    check_result(out, xs, g, "int32")
