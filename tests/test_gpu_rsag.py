"""Parity of the standalone ReduceScatter / AllGather
through the C ABI with the oracle, simulated-rank mode on one B200: results
bit-exact against Layer 1 (oracle/semantic.py reduce_scatter / all_gather) for
every dtype, ragged and unaligned shard strides, with and without faults;
failover records and per-channel bytes equal to Layer 2 (oracle/protocol.py
with op = reduce_scatter / all_gather)."""
import numpy as np
import pytest
import torch

import r2inputs
from oracle import protocol as OP
from oracle import semantic as OS
from oracle.geometry import Geometry
from tests.scenario import effective_chunk_bytes
from tests.gpu_util import TD, norm_event, oracle_faults, same_bits, sim_comm, to_np
from paper_2512_25059_b200 import build as B
from paper_2512_25059_b200 import r2ccl as R
from paper_2512_25059_b200 import torch_api as T

pytestmark = pytest.mark.gpu

RS, AG = "reduce_scatter", "all_gather"


@pytest.fixture(scope="module", autouse=True)
def setup(cuda_required):
    B.build()
    torch.cuda.set_device(0)


def rows(arrs, count, dtype, poison=False):
    """[k, roundup(count, V)] device tensor holding arrs (or poison)."""
    v = 16 // r2inputs.elem_bytes(dtype)
    L = max(-(-count // v) * v, v)
    if poison:
        t = torch.empty((len(arrs), L), dtype=TD[dtype], device="cuda")
        t.view(torch.uint8).fill_(0xFF)
        return t
    a = np.zeros((len(arrs), L), dtype=arrs[0].dtype)
    for i, x in enumerate(arrs):
        a[i, :len(x)] = x
    if dtype == "bfloat16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(a).cuda()


def geom(comm, op, count, dtype):
    E = r2inputs.elem_bytes(dtype)
    K, W, ch = comm.cfg.nchannels, comm.cfg.ctas_per_channel, comm.cfg.chunk_bytes
    return Geometry(comm.n, K, count, E, effective_chunk_bytes(count, comm.n, K, E, ch, W, op), op)


def inputs(op, n, count, dtype, seed):
    return r2inputs.inputs(n, n * count if op == RS else count, dtype, seed=seed)


def run_op(comm, op, xs, count, dtype):
    n = comm.n
    send = rows(xs, len(xs[0]), dtype)
    rcount = count if op == RS else n * count
    recv = rows([None] * n, rcount, dtype, poison=True)
    if op == RS:
        T.reduce_scatter(comm, send, recv, recvcount=count)
    else:
        T.all_gather(comm, send, recv, sendcount=count)
    rc = comm.sync()
    out = to_np(recv, dtype)
    if out.shape[1] > rcount:   # the row padding is never written
        assert np.all(out[:, rcount:].view(np.uint8) == 0xFF), "wrote past count"
    return rc, out[:, :rcount]


def expected(op, xs, count, dtype, n):
    if op == RS:
        return OS.reduce_scatter(xs, count, dtype)
    return [OS.all_gather(xs)] * n


def check(op, out, xs, count, dtype):
    want = expected(op, xs, count, dtype, out.shape[0])
    for r in range(out.shape[0]):
        if not same_bits(out[r], want[r]):
            bad = np.nonzero(out[r].view(np.uint8) != np.asarray(want[r]).view(np.uint8))[0]
            raise AssertionError(f"rank {r}: {len(bad)} bytes differ, first at byte {bad[:8]}")


_COMMS = {}


def comm_for(n, K=4, W=2, chunk=64 * 1024, strategy="BALANCE"):
    key = (n, K, W, chunk, strategy)
    if key not in _COMMS:
        _COMMS[key] = sim_comm(n, K, W, chunk, strategy=strategy)
    return _COMMS[key]


# ------------------------------------------------------------ fault-free

@pytest.mark.parametrize("op", [RS, AG])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("count", [1, 1000, 12347, (1 << 18) + 5])
def test_fault_free_parity(op, dtype, n, count):
    """Ragged counts: shard strides that are not a multiple of 16 bytes take
    the element-wise user-access path; padding of the channel split is never
    written."""
    comm = comm_for(n)
    xs = inputs(op, n, count, dtype, 2000 + n)
    rc, out = run_op(comm, op, xs, count, dtype)
    assert rc == R.SUCCESS
    check(op, out, xs, count, dtype)


@pytest.mark.parametrize("op", [RS, AG])
@pytest.mark.parametrize("K,W,chunk", [(1, 1, 16), (2, 3, 4096), (8, 2, 512 * 1024), (3, 1, 48)])
def test_fault_free_configs(op, K, W, chunk):
    n, count, dtype = 4, 50_001, "bfloat16"
    comm = comm_for(n, K, W, chunk)
    xs = inputs(op, n, count, dtype, 78)
    rc, out = run_op(comm, op, xs, count, dtype)
    assert rc == R.SUCCESS
    check(op, out, xs, count, dtype)


def test_rs_then_ag_is_allreduce():
    """AllGather(ReduceScatter(x)) == AllReduce(x), bit for bit, when the
    shard is a multiple of K*V (both geometries coincide)."""
    n, K, dtype = 4, 4, "bfloat16"
    comm = comm_for(n, K)
    count = K * 8 * 1000
    xs = inputs(RS, n, count, dtype, 5)
    rc, rs = run_op(comm, RS, xs, count, dtype)
    assert rc == R.SUCCESS
    rc, ag = run_op(comm, AG, list(rs), count, dtype)
    assert rc == R.SUCCESS
    y = OS.allreduce(xs, count, dtype)
    for r in range(n):
        assert same_bits(ag[r], y)


def test_invalid_args():
    comm = comm_for(4)
    x = torch.zeros((4, 64), dtype=torch.float32, device="cuda")
    with pytest.raises(Exception):
        comm.reduce_scatter(x.data_ptr(), x.data_ptr(), 16, R.FLOAT32)      # sim: out-of-place only
    with pytest.raises(Exception):
        comm.all_gather(x.data_ptr() + 4, x.data_ptr(), 16, R.FLOAT32)    # unaligned send row
    comm.reduce_scatter(x.data_ptr(), x.data_ptr(), 0, R.FLOAT32)          # count 0: no-op
    assert comm.sync() == R.SUCCESS


# ------------------------------------------------------------ faults

def faulted(op, n, K, W, count, dtype, faults, strategy, chunk=16384, seed=3):
    comm = sim_comm(n, K, W, chunk, strategy=strategy)
    for f in faults:
        comm.inject_fault(at_seq=1, **f)
    xs = inputs(op, n, count, dtype, seed)
    rc, out = run_op(comm, op, xs, count, dtype)
    return comm, xs, rc, out, geom(comm, op, count, dtype)


def oracle_of(op, xs, g, dtype, faults, strategy):
    return OP.simulate(xs, g, dtype, faults=oracle_faults(faults), strategy=strategy, seed=1)


@pytest.mark.parametrize("op", [RS, AG])
@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
@pytest.mark.parametrize("W", [1, 3])
@pytest.mark.parametrize("dtype", ["bfloat16", "int32"])
def test_link_fault_events_exact(op, strategy, W, dtype):
    n, K, count = 4, 4, 100_003
    step = 1 if op == RS else 2
    f = dict(kind="LINK", src_rank=2, channel=1, step=step, chunk=1, byte_offset=5000, poison=1)
    comm, xs, rc, out, g = faulted(op, n, K, W, count, dtype, [f], strategy)
    assert rc == R.SUCCESS
    check(op, out, xs, count, dtype)
    res = oracle_of(op, xs, g, dtype, [f], strategy)
    assert res.error is None
    assert [norm_event(e) for e in comm.events()] == [norm_event(e) for e in res.events]
    st = comm.status()
    assert np.array_equal(np.array(st["bytes"])[:, :K], res.bytes_sent)


@pytest.mark.parametrize("op", [RS, AG])
@pytest.mark.parametrize("kind", ["LOCAL", "REMOTE"])
def test_endpoint_faults(op, kind):
    n, K, count = 4, 3, 60_000
    f = dict(kind=kind, src_rank=1, channel=2, step=0, chunk=0, byte_offset=16 * 10, poison=1)
    comm, xs, rc, out, g = faulted(op, n, K, 2, count, "bfloat16", [f], "BALANCE", chunk=8192)
    assert rc == R.SUCCESS
    check(op, out, xs, count, "bfloat16")
    prim = [e for e in comm.events() if e["rank"] == 1 and e["origin"] == 2]
    assert len(prim) == 1 and prim[0]["resume"] == 0


def test_rs_fault_on_local_step_never_fires():
    """The ReduceScatter's final add uses no connection (reading R-5): a fault
    armed there is dropped, the call is healthy."""
    n, K, count = 4, 2, 10_000
    f = dict(kind="LINK", src_rank=0, channel=0, step=n - 1, chunk=0, byte_offset=16, poison=1)
    comm, xs, rc, out, g = faulted(RS, n, K, 2, count, "float32", [f], "BALANCE")
    assert rc == R.SUCCESS and comm.events() == []
    check(RS, out, xs, count, "float32")


@pytest.mark.parametrize("op", [RS, AG])
@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_brute_force_small(op, strategy):
    """Every (rank, channel, q) with a LINK fault on n=3, K=3, m=2: buffers
    bit-exact, records equal to the oracle's."""
    n, K, W = 3, 3, 2
    comm = sim_comm(n, K, W, chunk_bytes=64, strategy=strategy)
    count = K * 2 * 16          # int32: 4 vectors per chunk -> m = 2
    xs = inputs(op, n, count, "int32", 321)
    g = geom(comm, op, count, "int32")
    assert g.m == 2
    for r in range(n):
        for c in range(K):
            for q in range(g.steps * g.m):
                t, j = divmod(q, g.m)
                if g.local(t):
                    continue
                seq = comm.status()["seq"] + 1
                f = dict(kind="LINK", src_rank=r, channel=c, step=t, chunk=j, byte_offset=16, poison=1)
                comm.inject_fault(at_seq=seq, **f)
                ne = len(comm.events())
                rc, out = run_op(comm, op, xs, count, "int32")
                assert rc == R.SUCCESS, f
                check(op, out, xs, count, "int32")
                want = [norm_event(e) for e in oracle_of(op, xs, g, "int32", [f], strategy).events]
                assert [norm_event(e) for e in comm.events()[ne:]] == want, f
                comm.inject_fault(at_seq=seq + 1, kind="REPAIR", src_rank=r, channel=c)
                rc, out = run_op(comm, op, xs, count, "int32")
                assert rc == R.SUCCESS


# ------------------------------------------------------------ Broadcast (f1)

from oracle.geometry import BROADCAST  # noqa: E402


def run_bcast(comm, xs, count, dtype, root, inplace=False):
    n = comm.n
    send = rows(xs, count, dtype)
    recv = send if inplace else rows([None] * n, count, dtype, poison=True)
    from paper_2512_25059_b200 import torch_api as T2
    T2.broadcast(comm, send, recv, root, count=count)
    rc = comm.sync()
    out = to_np(recv, dtype)
    return rc, out[:, :count]


@pytest.mark.parametrize("dtype", ["int32", "bfloat16", "float32"])
@pytest.mark.parametrize("n,root", [(2, 1), (3, 0), (4, 2), (8, 5)])
@pytest.mark.parametrize("count", [1, 999, 100_003])
def test_broadcast_fault_free(dtype, n, root, count):
    comm = comm_for(n)
    xs = r2inputs.inputs(n, count, dtype, seed=n * 7 + root)
    rc, out = run_bcast(comm, xs, count, dtype, root)
    assert rc == R.SUCCESS
    for r in range(n):
        assert same_bits(out[r], xs[root]), r


def test_broadcast_inplace_root():
    comm = comm_for(4)
    xs = r2inputs.inputs(4, 50_001, "bfloat16", seed=3)
    rc, out = run_bcast(comm, xs, 50_001, "bfloat16", 1, inplace=True)
    assert rc == R.SUCCESS
    for r in range(4):
        assert same_bits(out[r], xs[1])


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
@pytest.mark.parametrize("root", [0, 2])
def test_broadcast_link_fault_events_exact(strategy, root):
    n, K, W, count = 4, 4, 2, 100_003
    comm = sim_comm(n, K, W, 16384, strategy=strategy)
    t = (1 - root) % n                       # rank 1's chain position: it sends there
    f = dict(kind="LINK", src_rank=1, channel=2, step=t, chunk=1, byte_offset=4000, poison=1)
    comm.inject_fault(at_seq=1, **f)
    xs = r2inputs.inputs(n, count, "int32", seed=11)
    rc, out = run_bcast(comm, xs, count, "int32", root)
    assert rc == R.SUCCESS
    for r in range(n):
        assert same_bits(out[r], xs[root])
    E = 4
    g = Geometry(n, K, count, E, effective_chunk_bytes(count, n, K, E, 16384, W, BROADCAST), BROADCAST, root=root)
    res = OP.simulate(xs, g, "int32", faults=oracle_faults([f]), strategy=strategy, seed=1)
    if t <= n - 2:
        assert [norm_event(e) for e in comm.events()] == [norm_event(e) for e in res.events]
        assert comm.events() and comm.events()[0]["resume"] == t * g.m + 1
    else:
        assert comm.events() == [] and res.events == []
    st = comm.status()
    assert np.array_equal(np.array(st["bytes"])[:, :K], res.bytes_sent)


@pytest.mark.parametrize("chunk", [16384, 512 * 1024])
def test_broadcast_at_max_bytes(chunk):
    """A Broadcast of exactly max_bytes (its one shard is n times an AllReduce
    shard, its chunks are capped at 128 KiB: the chunk table must hold it) --
    the bench's configuration."""
    n = 4
    comm = sim_comm(n, 8, 4, chunk, max_bytes=4 << 20)
    count = (4 << 20) // 4
    xs = r2inputs.inputs(n, count, "float32", seed=4)
    rc, out = run_bcast(comm, xs, count, "float32", 2)
    assert rc == R.SUCCESS
    for r in range(n):
        assert same_bits(out[r], xs[2])


def test_single_rank_degenerate_copies():
    """n = 1 (the degenerate case): every collective is a copy of the input."""
    comm = sim_comm(1, 2, 1, 4096)
    x = rows(r2inputs.inputs(1, 1001, "float32", seed=1), 1001, "float32")
    for fn in (lambda y: T.allreduce(comm, x, y, count=1001),
               lambda y: T.reduce_scatter(comm, x, y, recvcount=1001),
               lambda y: T.all_gather(comm, x, y, sendcount=1001),
               lambda y: T.broadcast(comm, x, y, 0, count=1001)):
        y = rows([None], 1001, "float32", poison=True)
        fn(y)
        assert comm.sync() == R.SUCCESS
        assert torch.equal(y[:, :1001], x[:, :1001])


@pytest.mark.parametrize("kind", ["LOCAL", "REMOTE"])
def test_broadcast_endpoint_faults(kind):
    """Endpoint faults on a Broadcast chain: the root's buffer still arrives
    everywhere bit for bit."""
    n, K, W, count, root = 4, 3, 2, 80_001, 1
    comm = sim_comm(n, K, W, 8192)
    src = 2                                   # chain position 1 for root 1
    f = dict(kind=kind, src_rank=src, channel=0, step=(src - root) % n, chunk=0, byte_offset=256, poison=1)
    comm.inject_fault(at_seq=1, **f)
    xs = r2inputs.inputs(n, count, "int32", seed=5)
    rc, out = run_bcast(comm, xs, count, "int32", root)
    assert rc == R.SUCCESS
    for r in range(n):
        assert same_bits(out[r], xs[root]), r
    assert any(e["rank"] == src for e in comm.events())
