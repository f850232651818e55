"""Parity of the line protocols -- LL (reading R-6) and
LL128 (reading R-12), every test run for both -- through the C ABI,
simulated-rank mode: AllReduce / ReduceScatter /
AllGather results bit-exact against oracle Layer 1, failover records equal to
Layer 2 over the LL step list (oracle/geometry.py ll=True), the alpha-beta
selection picks LL for latency-bound sizes and SIMPLE for bandwidth-bound
ones."""
import numpy as np
import pytest
import torch

import r2inputs
from oracle import protocol as OP
from oracle import semantic as OS
from oracle.geometry import Geometry
from tests.scenario import effective_chunk_bytes
from tests.gpu_util import check_result, norm_event, oracle_faults, run, same_bits, sim_comm
from tests.test_gpu_rsag import check as check_op
from tests.test_gpu_rsag import inputs as op_inputs
from tests.test_gpu_rsag import run_op
from paper_2512_25059_b200 import build as B
from paper_2512_25059_b200 import r2ccl as R

pytestmark = pytest.mark.gpu

AR, RS, AG = "allreduce", "reduce_scatter", "all_gather"


@pytest.fixture(params=["LL", "LL128"])
def proto(request):
    return request.param


@pytest.fixture(scope="module", autouse=True)
def setup(cuda_required):
    B.build()
    torch.cuda.set_device(0)


_COMMS = {}


def ll_comm(n, K=4, W=2, chunk=64 * 1024, strategy="BALANCE", protocol="LL"):
    key = (n, K, W, chunk, strategy, protocol)
    if key not in _COMMS:
        _COMMS[key] = sim_comm(n, K, W, chunk, strategy=strategy, protocol=protocol)
    return _COMMS[key]


def geom(comm, op, N, dtype, ll=True):
    E = r2inputs.elem_bytes(dtype)
    K, W, ch = comm.cfg.nchannels, comm.cfg.ctas_per_channel, comm.cfg.chunk_bytes
    return Geometry(comm.n, K, N, E, effective_chunk_bytes(N, comm.n, K, E, ch, W, op), op, ll=ll)


def run_any(comm, op, xs, count, dtype):
    if op == AR:
        return run(comm, xs, dtype)
    return run_op(comm, op, xs, count, dtype)


def check_any(op, out, xs, count, dtype, g):
    if op == AR:
        check_result(out, xs, g, dtype)
    else:
        check_op(op, out, xs, count, dtype)


def xs_for(op, n, count, dtype, seed):
    return r2inputs.inputs(n, count, dtype, seed=seed) if op == AR else op_inputs(op, n, count, dtype, seed)


@pytest.mark.parametrize("op", [AR, RS, AG])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("count", [1, 999, 20_001])
def test_ll_fault_free_parity(op, dtype, n, count, proto):
    comm = ll_comm(n, protocol=proto)
    xs = xs_for(op, n, count, dtype, 3000 + n)
    rc, out = run_any(comm, op, xs, count, dtype)
    assert rc == R.SUCCESS
    assert comm.status()["last_protocol"] == proto
    check_any(op, out, xs, count, dtype, geom(comm, op, count, dtype))


def test_ll_inplace_allreduce_and_many_calls(proto):
    comm = ll_comm(4, protocol=proto)
    N, dtype = 50_003, "bfloat16"
    xs = r2inputs.inputs(4, N, dtype, seed=8)
    g = geom(comm, AR, N, dtype)
    for _ in range(5):      # back-to-back: lines of the previous collective carry older seqs
        rc, out = run(comm, xs, dtype, inplace=True)
        assert rc == R.SUCCESS
        check_result(out, xs, g, dtype)


@pytest.mark.parametrize("op", [AR, RS, AG])
@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
@pytest.mark.parametrize("dtype", ["bfloat16", "int32"])
def test_ll_link_fault_events_exact(op, strategy, dtype, proto):
    n, K, W, count = 4, 4, 2, 30_001
    comm = sim_comm(n, K, W, 4096, strategy=strategy, protocol=proto)
    f = dict(kind="LINK", src_rank=2, channel=1, step=1, chunk=1, byte_offset=1000, poison=1)
    comm.inject_fault(at_seq=1, **f)
    xs = xs_for(op, n, count, dtype, 5)
    rc, out = run_any(comm, op, xs, count, dtype)
    assert rc == R.SUCCESS
    g = geom(comm, op, count, dtype)
    check_any(op, out, xs, count, dtype, g)
    res = OP.simulate(xs, g, dtype, faults=oracle_faults([f]), strategy=strategy, seed=1)
    assert res.error is None
    assert [norm_event(e) for e in comm.events()] == [norm_event(e) for e in res.events]
    st = comm.status()
    assert np.array_equal(np.array(st["bytes"])[:, :K], res.bytes_sent)


@pytest.mark.parametrize("op", [AR, AG])
def test_ll_brute_force_small(op, proto):
    """Every (rank, channel, q) LINK fault on n=3, K=3, m=2 with the LL step
    list (the unpack step is LOCAL: never a fault point).  Under LL128 a
    4-vector chunk is one line, so Balance parts share it (whole-line writes)."""
    n, K, W = 3, 3, 2
    comm = sim_comm(n, K, W, chunk_bytes=64, strategy="BALANCE", protocol=proto)
    count = (n * K if op == AR else K) * 2 * 16
    xs = xs_for(op, n, count, "int32", 77)
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
                rc, out = run_any(comm, op, xs, count, "int32")
                assert rc == R.SUCCESS, f
                check_any(op, out, xs, count, "int32", g)
                want = [norm_event(e) for e in OP.simulate(xs, g, "int32", faults=oracle_faults([f]),
                                                           strategy="BALANCE", seed=1).events]
                assert [norm_event(e) for e in comm.events()[ne:]] == want, f
                comm.inject_fault(at_seq=seq + 1, kind="REPAIR", src_rank=r, channel=c)
                rc, out = run_any(comm, op, xs, count, "int32")
                assert rc == R.SUCCESS


def test_auto_selects_by_alpha_beta():
    """AUTO: LL for a latency-bound size, LL128 for a mid size, SIMPLE above
    the line scratch (ll_max_bytes); results bit-identical between protocols."""
    n = 4
    comm = sim_comm(n, 4, 2, 64 * 1024, max_bytes=64 << 20, protocol="AUTO", ll_max_bytes=16 << 20)
    simple = sim_comm(n, 4, 2, 64 * 1024, max_bytes=64 << 20, protocol="SIMPLE")
    for N, want in ((4096, "LL"), (4 << 20, "LL128"), (16 << 20, "SIMPLE")):
        xs = r2inputs.inputs(n, N, "bfloat16", seed=N)
        rc, out = run(comm, xs, "bfloat16")
        assert rc == R.SUCCESS and comm.status()["last_protocol"] == want, N
        rc2, out2 = run(simple, xs, "bfloat16")
        assert rc2 == R.SUCCESS and simple.status()["last_protocol"] == "SIMPLE"
        assert same_bits(out, out2)
        y = OS.allreduce(xs, geom(comm, AR, N, "bfloat16").shard, "bfloat16")
        assert same_bits(out[0], y)


def test_ll_too_large_is_invalid(proto):
    comm = sim_comm(2, 2, 1, 4096, max_bytes=1 << 20, protocol=proto, ll_max_bytes=4096)
    x = torch.zeros((2, 1 << 16), dtype=torch.float32, device="cuda")
    with pytest.raises(Exception):
        comm.allreduce(x.data_ptr(), x.data_ptr(), 1 << 16, R.FLOAT32)


def test_ll_no_backup_releases_stream(proto):
    """A chain exhausted mid-collective under LL: data warps spinning on lines
    that will never arrive are released by the abort; NO_BACKUP reported."""
    n, K, N = 3, 2, 30_000
    comm = sim_comm(n, K, 1, 8192, strategy="HOT_REPAIR", protocol=proto)
    comm.inject_fault(at_seq=1, kind="LINK", src_rank=1, channel=0, step=1, chunk=0, byte_offset=0)
    comm.inject_fault(at_seq=1, kind="LINK", src_rank=1, channel=1, step=2, chunk=0, byte_offset=0, origin_channel=0)
    xs = r2inputs.inputs(n, N, "int32", seed=1)
    rc, out = run(comm, xs, "int32")
    assert rc == R.ERR_NO_BACKUP
    # the communicator stays usable after the abort (fresh calls with the dead links are NO_BACKUP up front)
    assert comm.status()["last_error"] == R.ERR_NO_BACKUP


def test_ll_speculation_with_midcall_fault_many_points(proto):
    """Healthy static plan (speculative LL publishing) with a fault firing at
    several points of an AllReduce: bit-exact each time."""
    n, K, W, N = 4, 3, 2, 40_000
    comm = sim_comm(n, K, W, 4096, strategy="BALANCE", protocol=proto)
    xs = r2inputs.inputs(n, N, "bfloat16", seed=12)
    g = geom(comm, AR, N, "bfloat16")
    for t in range(0, g.steps - 1, 2):
        seq = comm.status()["seq"] + 1
        comm.inject_fault(at_seq=seq, kind="LINK", src_rank=t % n, channel=t % K, step=t, chunk=0, byte_offset=64,
                          poison=1)
        rc, out = run(comm, xs, "bfloat16")
        assert rc == R.SUCCESS, t
        check_result(out, xs, g, "bfloat16")
        comm.inject_fault(at_seq=seq + 1, kind="REPAIR", src_rank=t % n, channel=t % K)
        rc, out = run(comm, xs, "bfloat16")
        assert rc == R.SUCCESS


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_ll_inplace_with_fault(strategy, proto):
    """In-place AllReduce under LL with a mid-collective LINK fault in the fused
    final-add step (the staged own shard protects the overwritten input)."""
    n, K, W, N = 4, 3, 2, 40_003
    comm = sim_comm(n, K, W, 4096, strategy=strategy, protocol=proto)
    f = dict(kind="LINK", src_rank=1, channel=2, step=n - 1, chunk=1, byte_offset=512, poison=1)
    comm.inject_fault(at_seq=1, **f)
    xs = r2inputs.inputs(n, N, "bfloat16", seed=44)
    rc, out = run(comm, xs, "bfloat16", inplace=True)
    assert rc == R.SUCCESS
    g = geom(comm, AR, N, "bfloat16")
    check_result(out, xs, g, "bfloat16")
    res = OP.simulate(xs, g, "bfloat16", faults=oracle_faults([f]), strategy=strategy, seed=1, inplace=True)
    assert [norm_event(e) for e in comm.events()] == [norm_event(e) for e in res.events]


@pytest.mark.parametrize("step", [0, 2, 4])
def test_speculation_on_degraded_ring_with_midcall_fault(proto, step):
    """A statically degraded ring (rank 1 lost channel 1: Balance parts of one
    channel in other channels' lanes) speculates; a LOCAL fault at rank 2 in
    the middle of the call re-plans lanes that hold spinning items -- they are
    abandoned and re-issued (reading R-6), never a watchdog abort."""
    import time
    n, K, W, N = 4, 4, 2, 60_003
    comm = sim_comm(n, K, W, 4096, strategy="BALANCE", protocol=proto, rerank=0)
    s = comm.status()["seq"] + 1
    comm.inject_fault(at_seq=s, kind="LOCAL", src_rank=1, channel=1, step=0, chunk=0, byte_offset=0)
    xs0 = r2inputs.inputs(n, 4096, "int32", seed=1)
    rc, _ = run(comm, xs0, "int32")
    assert rc == R.SUCCESS
    t0 = time.time()
    while (1, 1) not in comm.status()["dead_endpoints"]:
        assert time.time() - t0 < 5
        time.sleep(0.002)
    xs = r2inputs.inputs(n, N, "bfloat16", seed=50 + step)
    g = geom(comm, AR, N, "bfloat16")
    s = comm.status()["seq"] + 1
    comm.inject_fault(at_seq=s, kind="LOCAL", src_rank=2, channel=2, step=step, chunk=0, byte_offset=512, poison=1)
    rc, out = run(comm, xs, "bfloat16")
    assert rc == R.SUCCESS
    assert comm.status()["last_protocol"] == proto
    check_result(out, xs, g, "bfloat16")
    comm.finalize()
