"""Topology-aware logical re-ranking on the GPU (Algorithm 1,
PAPER.md App. D :528-563, §6 :726; readings C-19, R-13),
simulated ranks on one B200, through the C ABI: after disjoint endpoint
losses on neighbouring ranks (and after every link of a ring neighbour pair
died) the planner runs the next AllReduce on oracle.rerank's R', the result
is bit-exact against oracle.semantic.allreduce_ring over R', and a fault
inside a collective on the re-ranked ring is recovered bit-exact."""
import time

import pytest
import torch

import r2inputs
from oracle import rerank as ORR
from oracle import semantic as OS
from oracle.geometry import Geometry
from tests.gpu_util import poisoned, same_bits, sim_comm, to_dev, to_np
from tests.scenario import effective_chunk_bytes
from paper_2512_25059_b200 import build as B
from paper_2512_25059_b200 import r2ccl as R
from paper_2512_25059_b200 import torch_api as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def setup(cuda_required):
    B.build()
    torch.cuda.set_device(0)


def kill(comm, kind, f, c, key, ok=(R.SUCCESS,)):
    """A LOCAL (endpoint) or LINK fault mid-collective, triangulated by the
    monitor; the verdict applies from the next collective on."""
    n = comm.n
    s = comm.status()["seq"] + 1
    comm.inject_fault(at_seq=s, kind=kind, src_rank=f, channel=c, step=0, chunk=0, byte_offset=0)
    xs = r2inputs.inputs(n, 4096, "int32", seed=c)
    T.allreduce(comm, to_dev(xs, "int32"), poisoned(n, 4096, "int32"), count=4096)
    assert comm.sync() in ok
    t0 = time.time()
    while (f, c) not in comm.status()[key]:
        assert time.time() - t0 < 5, "verdict not applied"
        time.sleep(0.002)


def run_ar(comm, xs, dtype):
    n, N = len(xs), len(xs[0])
    send = to_dev(xs, dtype)
    recv = poisoned(n, N, dtype)
    T.allreduce(comm, send, recv, count=N)
    rc = comm.sync()
    return rc, to_np(recv, dtype)[:, :N]


def expected_order(comm):
    st = comm.status()
    n, K = comm.n, comm.K
    rails = {u: frozenset(c for c in range(K) if (u, c) not in st["dead_endpoints"]) for u in range(n)}
    dead = {(r, (r + 1) % n, c) for r, c in st["dead_links"]}
    return ORR.rerank(list(range(n)), rails, ORR.link_cap(rails, dead))


def shard_of(comm, N, dtype, proto):
    E = r2inputs.elem_bytes(dtype)
    K, W, ch = comm.cfg.nchannels, comm.cfg.ctas_per_channel, comm.cfg.chunk_bytes
    return Geometry(comm.n, K, N, E, effective_chunk_bytes(N, comm.n, K, E, ch, W),
                    ll=proto in ("LL", "LL128")).shard


@pytest.mark.parametrize("protocol", ["SIMPLE", "LL"])
@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_disjoint_endpoint_losses_rerank(dtype, protocol):
    """Rank 1 loses channel 1, rank 2 loses channel 2 ("node u loses rail
    r while neighbor v loses rail r'"): the edge 1 -> 2 keeps 2 of 4 channels,
    B_global = 3, Algorithm 1 bridges it with rank 0 -> R' = [1, 0, 2, 3]."""
    n, K = 4, 4
    comm = sim_comm(n, K=K, W=2, chunk_bytes=16 * 1024, max_bytes=16 << 20, protocol=protocol)
    kill(comm, "LOCAL", 1, 1, "dead_endpoints")
    kill(comm, "LOCAL", 2, 2, "dead_endpoints")
    want = expected_order(comm)
    assert want == [1, 0, 2, 3]
    for N in (1, 777, 100_003):
        xs = r2inputs.inputs(n, N, dtype, seed=N)
        rc, out = run_ar(comm, xs, dtype)
        assert rc == R.SUCCESS
        st = comm.status()
        assert st["ring_order"] == want and st["n_rerank"] >= 1
        y = OS.allreduce_ring(xs, want, shard_of(comm, N, dtype, st["last_protocol"]), dtype)
        for r in range(n):
            assert same_bits(out[r], y), (N, r)
    comm.finalize()


def test_rerank_disabled_keeps_rank_order():
    n, K = 4, 4
    comm = sim_comm(n, K=K, W=2, chunk_bytes=16 * 1024, max_bytes=16 << 20, rerank=0)
    kill(comm, "LOCAL", 1, 1, "dead_endpoints")
    kill(comm, "LOCAL", 2, 2, "dead_endpoints")
    xs = r2inputs.inputs(n, 50_001, "bfloat16", seed=3)
    rc, out = run_ar(comm, xs, "bfloat16")
    assert rc == R.SUCCESS and comm.status()["ring_order"] == [0, 1, 2, 3]
    y = OS.allreduce(xs, shard_of(comm, 50_001, "bfloat16", "SIMPLE"), "bfloat16")
    assert all(same_bits(out[r], y) for r in range(n))
    comm.finalize()


@pytest.mark.parametrize("strategy", ["BALANCE", "HOT_REPAIR"])
def test_fault_on_reranked_ring(strategy):
    """A LINK-free endpoint fault inside a collective that runs on R' (rank 3
    loses channel 0 mid-call): recovered bit-exact against the R' fold."""
    n, K, N, dtype = 5, 4, 200_003, "bfloat16"
    comm = sim_comm(n, K=K, W=2, chunk_bytes=16 * 1024, max_bytes=16 << 20, strategy=strategy)
    kill(comm, "LOCAL", 1, 1, "dead_endpoints")
    kill(comm, "LOCAL", 2, 2, "dead_endpoints")
    order = expected_order(comm)
    assert order != list(range(n))
    xs = r2inputs.inputs(n, N, dtype, seed=11)
    s = comm.status()["seq"] + 1
    comm.inject_fault(at_seq=s, kind="LOCAL", src_rank=3, channel=0, step=2, chunk=1, byte_offset=4096, poison=1)
    rc, out = run_ar(comm, xs, dtype)
    assert rc == R.SUCCESS
    assert comm.status()["ring_order"] == order
    y = OS.allreduce_ring(xs, order, shard_of(comm, N, dtype, "SIMPLE"), dtype)
    assert all(same_bits(out[r], y) for r in range(n))
    comm.finalize()


def test_all_links_of_a_pair_dead_relay_by_rerank():
    """Reading R-13: every channel's link 1 -> 2 dies (successive LINK faults).
    While one link is left the ring stays (Balance carries the pair); when
    the last dies (that collective's chain is exhausted: NO_BACKUP), later
    AllReduces run on a ring in which 1 and 2 are no longer neighbours (the
    bridge is the 2-hop relay) instead of failing."""
    n, K = 4, 3
    comm = sim_comm(n, K=K, W=1, chunk_bytes=16 * 1024, max_bytes=16 << 20)
    for c in range(K - 1):
        kill(comm, "LINK", 1, c, "dead_links")
    assert expected_order(comm) == [0, 1, 2, 3]
    kill(comm, "LINK", 1, K - 1, "dead_links", ok=(R.SUCCESS, R.ERR_NO_BACKUP))
    order = expected_order(comm)
    assert order[(order.index(1) + 1) % n] != 2
    xs = r2inputs.inputs(n, 30_001, "int32", seed=5)
    rc, out = run_ar(comm, xs, "int32")
    assert rc == R.SUCCESS and comm.status()["ring_order"] == order
    y = OS.allreduce_ring(xs, order, shard_of(comm, 30_001, "int32", comm.status()["last_protocol"]), "int32")
    assert all(same_bits(out[r], y) for r in range(n))
    comm.finalize()
