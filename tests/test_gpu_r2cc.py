"""R²CCL-AllReduce on the GPU (§5.2,
App. A :358-447; readings R-9, R-10, R-11), simulated ranks on one
B200, through the C ABI: bit-exact against the oracle's
oracle.semantic.r2cc_allreduce, the planner's (f, X, Y, N_A, N_P) equal to
App. A's optimal partition and the split rule, faults inside either stage
recovered bit-exact, and the AUTO strategy choice equal to the oracle's
alpha-beta model on both sides of the crossover."""
import time

import numpy as np
import pytest
import torch

import r2inputs
from oracle import cost as OC
from oracle import semantic as OS
from oracle.geometry import Geometry
from tests.gpu_util import poisoned, same_bits, sim_comm, to_dev, to_np
from paper_2512_25059_b200 import build as B
from paper_2512_25059_b200 import r2ccl as R
from paper_2512_25059_b200 import torch_api as T

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def setup(cuda_required):
    B.build()
    torch.cuda.set_device(0)


def degrade(comm, f, chans, dtype="int32"):
    """Kill endpoint (f, c) for every c in chans the way a real failure does:
    a LOCAL fault mid-collective, triangulated to LOCAL_ENDPOINT(f) by the
    monitor (dead from the next collective on)."""
    n = comm.n
    for c in chans:
        s = comm.status()["seq"] + 1
        comm.inject_fault(at_seq=s, kind="LOCAL", src_rank=f, channel=c, step=0, chunk=0, byte_offset=0)
        xs = r2inputs.inputs(n, 256, dtype, seed=c)
        send = to_dev(xs, dtype)
        T.allreduce(comm, send, poisoned(n, 256, dtype), count=256)
        assert comm.sync() == R.SUCCESS
        t0 = time.time()
        while (f, c) not in comm.status()["dead_endpoints"]:
            assert time.time() - t0 < 5, "verdict not applied"
            time.sleep(0.002)


def r2cc_comm(n, K=4, W=2, algo="R2CC", **kw):
    return sim_comm(n, K=K, W=W, chunk_bytes=64 * 1024, max_bytes=16 << 20, allreduce_algo=algo, **kw)


def expected(comm, xs, dtype, f, dead, K):
    """The oracle's planner (App. A) and result for this degraded communicator."""
    n, N = len(xs), len(xs[0])
    E = r2inputs.elem_bytes(dtype)
    V = 16 // E
    X = OC.lost_fraction([1] * K, dead)
    Y = OC.optimal_partition(n, 1, X)
    NA, NP = OC.r2cc_split(N, V, Y)
    KA, KP = K - len(dead), len(dead)
    shA = Geometry(n, KA, NA, E, 16).shard if NA else 1
    shP = Geometry(n - 1, KP, NP, E, 16).shard if NP else 1
    return X, Y, NA, NP, OS.r2cc_allreduce(xs, dtype, f, NA, shA, shP)


def run_ar(comm, xs, dtype, inplace=False):
    n, N = len(xs), len(xs[0])
    send = to_dev(xs, dtype)
    recv = send if inplace else poisoned(n, N, dtype)
    T.allreduce(comm, send, recv, count=N)
    rc = comm.sync()
    return rc, to_np(recv, dtype)[:, :N]


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
@pytest.mark.parametrize("n,f", [(4, 1), (5, 4)])
def test_r2cc_parity(dtype, n, f):
    K, dead = 4, [0, 2]
    comm = r2cc_comm(n, K)
    degrade(comm, f, dead)
    N = 300_001
    xs = r2inputs.inputs(n, N, dtype, seed=7 * n + f)
    X, Y, NA, NP, y = expected(comm, xs, dtype, f, dead, K)
    calls0 = comm.status()["r2cc"]["calls"]
    rc, out = run_ar(comm, xs, dtype)
    assert rc == R.SUCCESS
    st = comm.status()["r2cc"]
    assert st["calls"] == calls0 + 1 and st["rank"] == f
    assert st["X"] == X and st["Y"] == Y and (st["NA"], st["NP"]) == (NA, NP)
    assert NP > 0 and NA > 0
    for r in range(n):
        assert same_bits(out[r], y), f"rank {r} differs from oracle r2cc_allreduce"
    comm.finalize()


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
def test_r2cc_inplace_and_ragged(dtype):
    n, K, f, dead = 4, 4, 3, [1, 3]
    comm = r2cc_comm(n, K)
    degrade(comm, f, dead)
    for N in (7, 1001, 65_539):
        xs = r2inputs.inputs(n, N, dtype, seed=N)
        *_, NP, y = expected(comm, xs, dtype, f, dead, K)
        rc, out = run_ar(comm, xs, dtype, inplace=True)
        assert rc == R.SUCCESS
        for r in range(n):
            assert same_bits(out[r], y), (N, r)
    comm.finalize()


@pytest.mark.parametrize("stage,rank,chan", [(1, 0, 1), (1, 2, 0), (1, 1, 3), (2, 0, 1), (2, 3, 3)])
def test_r2cc_fault_in_a_stage(stage, rank, chan):
    """A LINK fault inside stage 1 (global ring on channels {1, 3}, or the
    partial ring on {0, 2}) or inside stage 2: rollback + Balance within the
    ring's channels; the result equals the fault-free R²CCL-AllReduce."""
    n, K, f, dead, dtype = 4, 4, 1, [0, 2], "int32"
    comm = r2cc_comm(n, K, W=1)
    degrade(comm, f, dead)
    N = 200_003
    xs = r2inputs.inputs(n, N, dtype, seed=11, dist="wrap")
    *_, y = expected(comm, xs, dtype, f, dead, K)
    s = comm.status()["seq"] + stage           # stage 1 = next seq, stage 2 = the one after
    step = 1 if stage == 1 else (rank - f) % n
    comm.inject_fault(at_seq=s, kind="LINK", src_rank=rank, channel=chan, step=step, chunk=0, byte_offset=4096)
    ev0 = len(comm.events())
    rc, out = run_ar(comm, xs, dtype)
    assert rc == R.SUCCESS
    for r in range(n):
        assert same_bits(out[r], y), r
    ev = comm.events()[ev0:]
    assert len(ev) >= 1 and ev[0]["rank"] == rank and ev[0]["stopped_channel"] == chan, ev
    comm.finalize()


def test_auto_choice_matches_the_cost_model():
    """AUTO: the library runs R²CCL-AllReduce exactly when the oracle's
    alpha-beta model (reading R-11) predicts it faster: below and above the
    crossover size."""
    n, K, f, dead = 4, 4, 0, [0, 1, 2]          # X = 3/4
    comm = r2cc_comm(n, K, algo="AUTO")
    degrade(comm, f, dead)
    cfg = comm.cfg
    for N in (1024, 16 * 1024, 256 * 1024, 2 * 1024 * 1024):
        xs = r2inputs.inputs(n, N, "float32", seed=N)
        X, Y, NA, NP, y = expected(comm, xs, "float32", f, dead, K)
        t_ring, t_r2 = OC.algo_times(n, X, NP / N, N * 4.0, float(cfg.alpha_simple_ns), cfg.beta_mbps / 1000.0,
                                     float(cfg.alpha_launch_ns), cfg.r2cc_stage1_eff_pct / 100.0,
                                     cfg.r2cc_stage2_eff_pct / 100.0)
        calls0 = comm.status()["r2cc"]["calls"]
        rc, out = run_ar(comm, xs, "float32")
        assert rc == R.SUCCESS
        ran = comm.status()["r2cc"]["calls"] - calls0
        assert ran == (1 if t_r2 < t_ring else 0), (N, t_ring, t_r2)
        if ran:
            for r in range(n):
                assert same_bits(out[r], y)
    comm.finalize()


def test_ring_algo_never_runs_r2cc():
    n, K, f, dead = 4, 4, 2, [0, 1, 3]
    comm = r2cc_comm(n, K, algo="RING")
    degrade(comm, f, dead)
    xs = r2inputs.inputs(n, 100_000, "int32", seed=1)
    rc, out = run_ar(comm, xs, "int32")
    assert rc == R.SUCCESS and comm.status()["r2cc"]["calls"] == 0
    y = OS.allreduce(xs, Geometry(n, K, 100_000, 4, 16).shard, "int32")
    assert same_bits(out[0], y)
    comm.finalize()
