"""The C-ABI library loads and exports every symbol include/r2ccl.h declares;
its pure host logic (no GPU needed) matches the oracle; the shared-memory
OOB works across 2 processes bootstrapped with torch.distributed (gloo)."""
import itertools
import os
import re

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import r2inputs
from oracle import balance as OB
from oracle import ledger as OL
from oracle import rerank as ORR
from oracle import triangulation as OT
from oracle.geometry import Geometry
from tests.scenario import effective_chunk_bytes
from paper_2512_25059_b200 import build as B
from paper_2512_25059_b200 import r2ccl as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    B.build()


def header_symbols():
    src = open(os.path.join(ROOT, "include", "r2ccl.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(r2_[a-z_]+)\s*\(", src))


def test_every_declared_symbol_is_exported():
    syms = header_symbols()
    assert len(syms) >= 20
    lib = R.lib()
    for s in syms:
        assert hasattr(lib, s), s
    assert syms == set(R.EXPORTS), syms ^ set(R.EXPORTS)


def test_strerror():
    for code in range(8):
        assert R.lib().r2_strerror(code)
    assert b"exhausted" in R.lib().r2_strerror(R.ERR_NO_BACKUP)


def test_triangulate_matches_oracle_exhaustively():
    for ab, ba in itertools.product(OT.OUTCOMES, repeat=2):
        assert R.triangulate([ab, ba], False) == OT.triangulate(ab, ba)
    for o in itertools.product(OT.OUTCOMES, repeat=4):
        assert R.triangulate(list(o), True) == OT.triangulate(*o)


def test_balance_shares_match_oracle():
    rng = np.random.default_rng(4)
    for _ in range(3000):
        K = int(rng.integers(1, 17))
        w = [int(x) for x in rng.integers(1, 1000, size=K)]
        healthy = [c for c in range(K) if rng.random() < 0.8]
        if not healthy:
            continue
        Rv = int(rng.integers(0, 1 << 40))
        want = OB.redistribute(Rv, dict(enumerate(w)), set(range(K)) - set(healthy))
        assert R.balance_shares(Rv, w, healthy) == want


def test_balance_all_failed_is_no_backup():
    with pytest.raises(R.R2Error) as e:
        R.balance_shares(10, [1, 1], [])
    assert e.value.code == R.ERR_NO_BACKUP


def test_chain_and_rollback_match_oracle():
    for K in range(1, 17):
        for c in range(K):
            assert R.failover_chain(c, K) == OL.failover_chain(c, K)
    for k in range(0, 10):
        for mask in itertools.product([False, True], repeat=k):
            assert R.rollback(list(mask)) == OL.rollback(list(mask))


def test_rerank_matches_oracle():
    """r2_rerank (Algorithm 1, reading R-13) == oracle/rerank.py on random
    rail-failure patterns with and without dead standard links (2000 cases,
    n = 3..16, K = 1..8) and on every pattern of n = 4, K = 2."""
    import random
    rng = random.Random(7)
    cases = []
    for combo in itertools.product(range(1, 4), repeat=4):
        cases.append((4, 2, list(combo), [0] * 4))
    for _ in range(2000):
        n, K = rng.randint(3, 16), rng.randint(1, 8)
        full = (1 << K) - 1
        rails = [rng.choice([full, full, rng.randint(1, full)]) for _ in range(n)]
        dead = [rng.choice([0, 0, 0, rng.randint(0, full)]) for _ in range(n)] if rng.random() < 0.5 else [0] * n
        cases.append((n, K, rails, dead))
    for n, K, rails, dead in cases:
        order = list(range(n))
        random.Random(n * 31 + K).shuffle(order)
        rs = {u: frozenset(c for c in range(K) if rails[u] >> c & 1) for u in range(n)}
        dl = {(u, (u + 1) % n, c) for u in range(n) for c in range(K) if dead[u] >> c & 1}
        want = ORR.rerank(order, rs, ORR.link_cap(rs, dl))
        assert R.rerank(order, rails, dead) == want, (order, rails, dead)


def test_geometry_matches_oracle():
    rng = np.random.default_rng(5)
    for _ in range(3000):
        dt = ["int32", "float32", "bfloat16"][int(rng.integers(3))]
        E = r2inputs.elem_bytes(dt)
        n, K, W = int(rng.integers(1, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 5))
        N = int(rng.integers(1, 1 << 22))
        chunk = int(rng.integers(1, 1 << 16)) * 16
        g = R.geometry(N, R.DTYPE_NAMES[dt], n, K, W, chunk)
        og = Geometry(n, K, N, E, effective_chunk_bytes(N, n, K, E, chunk, W))
        assert (g.Np, g.shard, g.slice, g.chunk, g.m, g.steps, g.V) == \
            (og.Np, og.shard, og.slice, og.chunk, og.m, og.steps, og.V)


@pytest.mark.parametrize("op", ["reduce_scatter", "all_gather"])
def test_geometry_op_matches_oracle(op):
    """ReduceScatter / AllGather geometry (f1): shard padding, stride, steps,
    AllGather's step offset and the ReduceScatter's LOCAL step."""
    rng = np.random.default_rng(7)
    for _ in range(2000):
        dt = ["int32", "float32", "bfloat16"][int(rng.integers(3))]
        E = r2inputs.elem_bytes(dt)
        n, K, W = int(rng.integers(2, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 5))
        count = int(rng.integers(1, 1 << 20))
        chunk = int(rng.integers(1, 1 << 16)) * 16
        g = R.geometry(count, R.DTYPE_NAMES[dt], n, K, W, chunk, R.OPS[op])
        og = Geometry(n, K, count, E, effective_chunk_bytes(count, n, K, E, chunk, W, op), op)
        assert (g.N, g.Np, g.shard, g.slice, g.chunk, g.m, g.steps, g.stride, g.t0) == \
            (og.total, og.Np, og.shard, og.slice, og.chunk, og.m, og.steps, og.stride, og.t0)
        assert g.local_step == (n - 1 if op == "reduce_scatter" else -1)
        assert all(og.local(t) == (t == g.local_step) for t in range(og.steps))


# ------------------------------------------------------------ OOB, 2 procs

def _oob_worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    name = [R.unique_name() if rank == 0 else None]
    dist.broadcast_object_list(name, src=0)
    o = R.oob_shm_open(name[0], rank, world)
    got = R.oob_allgather(o, bytes([rank + 1]) * 40, world)
    ok = got == [bytes([r + 1]) * 40 for r in range(world)]
    R.oob_barrier(o)
    # every rank posts one message to every other rank (bilateral notify)
    for d in range(world):
        if d != rank:
            R.oob_post(o, d, f"notify {rank}->{d}".encode())
    seen = set()
    import time
    t0 = time.time()
    while len(seen) < world - 1 and time.time() - t0 < 20:
        m = R.oob_poll(o)
        if m:
            seen.add((m[0], m[1].decode()))
    ok = ok and seen == {(s, f"notify {s}->{rank}") for s in range(world) if s != rank}
    R.oob_barrier(o)
    R.oob_shm_close(o)
    out[rank] = int(ok)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_oob_shm_multiprocess_gloo(world):
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    port = 29500 + (os.getpid() % 500) + world
    procs = [ctx.Process(target=_oob_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
        assert p.exitcode == 0
    assert list(out) == [1] * world


def test_geometry_broadcast_matches_oracle():
    """Broadcast geometry (f1): one shard = the whole padded buffer."""
    from oracle.geometry import BROADCAST
    rng = np.random.default_rng(9)
    for _ in range(2000):
        dt = ["int32", "float32", "bfloat16"][int(rng.integers(3))]
        E = r2inputs.elem_bytes(dt)
        n, K, W = int(rng.integers(2, 9)), int(rng.integers(1, 9)), int(rng.integers(1, 5))
        count = int(rng.integers(1, 1 << 20))
        chunk = int(rng.integers(1, 1 << 16)) * 16
        g = R.geometry(count, R.DTYPE_NAMES[dt], n, K, W, chunk, R.OP_BROADCAST)
        og = Geometry(n, K, count, E, effective_chunk_bytes(count, n, K, E, chunk, W, BROADCAST), BROADCAST)
        assert (g.N, g.Np, g.shard, g.slice, g.chunk, g.m, g.steps, g.stride) == \
            (og.total, og.Np, og.shard, og.slice, og.chunk, og.m, og.steps, og.stride)
