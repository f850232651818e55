"""Helpers shared by the -m gpu tests: seeded inputs -> device tensors, the
oracle's expectations, and event comparison.  Test code only."""
from __future__ import annotations

import numpy as np
import torch

import r2inputs
from oracle import protocol as OP
from oracle import semantic as OS
from oracle.geometry import Geometry
from tests.scenario import effective_chunk_bytes
from paper_2512_25059_b200 import r2ccl as R
from paper_2512_25059_b200 import torch_api as T

TD = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}


def row_len(N: int, dtype: str) -> int:
    """Sim-mode rank rows are 16-byte aligned: roundup(N, 16 / elem)."""
    v = 16 // r2inputs.elem_bytes(dtype)
    return max(-(-N // v) * v, v)


def to_dev(arrs: list, dtype: str) -> torch.Tensor:
    N = len(arrs[0])
    a = np.zeros((len(arrs), row_len(N, dtype)), dtype=arrs[0].dtype)
    a[:, :N] = np.stack(arrs)
    if dtype == "bfloat16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(a.copy()).cuda()


def to_np(t: torch.Tensor, dtype: str) -> np.ndarray:
    t = t.cpu()
    if dtype == "bfloat16":
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def poisoned(n: int, N: int, dtype: str) -> torch.Tensor:
    t = torch.empty((n, row_len(N, dtype)), dtype=TD[dtype], device="cuda")
    t.view(torch.uint8).fill_(0xFF)
    return t


def sim_comm(n, K=4, W=2, chunk_bytes=64 * 1024, max_bytes=16 << 20, strategy="BALANCE", protocol="SIMPLE",
             **kw) -> R.Comm:
    """Simulated-rank communicator.  The protocol is pinned (SIMPLE unless a
    test asks for LL / AUTO) so that the oracle's step list is known."""
    cfg = R.config_default(sim_ranks=n, nchannels=K, ctas_per_channel=W, chunk_bytes=chunk_bytes,
                           max_bytes=max_bytes, strategy=strategy, protocol=protocol, **kw)
    return R.Comm(0, 1, torch.cuda.current_device(), None, cfg)


def oracle_geom(comm: R.Comm, N: int, dtype: str) -> Geometry:
    E = r2inputs.elem_bytes(dtype)
    cfg = comm.cfg
    return Geometry(comm.n, cfg.nchannels, N, E,
                    effective_chunk_bytes(N, comm.n, cfg.nchannels, E, cfg.chunk_bytes, cfg.ctas_per_channel))


def run(comm: R.Comm, xs: list, dtype: str, inplace=False):
    n = len(xs)
    N = len(xs[0])
    send = to_dev(xs, dtype)
    recv = send if inplace else poisoned(n, N, dtype)
    T.allreduce(comm, send, recv, count=N)
    rc = comm.sync()
    out = to_np(recv, dtype)
    # the row padding past N must never be written (out-of-place: still poison)
    if not inplace and out.shape[1] > N:
        assert np.all(out[:, N:].view(np.uint8) == 0xFF), "wrote past count"
    return rc, out[:, :N]


def same_bits(a, b) -> bool:
    return np.array_equal(np.asarray(a).view(np.uint8), np.asarray(b).view(np.uint8))


def check_result(out: np.ndarray, xs: list, g: Geometry, dtype: str):
    y = OS.allreduce(xs, g.shard, dtype)
    for r in range(out.shape[0]):
        if not same_bits(out[r], y):
            bad = np.nonzero(out[r].view(np.uint8) != y.view(np.uint8))[0]
            raise AssertionError(f"rank {r}: {len(bad)} bytes differ, first at byte {bad[:8]}")


EV_KEYS = ("rank", "origin", "stopped_channel", "verdict", "a", "b", "aux", "outcomes", "resume", "floor",
           "retransmit")


def norm_event(e: dict) -> dict:
    d = {k: e[k] for k in EV_KEYS}
    d["outcomes"] = tuple(e["outcomes"])
    if "assignee" in e:
        d["assignee"], d["chain_pos"] = e["assignee"], e["chain_pos"]
    if "shares" in e:
        d["shares"] = {int(k): int(v) for k, v in e["shares"].items()}
    return d


def oracle_faults(faults: list) -> list:
    return [OP.Fault(f["kind"], f["src_rank"], f["channel"], f["step"], f["chunk"], f.get("byte_offset", 0),
                     None if f.get("origin_channel", -1) < 0 else f["origin_channel"]) for f in faults]
