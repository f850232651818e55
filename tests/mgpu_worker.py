"""Multi-GPU parity worker: one process per GPU under torchrun, the real
CUDA-IPC / NVLink path of libr2ccl.so.  Every rank draws every rank's seeded
inputs, runs the allreduce through the C ABI, compares its result bit-exactly
with the oracle; failover records are gathered to rank 0 and compared with
the oracle's.  Rank 0 writes a JSON summary to argv[1]."""
import json
import os
import sys
import traceback

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import r2inputs  # noqa: E402
from oracle import protocol as OP  # noqa: E402
from oracle import semantic as OS  # noqa: E402
from oracle.geometry import Geometry  # noqa: E402
from tests.scenario import effective_chunk_bytes  # noqa: E402
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402
from tests.gpu_util import norm_event  # noqa: E402

TD = {"int32": torch.int32, "float32": torch.float32, "bfloat16": torch.bfloat16}


def dev_tensor(x: np.ndarray, dtype: str) -> torch.Tensor:
    if dtype == "bfloat16":
        return torch.from_numpy(x.view(np.int16).copy()).view(torch.bfloat16).cuda()
    return torch.from_numpy(x.copy()).cuda()


def host(t: torch.Tensor, dtype: str) -> np.ndarray:
    t = t.cpu()
    return t.view(torch.int16).numpy().view(np.uint16) if dtype == "bfloat16" else t.numpy()


def case(comm, rank, world, N, dtype, faults=(), strategy="BALANCE", inplace=False, seed=0, check_events=True):
    xs = r2inputs.inputs(world, N, dtype, seed=seed)
    send = dev_tensor(xs[rank], dtype)
    if inplace:
        recv = send
    else:
        recv = torch.empty_like(send)
        recv.view(torch.uint8).fill_(0xFF)
    T.register(comm, recv)
    seq = comm.status()["seq"] + 1
    for f in faults:
        comm.inject_fault(at_seq=seq, **f)
    ne = len(comm.events())
    T.allreduce(comm, send, recv)
    rc = comm.sync()
    E = r2inputs.elem_bytes(dtype)
    cfg = comm.cfg
    proto = comm.status()["last_protocol"]
    ll = proto in ("LL", "LL128")      # the alpha-beta choice (f3) shapes the step list
    g = Geometry(world, cfg.nchannels, N, E,
                 effective_chunk_bytes(N, world, cfg.nchannels, E, cfg.chunk_bytes, cfg.ctas_per_channel), ll=ll)
    # the planner may have re-ranked the ring (f4, reading R-13): fold along its order
    y = OS.allreduce_ring(xs, comm.status()["ring_order"], g.shard, dtype)
    ok = rc == R.SUCCESS and np.array_equal(host(recv, dtype).view(np.uint8), y.view(np.uint8))
    evs = [norm_event(e) for e in comm.events()[ne:]]
    all_evs = [None] * world
    dist.all_gather_object(all_evs, evs)
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok))
    out = {"N": N, "dtype": dtype, "faults": list(faults), "strategy": strategy, "rc": rc, "ok": all(oks),
           "protocol": proto}
    if faults:
        got = sorted((e for ev in all_evs for e in ev), key=lambda e: (e["rank"], e["stopped_channel"], e["origin"]))
        res = OP.simulate(xs, g, dtype, strategy=strategy, seed=0, inplace=inplace,
                          faults=[OP.Fault(f["kind"], f["src_rank"], f["channel"], f["step"], f["chunk"],
                                           f.get("byte_offset", 0)) for f in faults])
        want = sorted((norm_event(e) for e in res.events), key=lambda e: (e["rank"], e["stopped_channel"], e["origin"]))
        if check_events:            # (the oracle here simulates a healthy static plan)
            out["events_equal"] = got == want
        out["events"] = got
        out["want"] = want
        fo = [e["failover_ms"] for ev in [comm.events()[ne:]] for e in ev]
        out["failover_ms_rank"] = fo
    return out


def case_op(comm, rank, world, op, count, dtype, faults=(), strategy="BALANCE", inplace=False, seed=0):
    """Standalone ReduceScatter / AllGather (f1) over the real NVLink path."""
    n = world
    xs = r2inputs.inputs(n, n * count if op == "reduce_scatter" else count, dtype, seed=seed)
    E = r2inputs.elem_bytes(dtype)
    if op == "reduce_scatter":
        send = dev_tensor(xs[rank], dtype)
        recv = send[rank * count:(rank + 1) * count] if inplace else torch.empty(count, dtype=TD[dtype], device="cuda")
        want = OS.reduce_scatter(xs, count, dtype)[rank]
    else:
        recv = torch.empty(n * count, dtype=TD[dtype], device="cuda")
        if inplace:
            recv[rank * count:(rank + 1) * count] = dev_tensor(xs[rank], dtype)
            send = recv[rank * count:(rank + 1) * count]
        else:
            send = dev_tensor(xs[rank], dtype)
        want = OS.all_gather(xs)
        T.register(comm, recv)
    if not inplace:
        recv.view(torch.uint8).fill_(0xFF)
    st = comm.status()
    health = {"dead_links": st["dead_links"], "dead_endpoints": st["dead_endpoints"]}
    seq = st["seq"] + 1
    for f in faults:
        comm.inject_fault(at_seq=seq, **f)
    ne = len(comm.events())
    if op == "reduce_scatter":
        T.reduce_scatter(comm, send, recv, recvcount=count)
    else:
        T.all_gather(comm, send, recv, sendcount=count)
    rc = comm.sync()
    proto = comm.status()["last_protocol"]
    ll = proto in ("LL", "LL128")
    ok = rc == R.SUCCESS and np.array_equal(host(recv, dtype).view(np.uint8), np.asarray(want).view(np.uint8))
    evs = [norm_event(e) for e in comm.events()[ne:]]
    all_evs = [None] * world
    dist.all_gather_object(all_evs, evs)
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok))
    out = {"op": op, "N": count, "dtype": dtype, "faults": list(faults), "strategy": strategy, "rc": rc,
           "inplace": inplace, "ok": all(oks), "protocol": proto}
    if faults:
        cfg = comm.cfg
        g = Geometry(world, cfg.nchannels, count, E, effective_chunk_bytes(
            count, world, cfg.nchannels, E, cfg.chunk_bytes, cfg.ctas_per_channel, op), op, ll=ll)
        got = sorted((e for ev in all_evs for e in ev), key=lambda e: (e["rank"], e["stopped_channel"], e["origin"]))
        res = OP.simulate(xs, g, dtype, strategy=strategy, seed=0, health=health,
                          faults=[OP.Fault(f["kind"], f["src_rank"], f["channel"], f["step"], f["chunk"],
                                           f.get("byte_offset", 0)) for f in faults])
        want_ev = sorted((norm_event(e) for e in res.events),
                         key=lambda e: (e["rank"], e["stopped_channel"], e["origin"]))
        out["events_equal"] = got == want_ev
        out["events"] = got
        out["want"] = want_ev
    return out


def case_bcast(comm, rank, world, count, dtype, root, faults=(), strategy="BALANCE", seed=0):
    """Broadcast (f1) over the real NVLink chain."""
    xs = r2inputs.inputs(world, count, dtype, seed=seed)
    recv = torch.empty(count, dtype=TD[dtype], device="cuda")
    recv.view(torch.uint8).fill_(0xFF)
    send = dev_tensor(xs[rank], dtype) if rank == root else None
    T.register(comm, recv)
    st = comm.status()
    health = {"dead_links": st["dead_links"], "dead_endpoints": st["dead_endpoints"]}
    seq = st["seq"] + 1
    for f in faults:
        comm.inject_fault(at_seq=seq, **f)
    ne = len(comm.events())
    T.broadcast(comm, send, recv, root)
    rc = comm.sync()
    ok = rc == R.SUCCESS and np.array_equal(host(recv, dtype).view(np.uint8), np.asarray(xs[root]).view(np.uint8))
    evs = [norm_event(e) for e in comm.events()[ne:]]
    all_evs = [None] * world
    dist.all_gather_object(all_evs, evs)
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok))
    out = {"op": "broadcast", "root": root, "N": count, "dtype": dtype, "faults": list(faults), "rc": rc,
           "ok": all(oks)}
    if faults:
        from oracle.geometry import BROADCAST
        cfg = comm.cfg
        E = r2inputs.elem_bytes(dtype)
        g = Geometry(world, cfg.nchannels, count, E, effective_chunk_bytes(
            count, world, cfg.nchannels, E, cfg.chunk_bytes, cfg.ctas_per_channel, BROADCAST), BROADCAST, root=root)
        got = sorted((e for ev in all_evs for e in ev), key=lambda e: (e["rank"], e["stopped_channel"], e["origin"]))
        res = OP.simulate(xs, g, dtype, strategy=strategy, seed=0, health=health,
                          faults=[OP.Fault(f["kind"], f["src_rank"], f["channel"], f["step"], f["chunk"],
                                           f.get("byte_offset", 0)) for f in faults])
        want = sorted((norm_event(e) for e in res.events), key=lambda e: (e["rank"], e["stopped_channel"], e["origin"]))
        out["events_equal"] = got == want
        out["events"], out["want"] = got, want
    return out


def case_fullsize(rank, world, n_sample=4096):
    """The bench's launch configuration (256 MiB bf16 per rank, K = 8 x W = 16,
    512 KiB chunks, torch's seeded device RNG): sampled outputs against the
    oracle fold, every rank."""
    S = 256 << 20
    count = S // 2
    comm = T.comm_from_env(R.config_default(nchannels=8, ctas_per_channel=16, max_bytes=S))
    send = torch.empty(count, dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1234 + rank)
    send.copy_(torch.randn(count, generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16))
    recv = torch.empty_like(send)
    T.register(comm, recv)
    T.allreduce(comm, send, recv)
    rc = comm.sync()
    rng = np.random.default_rng(5)
    idx = np.unique(rng.integers(0, count, size=n_sample))
    it = torch.from_numpy(idx).cuda()
    mine = send[it].view(torch.int16).cpu().numpy().view(np.uint16)
    allx = [None] * world
    dist.all_gather_object(allx, mine)
    got = recv[it].view(torch.int16).cpu().numpy().view(np.uint16)
    geo = R.geometry(count, R.BFLOAT16, world, 8, 16, 512 * 1024)
    bad = 0
    for col, i in enumerate(idx):
        want = OS.ring_fold([allx[r][col:col + 1] for r in range(world)], int(i) // geo.shard, "bfloat16")[0]
        bad += int(got[col] != want)
    oks = [None] * world
    dist.all_gather_object(oks, rc == R.SUCCESS and bad == 0)
    comm.finalize()
    return {"op": "fullsize", "N": count, "n_checked": int(len(idx)), "rc": rc, "ok": all(oks)}


def case_host(rank, world):
    """r2_allreduce_host on pinned buffers large enough for the pipelined
    (segmented) path, twice back to back: bit-identical to the oracle fold."""
    count = (24 << 20) // 2 + 13              # 24 MiB bf16, ragged
    comm = T.comm_from_env(R.config_default(nchannels=8, ctas_per_channel=16, max_bytes=32 << 20))
    xs = r2inputs.inputs(world, count, "bfloat16", seed=99)
    hs = torch.from_numpy(xs[rank].view(np.int16).copy()).view(torch.bfloat16).pin_memory()
    hr = torch.empty_like(hs).pin_memory()
    ok = True
    for _ in range(2):
        hr.view(torch.int16).fill_(-1)
        T.allreduce_host(comm, hs, hr)
        rc = comm.sync()
        torch.cuda.synchronize()
        E = 2
        cfg = comm.cfg
        nseg = min(8, max(1, count * E // (4 << 20)))
        seg = (count + nseg - 1) // nseg // 8 * 8 + 8
        got = hr.view(torch.int16).numpy().view(np.uint16)
        for lo in range(0, count, seg):       # every segment is one collective
            hi = min(count, lo + seg)
            g = Geometry(world, cfg.nchannels, hi - lo, E,
                         effective_chunk_bytes(hi - lo, world, cfg.nchannels, E, cfg.chunk_bytes, cfg.ctas_per_channel))
            y = OS.allreduce([x[lo:hi] for x in xs], g.shard, "bfloat16")
            ok &= rc == R.SUCCESS and np.array_equal(got[lo:hi], y)
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok))
    comm.finalize()
    return {"op": "allreduce_host", "N": count, "ok": all(oks)}


def main():
    out_path = sys.argv[1]
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    results = []
    try:
        for strategy in ("BALANCE", "HOT_REPAIR"):
            cfg = R.config_default(nchannels=4, ctas_per_channel=2, chunk_bytes=64 * 1024, max_bytes=64 << 20,
                                   strategy=strategy)
            comm = T.comm_from_env(cfg)
            if strategy == "BALANCE":
                for dtype in ("int32", "float32", "bfloat16"):
                    for N in (1, 777, 100_003, (1 << 22) + 5):
                        results.append(case(comm, rank, world, N, dtype, seed=N))
                results.append(case(comm, rank, world, 300_001, "bfloat16", inplace=True, seed=7))
            f = dict(kind="LINK", src_rank=world - 1, channel=1, step=max(0, world - 2), chunk=1,
                     byte_offset=12345, poison=1)
            results.append(case(comm, rank, world, 1 << 20, "bfloat16", [f], strategy, seed=11))
            # Broadcast (f1): every root, and one LINK fault on a sending rank
            if strategy == "BALANCE":
                for root in range(world):
                    results.append(case_bcast(comm, rank, world, 100_003, "bfloat16", root, seed=root))
            fb = dict(kind="LINK", src_rank=(1 % world), channel=1, step=(1 % world) if world > 1 else 0, chunk=0,
                      byte_offset=2048, poison=1)
            results.append(case_bcast(comm, rank, world, 1 << 18, "int32", 0, [fb], strategy, seed=23))
            # standalone ReduceScatter / AllGather: healthy (ragged, in-place) and one LINK fault
            for op in ("reduce_scatter", "all_gather"):
                if strategy == "BALANCE":
                    for dtype, count in (("bfloat16", 100_003), ("float32", 1 << 18), ("int32", 777)):
                        results.append(case_op(comm, rank, world, op, count, dtype, seed=count))
                    results.append(case_op(comm, rank, world, op, 65_537, "bfloat16", inplace=True, seed=3))
                fo = dict(kind="LINK", src_rank=0, channel=2, step=0, chunk=1, byte_offset=4096, poison=1)
                results.append(case_op(comm, rank, world, op, 1 << 18, "bfloat16", [fo], strategy, seed=17))
            # degraded steady state (channel 1 of rank world-1 now dead): static plan
            results.append(case(comm, rank, world, 1 << 20, "float32", seed=12))
            comm.finalize()
        results.append(case_fullsize(rank, world))
        results.append(case_host(rank, world))
        # the line protocols (f3) forced, over the real NVLink path: LL (R-6) and LL128 (R-12)
        for proto in ("LL", "LL128"):
            cfg = R.config_default(nchannels=4, ctas_per_channel=2, chunk_bytes=16 * 1024, max_bytes=16 << 20,
                                   protocol=proto)
            comm = T.comm_from_env(cfg)
            for dtype, N in (("bfloat16", 100_003), ("float32", 1 << 16), ("int32", 5)):
                results.append(case(comm, rank, world, N, dtype, seed=N + 1))
            results.append(case(comm, rank, world, 77_777, "bfloat16", inplace=True, seed=2))
            for op in ("reduce_scatter", "all_gather"):
                results.append(case_op(comm, rank, world, op, 33_333, "bfloat16", seed=4))
            f = dict(kind="LINK", src_rank=world - 1, channel=1, step=1, chunk=1, byte_offset=4096, poison=1)
            results.append(case(comm, rank, world, 1 << 19, "bfloat16", [f], "BALANCE", seed=19))
            # the ring is now statically degraded (link world-1 -> 0 on channel 1) and
            # still speculates; a LOCAL fault on another rank mid-call re-plans lanes
            # that hold spinning items: abandoned and re-issued (reading R-6)
            f2 = dict(kind="LOCAL", src_rank=0, channel=2, step=1, chunk=0, byte_offset=2048, poison=1)
            results.append(case(comm, rank, world, 1 << 19, "bfloat16", [f2], "BALANCE", seed=20, check_events=False))
            comm.finalize()
        # LL128 at the bench's mid size with the bench's 8 x 16 CTAs (config-5 bucket)
        cfg = R.config_default(nchannels=8, ctas_per_channel=16, max_bytes=32 << 20, protocol="LL128")
        comm = T.comm_from_env(cfg)
        results.append(case(comm, rank, world, 12_500_000, "bfloat16", seed=25))
        f = dict(kind="LINK", src_rank=world - 1, channel=5, step=1, chunk=3, byte_offset=8192, poison=1)
        results.append(case(comm, rank, world, 12_500_000, "bfloat16", [f], "BALANCE", seed=26))
        comm.finalize()
        # re-probe (f4): LINK fault, HEAL (the library is not told), re-admission by re-probing
        cfg = R.config_default(nchannels=4, ctas_per_channel=2, chunk_bytes=32 * 1024, max_bytes=16 << 20,
                               reprobe_us=300, reprobe_max_us=5000)
        comm = T.comm_from_env(cfg)
        f = dict(kind="LINK", src_rank=world - 1, channel=3, step=0, chunk=0, byte_offset=1024)
        results.append(case(comm, rank, world, 200_003, "bfloat16", [f], "BALANCE", seed=41))
        results.append(case(comm, rank, world, 200_003, "bfloat16", seed=42))        # degraded
        seq = comm.status()["seq"] + 1
        comm.inject_fault(at_seq=seq, kind="HEAL", src_rank=world - 1, channel=3)
        results.append(case(comm, rank, world, 200_003, "bfloat16", seed=43))        # fabric healed
        import time
        deadline = time.time() + 3.0
        while rank == world - 1 and comm.status()["n_readmits"] == 0 and time.time() < deadline:
            time.sleep(0.005)
        dist.barrier()
        results.append(case(comm, rank, world, 200_003, "bfloat16", seed=44))        # re-admitted
        st = comm.status()
        ok = rank != world - 1 or ((world - 1, 3) not in st["dead_links"] and st["n_readmits"] >= 1)
        oks = [None] * world
        dist.all_gather_object(oks, bool(ok))
        results.append({"op": "reprobe", "ok": all(oks), "status": {k: st[k] for k in ("n_reprobes", "n_readmits")}})
        comm.finalize()
        if world >= 2:
            cfg = R.config_default(nchannels=3, ctas_per_channel=2, chunk_bytes=32 * 1024, max_bytes=64 << 20)
            comm = T.comm_from_env(cfg)
            f = dict(kind="LOCAL", src_rank=0, channel=2, step=1, chunk=0, byte_offset=4096)
            r = case(comm, rank, world, 500_000, "int32", [f], "BALANCE", seed=13)
            r.pop("events_equal", None)   # secondary connection's record is timing-dependent
            results.append(r)
            comm.finalize()
    except Exception:
        traceback.print_exc()
        results.append({"error": traceback.format_exc()})
    if rank == 0:
        with open(out_path, "w") as fh:
            json.dump(results, fh, indent=1, default=str)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
