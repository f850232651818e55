"""bench.py -- R²CCL hot path on B200: fault-tolerant ring allreduce.

Workload (BASELINE.json configs[2]): 256 MiB bf16
per rank, K = 8 channels, 512 KiB chunks (1 MiB on GPUs, --chunk).
  N = 1  (default): 8 simulated ranks on one B200 in one cooperative kernel
         (the "1 GPU local reduce" configuration; all traffic is HBM).
  N > 1 (torchrun): one process per GPU, CUDA-IPC peer stores over NVLink 5.
One step = one allreduce (one kernel launch) over inputs resident in HBM
(2 GiB touched per step > 126 MB L2: no flush needed).  Metric: aggregate
bus bandwidth = sum over ranks of 2(n-1)/n * S / t (nccl-tests bus bytes).
After the timed healthy steps the same run measures the single-failure
scenario: failover latency, the faulted call, degraded Balance / HotRepair
steady state against the surviving-bandwidth bound, bit-identity.

--impl reference: the CPU oracle (oracle/, test infrastructure) timed on the
host cores on a bounded sample of the same workload, same metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

MIB = 1 << 20


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="r2", choices=["r2", "reference"])
    ap.add_argument("--bytes", type=int, default=256 * MIB, help="payload per rank")
    ap.add_argument("--sim-ranks", type=int, default=8)
    ap.add_argument("--channels", type=int, default=8)
    ap.add_argument("--ctas-small", type=int, default=4,
                    help="N>1: also time the headline with this many CTAs per channel (0 = skip)")
    ap.add_argument("--ctas", type=int, default=0, help="CTAs per channel (0 = auto)")
    ap.add_argument("--threads", type=int, default=0,
                    help="threads per CTA (0 = auto: 512 for the HBM-bound simulated ranks, 256 on GPUs -- "
                         "profiles/r01_sweep_threads_n4.log)")
    ap.add_argument("--chunk", type=int, default=0,
                    help="chunk bytes (0 = auto: 512 KiB for the simulated ranks, 1 MiB on GPUs -- "
                         "profiles/r02_chunk_n24.txt)")
    ap.add_argument("--no-fault", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-nccl", action="store_true")
    ap.add_argument("--no-coll", action="store_true", help="skip the standalone ReduceScatter / AllGather section")
    ap.add_argument("--protocol", default="AUTO", choices=["AUTO", "SIMPLE", "LL", "LL128"])
    ap.add_argument("--bw-model-gbps", type=int, default=80,
                    help="per-channel bandwidth of the channel-as-NIC fault section (0 = skip; r2ccl.h channel_gbps)")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no extras)")
    ap.add_argument("--per-step", action="store_true", help="debug: per-step CUDA-event times to stderr")
    ap.add_argument("--clock-ms", type=int, default=20, help="nvidia-smi sampling period (ms)")
    ap.add_argument("--clock-test", action="store_true", help="debug: timing with/without the sampler")
    ap.add_argument("--recreate", type=int, default=0, help="debug: re-create the comm R times, time each")
    return ap.parse_args()


def peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:
        return {}


# ------------------------------------------------------------------ clocks
class Clocks:
    """nvidia-smi sampler running during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    period_ms = 20

    def __init__(self, gpu):
        self.gpu = gpu if isinstance(gpu, str) else str(gpu)   # "0" or "0,1,2,3"
        self.p = None
        self.lines = []
        self.armed = False
        self.out = ""

    def _reader(self):
        for line in self.p.stdout:
            if self.armed:
                self.lines.append(line)

    def __enter__(self):
        import threading
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-lms", str(self.period_ms), "-i", self.gpu], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            for _ in range(self.gpu.count(",") + 1):
                self.p.stdout.readline()  # sampler is live before the timed region starts
            threading.Thread(target=self._reader, daemon=True).start()
            self.armed = True
        except Exception:
            self.p = None
        return self

    def __exit__(self, *a):
        self.armed = False
        self.out = "".join(self.lines)
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                pass

    def summary(self) -> dict:
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 8:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for nm, v in zip(names, f[4:8]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


# ------------------------------------------------------------------ oracle baseline
def oracle_rate(k: int, sample_bytes: int, reps: int = 1) -> dict:
    """Time the CPU oracle (Layer 2 protocol simulator) on k ranks x sample."""
    os.environ.setdefault("OMP_NUM_THREADS", "1")
    import r2inputs
    from oracle import protocol as OP
    from oracle.geometry import Geometry
    from tests.scenario import effective_chunk_bytes
    N = sample_bytes // 2
    xs = r2inputs.inputs(k, N, "bfloat16", seed=1)
    g = Geometry(k, 8, N, 2, effective_chunk_bytes(N, k, 8, 2, 512 * 1024, 1))
    t0 = time.perf_counter()
    for _ in range(reps):
        OP.simulate(xs, g, "bfloat16", seed=0)
    t = (time.perf_counter() - t0) / reps
    agg = k * 2 * (k - 1) / k * sample_bytes / t / 1e9
    return {"seconds": t, "agg_busbw_GBs": agg}


def cpu_info() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------ GPU arm
def fill_inputs(send, seed):
    import torch
    g = torch.Generator(device=send.device)
    g.manual_seed(seed)
    send.copy_(torch.randn(send.shape, generator=g, device=send.device, dtype=torch.float32).to(send.dtype))


class stdout_to_stderr:
    """Route fd 1 to fd 2 (library banners must not break the one-line JSON)."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def timed(fn, steps, stream):
    import torch
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(steps):
        fn()
    e1.record(stream)
    e1.synchronize()
    return e0.elapsed_time(e1) / steps  # ms


def fault_scenario(make_comm, run_step, healthy_ms, S, n, K, geom_m, strategy, get_result, ref_result,
                   fault_rank=3, fault_ch=5, t=3, j=4, b=256 * 1024, degraded_steps=20, stream=None,
                   barrier=lambda: None, reduce_max=lambda x: x, is_root=True, gather=lambda evs: evs):
    """Config 3: one LINK fault mid-collective, then the degraded steady state."""
    import torch
    comm = make_comm(strategy)
    comm.inject_fault(at_seq=2, kind="LINK", src_rank=fault_rank % n, channel=fault_ch % K, step=min(t, 2 * n - 3),
                      chunk=min(j, geom_m - 1), byte_offset=b, poison=1)
    run_step(comm)                       # seq 1: healthy warm-up on this comm
    torch.cuda.synchronize()
    barrier()
    ms_faulted = reduce_max(timed(lambda: run_step(comm), 1, stream))     # seq 2: faulted
    rc = comm.sync()
    identical = bool(torch.equal(get_result(), ref_result)) if ref_result is not None else None
    identical = bool(reduce_max(0.0 if identical else 1.0) == 0.0)
    evs = gather(comm.events())
    for _ in range(2):
        run_step(comm)
    torch.cuda.synchronize()
    barrier()
    ms_deg = reduce_max(timed(lambda: run_step(comm), degraded_steps, stream))
    rc2 = comm.sync()
    busbw = lambda ms: 2 * (n - 1) / n * S / (ms * 1e-3) / 1e9
    bound = busbw(healthy_ms) * (K - 1) / K if strategy == "BALANCE" else busbw(healthy_ms) * 0.5
    out = {"strategy": strategy, "rc_faulted": rc, "rc_degraded": rc2, "bit_identical_to_healthy": identical,
           "failover_ms": [e["failover_ms"] for e in evs], "events": [
               {k2: e[k2] for k2 in ("rank", "origin", "verdict", "resume", "floor", "retransmit")} for e in evs],
           "ms_faulted_call": ms_faulted, "ms_healthy_call": healthy_ms,
           "extra_ms_faulted": ms_faulted - healthy_ms,
           "busbw_per_rank_degraded": busbw(ms_deg), "busbw_per_rank_healthy": busbw(healthy_ms),
           "degraded_over_healthy": healthy_ms / ms_deg,
           "surviving_bound_busbw": bound, "degraded_over_bound": busbw(ms_deg) / bound,
           "model": "Balance bound (K-1)/K of healthy; HotRepair model 1/2 (S:742-743)"}
    comm.finalize()
    return out


def coll_section(a, T, R, world, rank, K, W, S, send, recv, stream, barrier, reduce_max, pg):
    """standalone ReduceScatter / AllGather on the same S-byte
    n-shard buffers, healthy and with one channel of one rank dead (Balance;
    the paper reports 85-89 % of normal throughput), NCCL beside.
    busbw = (n-1)/n * S / t (nccl-tests convention for RS/AG)."""
    import torch
    import torch.distributed as dist
    n = world
    cnt = S // 2 // n
    steps = max(5, min(a.steps, 50))
    shard = recv[:cnt]
    out = {}
    busbw = lambda ms: (n - 1) / n * S / (ms * 1e-3) / 1e9  # noqa: E731
    for strategy in ("BALANCE",):
        for degraded in (False, True):
            # 512 threads: the ReduceScatter's local final add is HBM-bound (256 halves it)
            c = T.comm_from_env(R.config_default(nchannels=K, ctas_per_channel=W, threads_per_cta=512,
                                                 chunk_bytes=a.chunk, max_bytes=S, strategy=strategy))
            T.register(c, recv)
            if degraded:   # the config-3 LINK fault, then the steady state with the channel dead
                c.inject_fault(at_seq=1, kind="LINK", src_rank=3 % n, channel=5 % K, step=0, chunk=0,
                               byte_offset=4096)
            ops = {"reduce_scatter": lambda: T.reduce_scatter(c, send, shard, recvcount=cnt),
                   "all_gather": lambda: T.all_gather(c, send[:cnt], recv, sendcount=cnt),
                   "broadcast": lambda: T.broadcast(c, send if rank == 0 else None, recv, 0)}
            for name, fn in ops.items():
                for _ in range(3):
                    fn()
                barrier()
                ms = reduce_max(timed(fn, steps, stream))
                d = out.setdefault(name, {})
                d["degraded_busbw" if degraded else "busbw"] = busbw(ms)
                d["degraded_ms" if degraded else "ms"] = ms
            assert c.sync() == R.SUCCESS
            c.finalize()
    # Broadcast: nccl-tests busbw = algbw = S / t (the whole buffer crosses every link of the chain)
    if "broadcast" in out:
        d = out["broadcast"]
        d["busbw"] = S / (d["ms"] * 1e-3) / 1e9
        d["degraded_busbw"] = S / (d["degraded_ms"] * 1e-3) / 1e9
    for name, d in out.items():
        d["degraded_over_healthy"] = d["degraded_busbw"] / d["busbw"]
        d["degraded_over_bound"] = d["degraded_busbw"] / (d["busbw"] * (K - 1) / K)
    if pg is not None:
        rs_out = torch.empty(cnt, dtype=send.dtype, device="cuda")
        ag_out = torch.empty(n * cnt, dtype=send.dtype, device="cuda")
        bc = send.clone()
        nc = {"reduce_scatter": lambda: dist.reduce_scatter_tensor(rs_out, send[:n * cnt], group=pg),
              "all_gather": lambda: dist.all_gather_into_tensor(ag_out, send[:cnt], group=pg),
              "broadcast": lambda: dist.broadcast(bc, 0, group=pg)}
        for name, fn in nc.items():
            for _ in range(3):
                fn()
            barrier()
            ms_n = reduce_max(timed(fn, steps, stream))
            out[name]["nccl_busbw"] = (S / (ms_n * 1e-3) / 1e9) if name == "broadcast" else busbw(ms_n)
    out["note"] = ("S-byte n-shard buffer per rank (RS input / AG output; Broadcast buffer, root 0), bf16; "
                   "degraded = one LINK fault (rank 3 % n, ch 5), Balance; bound (K-1)/K of healthy")
    return out


def host_segments(count, elem_bytes):
    """Segments of the pipelined r2_allreduce_host (one rank per process; mirrors
    r2_comm.cpp): up to 8 segments of >= 4 MiB from 8 MiB on, else one."""
    nbytes = count * elem_bytes
    if nbytes < (8 << 20):
        return [(0, count)]
    V = 16 // elem_bytes
    nseg = min(8, max(1, nbytes // (4 << 20)))
    seg = (count + nseg - 1) // nseg // V * V + V
    return [(lo, min(count, lo + seg)) for lo in range(0, count, seg)][:nseg]


def guarded(fn):
    """Run an auxiliary bench section; on an exception record it (the
    headline measurement is printed regardless)."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        print(f"bench: auxiliary section failed: {e!r}", file=sys.stderr, flush=True)
        return {"error": repr(e)}


def successive_scenario(make_comm, run_step, healthy_ms, n, K, geom_m, strategy, get_result, ref_result,
                        fault_rank=3, fault_ch=5, t=3, j=4, b=256 * 1024, stream=None, barrier=lambda: None,
                        reduce_max=lambda x: x, gather=lambda evs: evs):
    """Config 4: the config-3 LINK fault, then a second LINK fault on the
    adopting backup (chain[0] = ch+1) while it carries the residual (P:36
    successive failover: roll back again, move to the next chain entry)."""
    import torch
    comm = make_comm(strategy)
    steps = 2 * n - 2
    t1, j1 = min(t, steps - 2), min(j, geom_m - 1)
    t2 = t1 + 1
    r, c1, c2 = fault_rank % n, fault_ch % K, (fault_ch + 1) % K
    comm.inject_fault(at_seq=2, kind="LINK", src_rank=r, channel=c1, step=t1, chunk=j1, byte_offset=b, poison=1)
    comm.inject_fault(at_seq=2, kind="LINK", src_rank=r, channel=c2, step=t2, chunk=j1, byte_offset=b // 2,
                      origin_channel=c1, poison=1)
    run_step(comm)
    torch.cuda.synchronize()
    barrier()
    ms = reduce_max(timed(lambda: run_step(comm), 1, stream))
    rc = comm.sync()
    identical = bool(torch.equal(get_result(), ref_result)) if ref_result is not None else None
    identical = bool(reduce_max(0.0 if identical else 1.0) == 0.0)
    evs = gather(comm.events())
    out = {"strategy": strategy, "rc": rc, "bit_identical_to_healthy": identical, "ms_faulted_call": ms,
           "extra_ms": ms - healthy_ms,
           "events": [{k2: e.get(k2) for k2 in ("rank", "origin", "stopped_channel", "verdict", "resume", "retransmit",
                                            "assignee", "chain_pos", "failover_ms")} for e in evs]}
    comm.finalize()
    return out


def run_sim(a):
    """N = 1: k simulated ranks on one B200."""
    import torch
    from paper_2512_25059_b200 import build as B
    from paper_2512_25059_b200 import r2ccl as R
    from paper_2512_25059_b200 import torch_api as T
    B.build()
    torch.cuda.set_device(0)
    k, K, S = a.sim_ranks, a.channels, a.bytes
    W = a.ctas or max(1, min(4, 148 // (k * K)))
    a.chunk = a.chunk or 512 * 1024
    count = S // 2
    mk = lambda strategy: R.Comm(0, 1, 0, None, R.config_default(
        sim_ranks=k, nchannels=K, ctas_per_channel=W, threads_per_cta=a.threads, chunk_bytes=a.chunk,
        max_bytes=S, strategy=strategy, protocol=a.protocol))
    comm = mk("BALANCE")
    send = torch.empty((k, count), dtype=torch.bfloat16, device="cuda")
    recv = torch.empty_like(send)
    fill_inputs(send, 1234)
    stream = torch.cuda.current_stream()
    step = lambda c=comm: T.allreduce(c, send, recv)
    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    with Clocks(0) as clk:
        ms = timed(step, a.steps, stream)
    assert comm.sync() == R.SUCCESS
    g = R.geometry(count, R.BFLOAT16, k, K, W, a.chunk)
    res = {"ms": ms, "clocks": clk.summary(), "W": W, "m": g.m}
    if a.profile:
        return res, None
    ref = recv.clone()
    if not a.no_e2e:
        hs = torch.empty((k, count), dtype=torch.bfloat16).pin_memory()
        hr = torch.empty_like(hs).pin_memory()
        hs.copy_(send.cpu())
        e2e_steps = max(3, min(a.steps, 10))
        T.allreduce_host(comm, hs, hr)
        comm.sync()
        ms_e2e = timed(lambda: T.allreduce_host(comm, hs, hr), e2e_steps, stream)
        # the host path reduces each segment as its own collective (r2ccl.h): compare
        # with the device path over the same segments
        seg_ref = torch.empty_like(send)
        for lo, hi in host_segments(count, 2):
            w = -(-(hi - lo) // 8) * 8
            buf = torch.zeros((k, w), dtype=send.dtype, device="cuda")
            buf[:, :hi - lo] = send[:, lo:hi]
            T.allreduce(comm, buf, buf, count=hi - lo)
            seg_ref[:, lo:hi] = buf[:, :hi - lo]
        comm.sync()
        res["e2e"] = {"ms": ms_e2e, "h2d": k * S, "d2h": k * S, "steps": e2e_steps,
                      "equal": bool(torch.equal(hr.cuda(), seg_ref))}
        del hs, hr
    comm.finalize()
    if not a.no_fault:
        res["fault"] = [guarded(lambda strat=strat: fault_scenario(
            mk, lambda c: T.allreduce(c, send, recv), ms, S, k, K, g.m, strat, lambda: recv, ref, stream=stream))
            for strat in ("BALANCE", "HOT_REPAIR")]
        res["successive"] = [guarded(lambda strat=strat: successive_scenario(
            mk, lambda c: T.allreduce(c, send, recv), ms, k, K, g.m, strat, lambda: recv, ref, stream=stream))
            for strat in ("BALANCE", "HOT_REPAIR")]
    return res, None


def run_multi(a):
    """N > 1: one process per GPU under torchrun."""
    import torch
    import torch.distributed as dist
    from paper_2512_25059_b200 import build as B
    from paper_2512_25059_b200 import r2ccl as R
    from paper_2512_25059_b200 import torch_api as T
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    if rank == 0:
        B.build()
    dist.init_process_group("gloo")
    dist.barrier()
    B.build()
    K, S = a.channels, a.bytes
    W = a.ctas or 16          # 8 x 16 = 128 CTAs/GPU: best of the W sweep (profiles/r01_summary.md)
    a.chunk = a.chunk or 1024 * 1024   # one chunk per lane and step at N = 2 (profiles/r02_chunk_n24.txt)
    count = S // 2
    send = torch.empty(count, dtype=torch.bfloat16, device="cuda")
    recv = torch.empty_like(send)
    fill_inputs(send, 1234 + rank)

    def mk(strategy):
        c = T.comm_from_env(R.config_default(
            nchannels=K, ctas_per_channel=W, threads_per_cta=a.threads, chunk_bytes=a.chunk, max_bytes=S,
            strategy=strategy, protocol=a.protocol))
        T.register(c, recv)     # collective: recv mapped into every peer
        return c

    comm = mk("BALANCE")
    stream = torch.cuda.current_stream()
    step = lambda c=comm: T.allreduce(c, send, recv)

    def barrier():
        torch.cuda.synchronize()
        dist.barrier()

    def reduce_max(x):
        t = torch.tensor([x], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather(evs):
        out = [None] * world
        dist.all_gather_object(out, evs)
        return [e for part in out for e in part]

    for _ in range(a.warmup):
        step()
    barrier()
    if a.per_step:
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(a.steps + 1)]
        evs[0].record(stream)
        for i in range(a.steps):
            step()
            evs[i + 1].record(stream)
        evs[-1].synchronize()
        d = [evs[i].elapsed_time(evs[i + 1]) for i in range(a.steps)]
        print(f"[rank {rank}] per-step ms: min {min(d):.3f} med {statistics.median(d):.3f} max {max(d):.3f} "
              f"first10 {[round(x, 3) for x in d[:10]]}", file=sys.stderr, flush=True)
        barrier()
    for i in range(a.recreate):
        c2 = mk("BALANCE")
        s2 = lambda: T.allreduce(c2, send, recv)
        for _ in range(3):
            s2()
        barrier()
        t = reduce_max(timed(s2, a.steps, stream))
        t_again = reduce_max(timed(s2, a.steps, stream))
        c2.finalize()
        if rank == 0:
            print(f"recreate {i}: {t:.3f} / {t_again:.3f} ms/step", file=sys.stderr, flush=True)
    if a.clock_test:
        for per in (0, 500, 200, 50, 20, 0):
            barrier()
            if per:
                Clocks.period_ms = per
                with Clocks(local) as c2:
                    t = reduce_max(timed(step, a.steps, stream))
                ns = c2.summary()["samples"]
            else:
                t, ns = reduce_max(timed(step, a.steps, stream)), 0
            if rank == 0:
                print(f"clock-test period {per} ms: {t:.3f} ms/step, {ns} samples", file=sys.stderr, flush=True)
        Clocks.period_ms = a.clock_ms
    # one sampler for all GPUs of the job, live before the barrier that opens
    # the timed region (per-rank samplers starting inside it perturb the run)
    clk = Clocks(",".join(str(i) for i in range(world))) if local == 0 else None
    if clk:
        clk.__enter__()
    # bytes this rank's kernels pushed over NVLink, per channel, counted by the
    # kernel itself (r2_status bytes): hardware NVLink counters are not
    # exposed on these boxes (NVML NOT_SUPPORTED, `nvidia-smi nvlink -gt d`
    # N/A: profiles/r02_nvlink_counters_unavailable.txt) and ncu must not wrap
    # a multi-rank run
    b0 = sum(comm.status()["bytes"][0])
    barrier()
    ms = reduce_max(timed(step, a.steps, stream))
    if clk:
        clk.__exit__(None, None, None)
    barrier()
    assert comm.sync() == R.SUCCESS
    b1 = sum(comm.status()["bytes"][0])
    g = R.geometry(count, R.BFLOAT16, world, K, W, a.chunk)
    res = {"ms": ms, "clocks": clk.summary() if clk else None, "W": W, "m": g.m}
    alg = 2 * (world - 1) / world * S
    res["nvlink_all"] = gather([{"tx_bytes_per_launch": (b1 - b0) / a.steps,
                                 "tx_over_algorithmic": (b1 - b0) / a.steps / alg}])
    if a.ctas_small and not a.profile:
        res["small_footprint"] = guarded(lambda: small_footprint(a, T, R, send, recv, S, world, K, stream, barrier,
                                                                 reduce_max))
    if a.profile:
        return res, rank
    ref = recv.clone()
    def e2e_multi():
        hs = torch.empty(count, dtype=torch.bfloat16).pin_memory()
        hr = torch.empty_like(hs).pin_memory()
        hs.copy_(send.cpu())
        T.allreduce_host(comm, hs, hr)
        comm.sync()
        barrier()
        e2e_steps = max(3, min(a.steps, 10))
        ms_e2e = reduce_max(timed(lambda: T.allreduce_host(comm, hs, hr), e2e_steps, stream))
        # the host path reduces each segment as its own collective (r2ccl.h): compare
        # with the device path over the same segments (into the registered recv)
        for lo, hi in host_segments(count, 2):
            T.allreduce(comm, send[lo:hi], recv[lo:hi])
        comm.sync()
        return {"ms": ms_e2e, "h2d": S, "d2h": S, "steps": e2e_steps, "equal": bool(torch.equal(hr.cuda(), recv))}

    if not a.no_e2e:
        res["e2e"] = guarded(e2e_multi)
    if not a.no_nccl:
        os.environ["NCCL_NVLS_ENABLE"] = "0"
        with stdout_to_stderr():          # NCCL prints its version banner on stdout
            pg = dist.new_group(backend="nccl")
            buf = send.clone()
            for _ in range(3):
                dist.all_reduce(buf, group=pg)
            barrier()
        ms_nccl = reduce_max(timed(lambda: dist.all_reduce(buf, group=pg), a.steps, stream))
        res["nccl"] = {"ms": ms_nccl, "busbw_per_gpu": 2 * (world - 1) / world * S / (ms_nccl * 1e-3) / 1e9,
                       "nvls": "disabled (NCCL_NVLS_ENABLE=0; the paper disabled SHARP)",
                       "version": ".".join(map(str, torch.cuda.nccl.version()))}
    comm.finalize()
    # auxiliary sections: an error there is recorded, never loses the headline line
    if not a.no_coll and world >= 2:
        res["collectives"] = guarded(lambda: coll_section(a, T, R, world, rank, K, W, S, send, recv, stream, barrier,
                                                          reduce_max, pg if not a.no_nccl else None))
    if not a.no_fault and world >= 2:
        res["fault"] = [guarded(lambda strat=strat: fault_scenario(
            mk, lambda c: T.allreduce(c, send, recv), ms, S, world, K, g.m, strat, lambda: recv, ref,
            fault_rank=3 % world, stream=stream, barrier=barrier, reduce_max=reduce_max, is_root=rank == 0,
            gather=gather)) for strat in ("BALANCE", "HOT_REPAIR")]
        res["successive"] = [guarded(lambda strat=strat: successive_scenario(
            mk, lambda c: T.allreduce(c, send, recv), ms, world, K, g.m, strat, lambda: recv, ref,
            fault_rank=3 % world, stream=stream, barrier=barrier, reduce_max=reduce_max, gather=gather))
            for strat in ("BALANCE", "HOT_REPAIR")]
    if not a.no_fault and world >= 2:
        res["bucket_25MB"] = guarded(lambda: bucket_section(a, T, R, mk, send, recv, world, K, W, stream, barrier,
                                                           reduce_max, gather, pg if not a.no_nccl else None))
    if not a.no_fault and world >= 2 and a.bw_model_gbps > 0:
        res["fault_bw_model"] = guarded(lambda: bw_model_section(
            a, T, R, mk, send, recv, ref, S, world, K, W, g.m, stream, barrier, reduce_max, gather))
    if not a.no_fault and world >= 3 and a.bw_model_gbps > 0:
        res["r2cc_allreduce"] = guarded(lambda: r2cc_section(a, T, R, send, recv, S, world, K, W, stream, barrier,
                                                             reduce_max))
        res["rerank"] = guarded(lambda: rerank_section(a, T, R, send, recv, S, world, K, W, stream, barrier,
                                                       reduce_max))
    return res, rank


def bucket_section(a, T, R, mk, send, recv, world, K, W, stream, barrier, reduce_max, gather, pg):
    """BASELINE configs[4]'s bucket: 25,000,000 B bf16 per rank -- the healthy
    time (AUTO protocol) next to NCCL's, then one LINK fault mid-collective and
    the degraded steady state under Balance, unpaced and with channels paced
    as bandwidth units (Balance at 25 MB vs the (K-1)/K bound)."""
    import torch
    cb = 12_500_000
    S_b = cb * 2
    sb, rb = send[:cb], recv[:cb]
    out = {"bytes_per_rank": S_b}
    c = mk("BALANCE")
    step = lambda cc=c: T.allreduce(cc, sb, rb)  # noqa: E731
    for _ in range(3):
        step()
    barrier()
    ms = reduce_max(timed(step, 50, stream))
    assert c.sync() == R.SUCCESS
    out["protocol"] = c.status()["last_protocol"]
    out["ms"] = ms
    out["busbw_per_rank"] = 2 * (world - 1) / world * S_b / (ms * 1e-3) / 1e9
    ref = rb.clone()
    c.finalize()
    if pg is not None:
        import torch.distributed as dist
        buf = sb.clone()
        for _ in range(3):
            dist.all_reduce(buf, group=pg)
        barrier()
        msn = reduce_max(timed(lambda: dist.all_reduce(buf, group=pg), 50, stream))
        out["nccl_ms"] = msn
    g = R.geometry(cb, R.BFLOAT16, world, K, W, a.chunk)
    out["fault_unpaced"] = fault_scenario(mk, lambda cc: T.allreduce(cc, sb, rb), ms, S_b, world, K, g.m, "BALANCE",
                                          lambda: rb, ref, fault_rank=3 % world, b=4096, stream=stream,
                                          barrier=barrier, reduce_max=reduce_max, gather=gather)
    if a.bw_model_gbps > 0:
        def mkp(strategy):
            cc = T.comm_from_env(R.config_default(
                nchannels=K, ctas_per_channel=W, threads_per_cta=a.threads, chunk_bytes=a.chunk, max_bytes=a.bytes,
                strategy=strategy, protocol=a.protocol, channel_gbps=a.bw_model_gbps))
            T.register(cc, recv)
            return cc
        c = mkp("BALANCE")
        step = lambda cc=c: T.allreduce(cc, sb, rb)  # noqa: E731
        for _ in range(3):
            step()
        barrier()
        ms_p = reduce_max(timed(step, 50, stream))
        assert c.sync() == R.SUCCESS
        c.finalize()
        out["paced_healthy_ms"] = ms_p
        out["fault_paced"] = fault_scenario(mkp, lambda cc: T.allreduce(cc, sb, rb), ms_p, S_b, world, K, g.m,
                                            "BALANCE", lambda: rb, ref, fault_rank=3 % world, b=4096, stream=stream,
                                            barrier=barrier, reduce_max=reduce_max, gather=gather)
    return out


def small_footprint(a, T, R, send, recv, S, world, K, stream, barrier, reduce_max):
    """The headline allreduce with W = --ctas-small CTAs per channel (K x W
    CTAs per GPU instead of K x 16): what the bandwidth costs in SMs
    (weakness 6).  Result compared with the headline run's."""
    import torch
    want = recv.clone()
    c = T.comm_from_env(R.config_default(
        # 512 KiB chunks: with 4 CTAs per channel a lane then carries 4 chunks per step, whose
        # retires overlap the next chunk's transfer (N=2: 1 MiB 537 GB/s, 512 KiB 566; profiles/r02_summary.md)
        nchannels=K, ctas_per_channel=a.ctas_small, threads_per_cta=a.threads, chunk_bytes=512 * 1024, max_bytes=S,
        strategy="BALANCE", protocol=a.protocol))
    T.register(c, recv)
    step = lambda: T.allreduce(c, send, recv)  # noqa: E731
    for _ in range(3):
        step()
    barrier()
    ms = reduce_max(timed(step, a.steps, stream))
    assert c.sync() == R.SUCCESS
    equal = bool(torch.equal(recv, want))
    c.finalize()
    barrier()
    return {"ctas_per_gpu": K * a.ctas_small, "ctas_per_channel": a.ctas_small, "ms": ms,
            "busbw_per_rank": 2 * (world - 1) / world * S / (ms * 1e-3) / 1e9,
            "frac_of_770": 2 * (world - 1) / world * S / (ms * 1e-3) / 1e9 / 770.0, "result_equal_headline": equal}


def degrade(c, T, R, f, chans, send, recv, barrier):
    """Kill endpoint (f, c) for c in chans as a real failure would: a LOCAL
    fault mid-collective, triangulated to LOCAL_ENDPOINT(f) by the monitors
    (dead from the next collective on)."""
    import time as _t
    for ch in chans:
        s = c.status()["seq"] + 1
        c.inject_fault(at_seq=s, kind="LOCAL", src_rank=f, channel=ch, step=0, chunk=0, byte_offset=0)
        T.allreduce(c, send[:4096], recv[:4096])
        assert c.sync() == R.SUCCESS
        t0 = _t.time()
        while (f, ch) not in c.status()["dead_endpoints"] and _t.time() - t0 < 10:
            _t.sleep(0.002)
        barrier()


def rerank_section(a, T, R, send, recv, S, world, K, W, stream, barrier, reduce_max):
    """disjoint endpoint losses on neighbouring ranks (rank 1
    loses channel 1, rank 2 loses channel 2), channels as bandwidth
    units (channel_gbps).  Rank order leaves the edge 1 -> 2 with K-2
    channels; Algorithm 1's R' keeps every edge at >= K-1.  Both runs are
    Balance rings on the same degraded communicator; result compared."""
    import torch
    out = {"channel_gbps": a.bw_model_gbps, "lost": [[1, 1], [2, 2]], "cases": {}}
    results = {}
    for rr in (0, 1):
        c = T.comm_from_env(R.config_default(
            nchannels=K, ctas_per_channel=W, threads_per_cta=a.threads, chunk_bytes=a.chunk, max_bytes=S,
            strategy="BALANCE", protocol="SIMPLE", channel_gbps=a.bw_model_gbps, allreduce_algo="RING", rerank=rr))
        T.register(c, recv)
        degrade(c, T, R, 1, [1], send, recv, barrier)
        degrade(c, T, R, 2, [2], send, recv, barrier)
        step = lambda cc=c: T.allreduce(cc, send, recv)  # noqa: E731
        for _ in range(3):
            step()
        barrier()
        ms = reduce_max(timed(step, 20, stream))
        assert c.sync() == R.SUCCESS
        st = c.status()
        results[rr] = recv.clone()
        out["cases"]["rerank" if rr else "rank_order"] = {
            "ms": ms, "busbw_per_rank": 2 * (world - 1) / world * S / (ms * 1e-3) / 1e9,
            "ring_order": st["ring_order"], "n_rerank": st["n_rerank"]}
        c.finalize()
        barrier()
    out["speedup"] = out["cases"]["rank_order"]["ms"] / out["cases"]["rerank"]["ms"]
    # the two rings fold in different orders: equal for bf16 only up to rounding, so compare with the
    # tolerance the north star states (normwise, bf16 <= 1e-2)
    d = (results[0].float() - results[1].float()).norm() / results[1].float().norm()
    out["normwise_diff_vs_rank_order"] = float(d)
    return out


def r2cc_section(a, T, R, send, recv, S, world, K, W, stream, barrier, reduce_max):
    """one rank f loses d of its K channels (X = d/K lost
    bandwidth, channels as bandwidth units via channel_gbps).  Above App. A's
    threshold n/(3n-2) the planner runs R²CCL-AllReduce (global ring on f's
    healthy channels + partial ring of the healthy ranks on f's dead ones, then
    the tailored broadcast); compared with the Balance ring on the same
    degraded communicator.  Times are max over ranks of the CUDA-event mean."""
    f = 1 % world
    out = {"channel_gbps": a.bw_model_gbps, "degraded_rank": f, "threshold_X": world / (3 * world - 2), "cases": []}
    for d in (K // 2, 3 * K // 4):
        row = {"dead_channels": d, "X": d / K}
        for algo in ("RING", "R2CC", "AUTO"):
            c = T.comm_from_env(R.config_default(
                nchannels=K, ctas_per_channel=W, threads_per_cta=a.threads, chunk_bytes=a.chunk, max_bytes=S,
                strategy="BALANCE", protocol="SIMPLE", channel_gbps=a.bw_model_gbps, allreduce_algo=algo))
            T.register(c, recv)
            degrade(c, T, R, f, list(range(d)), send, recv, barrier)
            step = lambda cc=c: T.allreduce(cc, send, recv)  # noqa: E731
            for _ in range(3):
                step()
            barrier()
            ms = reduce_max(timed(step, 20, stream))
            assert c.sync() == R.SUCCESS
            st = c.status()
            row[algo.lower()] = {"ms": ms, "busbw_per_rank": 2 * (world - 1) / world * S / (ms * 1e-3) / 1e9,
                                 "r2cc_calls": st["r2cc"]["calls"]}
            if algo == "R2CC":
                row["Y"] = st["r2cc"]["Y"]
                row["NA_NP"] = [st["r2cc"]["NA"], st["r2cc"]["NP"]]
            if algo == "AUTO":       # the alpha-beta choice (reading R-11)
                row["auto_chose"] = "R2CC" if st["r2cc"]["calls"] > 0 else "RING"
            c.finalize()
            barrier()
        row["r2cc_speedup_over_ring"] = row["ring"]["ms"] / row["r2cc"]["ms"]
        out["cases"].append(row)
    return out


def bw_model_section(a, T, R, mk_default, send, recv, ref, S, world, K, W, m, stream, barrier, reduce_max, gather):
    """Config 3 with channels as bandwidth units (r2ccl.h channel_gbps): every
    lane paces its sends to channel_gbps / W, as a NIC would, so one dead
    channel of K costs bandwidth -- the setting of the paper's surviving-
    bandwidth bound (Balance (K-1)/K, HotRepair 1/2)."""
    def mk(strategy):
        c = T.comm_from_env(R.config_default(
            nchannels=K, ctas_per_channel=W, threads_per_cta=a.threads, chunk_bytes=a.chunk, max_bytes=S,
            strategy=strategy, protocol=a.protocol, channel_gbps=a.bw_model_gbps))
        T.register(c, recv)
        return c
    c = mk("BALANCE")
    step = lambda: T.allreduce(c, send, recv)  # noqa: E731
    for _ in range(3):
        step()
    barrier()
    ms_h = reduce_max(timed(step, 20, stream))
    assert c.sync() == R.SUCCESS
    c.finalize()
    out = {"channel_gbps": a.bw_model_gbps, "ms_healthy": ms_h,
           "busbw_per_rank_healthy": 2 * (world - 1) / world * S / (ms_h * 1e-3) / 1e9, "fault": []}
    for strat in ("BALANCE", "HOT_REPAIR"):
        out["fault"].append(fault_scenario(mk, lambda cc: T.allreduce(cc, send, recv), ms_h, S, world, K, m, strat,
                                           lambda: recv, ref, fault_rank=3 % world, stream=stream, barrier=barrier,
                                           reduce_max=reduce_max, gather=gather))
    return out


def ncu_traffic(a, n_ranks, W):
    """DRAM bytes per launch from the committed ncu --set full capture of this
    exact workload (the newest profiles/rNN_ncu_traffic.json, tools/ncu_traffic.py), else None."""
    import glob
    found = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles",
                                          "r[0-9][0-9]_ncu_traffic.json")))
    if not found:
        return None, None
    path = found[-1]
    if not (n_ranks == 8 and a.bytes == 256 * MIB and a.channels == 8 and W == 2 and a.chunk == 512 * 1024):
        return None, None
    try:
        with open(path) as f:
            d = json.load(f)
        return d["dram_bytes_per_launch"], d["source"]
    except (OSError, KeyError, ValueError):
        return None, None


def report(a, res, n_gpus, n_ranks, mode):
    P = peaks()
    S, K = a.bytes, a.channels
    ms = res["ms"]
    busbw_rank = 2 * (n_ranks - 1) / n_ranks * S / (ms * 1e-3) / 1e9
    agg = busbw_rank * n_ranks
    if mode == "sim":
        hbm = (5 * n_ranks - 4) * S
        peak = P.get("hbm_gbs", 6650.0)
        traffic, tsrc = ncu_traffic(a, n_ranks, res["W"])
        roof = {"bound": "hbm", "achieved": hbm / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": hbm / (ms * 1e-3) / 1e9 / peak, "traffic": traffic, "traffic_source": tsrc,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in P else "fallback 6.65 TB/s",
                "algorithmic_bytes_per_launch": hbm,
                "per_unit": "(5k-4) x S HBM bytes per simulated allreduce (SURVEY §8(d)), k=%d" % n_ranks}
    else:
        nv = 2 * (n_ranks - 1) / n_ranks * S
        peak = 770.0
        counters = res.get("nvlink_all") or []
        traffic = (statistics.mean(x["tx_bytes_per_launch"] for x in counters)
                   if counters and len(counters) == n_ranks else None)
        roof = {"bound": "nvlink", "achieved": nv / (ms * 1e-3) / 1e9, "peak": peak, "unit": "GB/s",
                "frac": nv / (ms * 1e-3) / 1e9 / peak, "traffic": traffic,
                "traffic_source": ("kernel-counted NVLink bytes per launch (mean over ranks; r2_status bytes): "
                                   "hardware NVLink counters are not exposed on these boxes "
                                   "(profiles/r02_nvlink_counters_unavailable.txt) and ncu must not wrap "
                                   "multi-rank runs"),
                "traffic_over_algorithmic": traffic / nv if traffic else None,
                "traffic_per_rank": [x["tx_bytes_per_launch"] for x in counters],
                "peak_source": "B200_PROFILING.md measured peer copy 770 GB/s/direction (900 nominal)",
                "sm_store_peak_gbs": 697.0,
                "sm_store_peak_source": "profiles/r01_p2p_store_n4.log: SM/TMA peer-store ceiling (copy engine 760)",
                "frac_of_nominal_900": nv / (ms * 1e-3) / 1e9 / 900.0,
                "algorithmic_bytes_per_launch": nv, "per_unit": "2(n-1)/n x S NVLink bytes per GPU"}
    line = {
        "metric": "allreduce aggregate bus bandwidth, 256 MiB bf16 per rank, healthy (+1-fault scenario in 'fault')",
        "value": agg, "unit": "GB/s", "n_gpus": n_gpus, "steps": a.steps, "warmup": a.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": {"workload": ("allreduce %d MiB bf16/rank, %d %s ranks, K=%d channels x W=%d CTAs, %d KiB chunks"
                                % (S // MIB, n_ranks, "simulated (1 GPU)" if mode == "sim" else "GPU", K, res["W"],
                                   a.chunk // 1024)),
                   "bytes_per_rank": S, "ranks": n_ranks, "mode": mode, "channels": K, "ctas_per_channel": res["W"],
                   "threads_per_cta": a.threads,
                   "chunks_per_slice": res["m"], "l2": "inputs larger than L2 (no flush)",
                   "parallelism": f"ring allreduce over {n_ranks} ranks"},
        "busbw_per_rank": busbw_rank,
        "roofline": roof,
        "gpu_launches": a.steps,
        "clocks": res["clocks"],
    }
    if "e2e" in res and "error" in res["e2e"]:
        line["e2e"] = res["e2e"]
    elif "e2e" in res:
        e = res["e2e"]
        line["e2e"] = {"value": 2 * (n_ranks - 1) / n_ranks * S / (e["ms"] * 1e-3) / 1e9 * n_ranks, "unit": "GB/s",
                       "h2d_bytes_per_step": e["h2d"], "d2h_bytes_per_step": e["d2h"], "ms_per_step": e["ms"],
                       "result_equal_device_path": e["equal"],
                       "api": "r2_allreduce_host (C ABI, pinned host buffers; segmented + pipelined from 8 MiB on, "
                              "compared with the device path over the same segments)"}
    if "nccl" in res:
        line["nccl_same_box"] = res["nccl"]
    if "small_footprint" in res:
        line["small_footprint"] = res["small_footprint"]
    if "collectives" in res:
        line["collectives"] = res["collectives"]
    if "fault" in res:
        line["fault"] = res["fault"]
    if "successive" in res:
        line["successive_failover"] = res["successive"]
    if "fault_bw_model" in res:
        line["fault_bandwidth_model"] = res["fault_bw_model"]
    if "r2cc_allreduce" in res:
        line["r2cc_allreduce"] = res["r2cc_allreduce"]
    if "rerank" in res:
        line["rerank"] = res["rerank"]
    if "bucket_25MB" in res:
        line["bucket_25MB"] = res["bucket_25MB"]
    return line


def main():
    a = parse()
    if a.impl == "reference":
        return reference_arm(a)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if not a.threads:
        a.threads = 256 if world > 1 else 512
    if world > 1:
        res, rank = run_multi(a)
        if rank == 0:
            print(json.dumps(report(a, res, world, world, "multi")), flush=True)
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()
        return
    res, _ = run_sim(a)
    line = report(a, res, 1, a.sim_ranks, "sim")
    if not a.no_cpu and not a.profile:
        s = 128 * MIB
        r = oracle_rate(a.sim_ranks, s)
        line["cpu_baseline"] = {"value": r["agg_busbw_GBs"], "unit": "GB/s", "cores": 1, "kind": "oracle",
                                "sample": f"{a.sim_ranks} ranks x {s // MIB} MiB bf16 (1/{a.bytes // s} of the "
                                          f"per-rank payload), oracle/protocol.py Layer 2, fault-free, 1 thread, "
                                          f"{r['seconds']:.1f} s on {cpu_info()} ({os.cpu_count()} cores on host)"}
    print(json.dumps(line), flush=True)


def reference_arm(a):
    """The oracle as it stands, timed on the host cores (bounded samples)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    k = a.sim_ranks if int(os.environ.get("WORLD_SIZE", "1")) == 1 else int(os.environ["WORLD_SIZE"])
    s = 1 * MIB
    oracle_rate(k, s)    # warm
    ts = []
    for _ in range(a.warmup):
        oracle_rate(k, s)
    for _ in range(a.steps):
        ts.append(oracle_rate(k, s)["seconds"])
    t = sum(ts) / len(ts)
    v = k * 2 * (k - 1) / k * s / t / 1e9
    line = {"impl": "reference",
            "metric": "allreduce aggregate bus bandwidth, 256 MiB bf16 per rank, healthy (+1-fault scenario in 'fault')",
            "value": v, "unit": "GB/s", "n_gpus": int(os.environ.get("WORLD_SIZE", "1")), "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": t * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": f"allreduce bf16, {k} ranks, sample {s // MIB} MiB/rank per step (oracle)"},
            "cpu_baseline": {"value": v, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"{k} ranks x {s // MIB} MiB bf16 per step, oracle/protocol.py Layer 2, "
                                       f"1 thread on {cpu_info()}"},
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
