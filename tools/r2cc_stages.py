"""R²CCL-AllReduce stage timing on one GPU (simulated ranks, channels paced as
bandwidth units): the Balance ring and R²CCL-AllReduce on the same degraded
communicator (rank 1 loses d of K channels).  Run under
`ncu --metrics gpu__time_duration.sum` for per-launch (per-stage) durations;
plain, it prints CUDA-event times per call."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import r2inputs  # noqa: E402
from tests.gpu_util import poisoned, to_dev  # noqa: E402
from paper_2512_25059_b200 import build as B  # noqa: E402
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def main():
    B.build()
    torch.cuda.set_device(0)
    n, K, W = 4, 8, 4
    N = int(os.environ.get("N", 32 << 20))          # elements per rank (bf16)
    d = int(os.environ.get("DEAD", 4))
    gbps = int(os.environ.get("GBPS", 20))
    iters = int(os.environ.get("ITERS", 5))
    for algo in ("RING", "R2CC"):
        comm = R.Comm(0, 1, 0, None, R.config_default(sim_ranks=n, nchannels=K, ctas_per_channel=W,
                                                      max_bytes=2 * N, channel_gbps=gbps, allreduce_algo=algo,
                                                      protocol="SIMPLE"))
        for c in range(d):
            s = comm.status()["seq"] + 1
            comm.inject_fault(at_seq=s, kind="LOCAL", src_rank=1, channel=c, step=0, chunk=0, byte_offset=0)
            xs = r2inputs.inputs(n, 256, "int32", seed=c)
            T.allreduce(comm, to_dev(xs, "int32"), poisoned(n, 256, "int32"), count=256)
            assert comm.sync() == R.SUCCESS
            t0 = time.time()
            while (1, c) not in comm.status()["dead_endpoints"] and time.time() - t0 < 5:
                time.sleep(0.002)
        x = torch.randn((n, N), device="cuda").to(torch.bfloat16)
        y = torch.empty_like(x)
        for _ in range(2):
            T.allreduce(comm, x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            T.allreduce(comm, x, y)
        e1.record()
        e1.synchronize()
        assert comm.sync() == R.SUCCESS
        st = comm.status()
        # device timeline of the LAST launch of one more call (R2_TRACE=1): for
        # R²CCL-AllReduce that is stage 2, the tailored broadcast
        tr = None
        if os.environ.get("R2_TRACE") == "1":
            import ctypes as C
            buf = (C.c_uint64 * 64)()
            R.lib().r2_trace(comm._h, 0, buf)            # arm
            f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            f0.record()
            T.allreduce(comm, x, y)
            f1.record()
            f1.synchronize()
            R.lib().r2_trace(comm._h, 0, buf)
            b = buf[0]
            tr = (f0.elapsed_time(f1), (buf[62] - b) / 1e6, (buf[1] - b) / 1e6)
        print(f"{algo}: {e0.elapsed_time(e1) / iters:.3f} ms/call  r2cc calls {st['r2cc']['calls']} "
              f"Y {st['r2cc']['Y']:.3f} NA/NP {st['r2cc']['NA']}/{st['r2cc']['NP']}"
              + (f"  | one call {tr[0]:.3f} ms, last launch first-CTA-start -> last exit {tr[1]:.3f} ms" if tr else ""),
              flush=True)
        if algo == "RING" and os.environ.get("BCAST"):
            # the same degraded communicator: a plain Broadcast chain from rank 1
            # over the stage-2 payload (R²CCL's Y share of the buffer)
            NP = int(N * float(os.environ.get("BCAST"))) // 8 * 8
            xb = x[:, :NP].contiguous()
            yb = torch.empty_like(xb)
            for _ in range(2):
                T.broadcast(comm, xb, yb, root=1)
            torch.cuda.synchronize()
            g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            g0.record()
            for _ in range(iters):
                T.broadcast(comm, xb, yb, root=1)
            g1.record()
            g1.synchronize()
            assert comm.sync() == R.SUCCESS
            print(f"BROADCAST root 1, {NP} elements: {g0.elapsed_time(g1) / iters:.3f} ms/call", flush=True)
        comm.finalize()


if __name__ == "__main__":
    main()
