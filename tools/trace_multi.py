"""Device timeline of one small / one large allreduce (torchrun, R2_TRACE=1).

Prints, per rank, the r2_trace slots relative to the first CTA start (us).
"""
import ctypes as C
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("R2_TRACE", "1")
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def trace(comm):
    buf = (C.c_uint64 * 64)()
    rc = R.lib().r2_trace(comm._h, 0, buf)
    assert rc == 0, rc
    return list(buf)


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    W = int(os.environ.get("W", 16))
    sizes = [int(s) for s in os.environ.get("SIZES", "65536,16777216,268435456").split(",")]
    proto = os.environ.get("PROTO", "AUTO")
    comm = T.comm_from_env(R.config_default(nchannels=8, ctas_per_channel=W, max_bytes=max(sizes), protocol=proto,
                                            chunk_bytes=int(os.environ.get("CHUNK", 512 * 1024))))
    steps = 2 * world - 1
    for S in sizes:
        x = torch.randn(S // 2, device="cuda").to(torch.bfloat16)
        y = torch.empty_like(x)
        T.register(comm, y)
        for _ in range(3):
            T.allreduce(comm, x, y)
        torch.cuda.synchronize()
        dist.barrier()
        trace(comm)  # arm
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        T.allreduce(comm, x, y)
        e1.record()
        e1.synchronize()
        tr = trace(comm)
        b = tr[0]
        rel = lambda v: (v - b) / 1e3 if 0 < v < (1 << 63) and v >= b else float("nan")  # noqa: E731
        pub = " ".join(f"{rel(tr[32 + t]):.1f}" for t in range(steps))
        ret = " ".join(f"{rel(tr[4 + t]):.1f}" for t in range(steps))
        line = (f"[rank {rank}] {comm.status()['last_protocol']} S={S >> 10}KiB event {e0.elapsed_time(e1) * 1e3:.1f}us | init {rel(tr[1]):.1f} "
                f"first-pub {rel(tr[2]):.1f} | step first-publish: {pub} | step last-retire: {ret} | ctl-end "
                f"{rel(tr[60]):.1f} drain {rel(tr[61]):.1f} exit {rel(tr[62]):.1f}")
        if os.environ.get("R2_TRACE") == "2":
            line += " | data take: " + " ".join(f"{rel(tr[40 + i]):.1f}" for i in range(8))
            line += " | data done: " + " ".join(f"{rel(tr[48 + i]):.1f}" for i in range(8))
            line += " | ctl publish: " + " ".join(f"{rel(tr[24 + i]):.1f}" for i in range(8))
            line += " | ctl retire: " + " ".join(f"{rel(tr[16 + i]):.1f}" for i in range(8))
        for r in range(world):
            if r == rank:
                print(line, file=sys.stderr, flush=True)
            dist.barrier()
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()
