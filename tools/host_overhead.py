"""Host enqueue cost vs GPU time per small collective (torchrun): is the
latency floor host-bound?"""
import os
import sys
import time

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank = dist.get_rank()
    comm = T.comm_from_env(R.config_default(nchannels=8, ctas_per_channel=16, max_bytes=1 << 20))
    x = torch.randn(512, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    T.register(comm, y)
    s = torch.cuda.current_stream()
    for _ in range(20):
        comm.allreduce(x.data_ptr(), y.data_ptr(), 512, R.BFLOAT16, s.cuda_stream)
    torch.cuda.synchronize()
    dist.barrier()
    n = 500
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    t0 = time.perf_counter()
    for _ in range(n):
        comm.allreduce(x.data_ptr(), y.data_ptr(), 512, R.BFLOAT16, s.cuda_stream)
    t1 = time.perf_counter()
    e1.record(s)
    e1.synchronize()
    host_us = (t1 - t0) / n * 1e6
    gpu_us = e0.elapsed_time(e1) / n * 1e3
    print(f"[rank {rank}] host enqueue {host_us:.1f} us/call, gpu {gpu_us:.1f} us/call", file=sys.stderr, flush=True)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()
