"""Debug helper (torchrun): one faulted 256 MiB bf16 allreduce across the job's
GPUs; run with R2_DEBUG=1 to get every rank's control-plane trace."""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    S = int(os.environ.get("BYTES", 256 << 20))
    comm = T.comm_from_env(R.config_default(nchannels=8, ctas_per_channel=16, max_bytes=S,
                                            strategy=os.environ.get("STRATEGY", "BALANCE")))
    x = torch.randn(S // 2, device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    T.register(comm, y)
    for _ in range(3):
        T.allreduce(comm, x, y)
    torch.cuda.synchronize()
    dist.barrier()
    seq = comm.status()["seq"] + 1
    comm.inject_fault(at_seq=seq, kind=os.environ.get("KIND", "LINK"), src_rank=3 % world, channel=5, step=1,
                      chunk=4, byte_offset=4096)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    T.allreduce(comm, x, y)
    e1.record()
    e1.synchronize()
    rc = comm.sync()
    evs = comm.events()
    fire = [e["t_fire_dev_ns"] for e in evs]
    retx = [e["t_first_retx_dev_ns"] for e in evs]
    print(f"[rank {rank}] rc {rc} faulted call {e0.elapsed_time(e1):.3f} ms fire {fire} retx {retx} events "
          f"{[(e['rank'], e['origin'], e['verdict'], e['resume'], round(e['failover_ms'], 3)) for e in evs]}",
          file=sys.stderr, flush=True)
    dist.barrier()
    comm.finalize()


if __name__ == "__main__":
    main()
