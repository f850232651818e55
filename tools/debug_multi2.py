"""Debug (torchrun, 4 GPUs): the worker's degraded-steady-state case after a
LINK fault, per (rerank, protocol): ok / protocol / ring order / bad spots."""
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from tests import mgpu_worker as MW  # noqa: E402
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def main():
    dist.init_process_group("gloo")
    rank, world = dist.get_rank(), dist.get_world_size()
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    for rr in (0, 1):
        for proto in ("SIMPLE", "LL", "LL128", "AUTO"):
            cfg = R.config_default(nchannels=4, ctas_per_channel=2, chunk_bytes=64 * 1024, max_bytes=64 << 20,
                                   strategy="BALANCE", rerank=rr, protocol=proto)
            comm = T.comm_from_env(cfg)
            a = MW.case(comm, rank, world, 100_003, "float32", seed=1)
            f = dict(kind="LINK", src_rank=world - 1, channel=1, step=max(0, world - 2), chunk=1,
                     byte_offset=12345, poison=1)
            b = MW.case(comm, rank, world, 1 << 20, "bfloat16", [f], "BALANCE", seed=11)
            st = comm.status()
            c = MW.case(comm, rank, world, 1 << 20, "float32", seed=12)
            st2 = comm.status()
            d = MW.case(comm, rank, world, 100_003, "int32", seed=13)
            if rank == 0:
                print(f"rerank={rr} proto={proto}: healthy ok={a['ok']} ({a['protocol']}) | fault ok={b['ok']} "
                      f"({b['protocol']}) dead_links={st['dead_links']} | degraded ok={c['ok']} ({c['protocol']}) "
                      f"ring={st2['ring_order']} | degraded int ok={d['ok']} ({d['protocol']})", flush=True)
            comm.finalize()
            dist.barrier()


if __name__ == "__main__":
    main()
