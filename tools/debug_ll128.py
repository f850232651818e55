"""Debug: LL128 with a mid-call LINK fault under speculation (the case of
tests/test_gpu_ll.py::test_ll_speculation_with_midcall_fault_many_points).
For each fault point, prints the wrong elements mapped onto the geometry
(shard, channel, chunk, vector in chunk, line) and the events."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import r2inputs  # noqa: E402
from oracle import semantic as OS  # noqa: E402
from tests.gpu_util import oracle_geom, run, sim_comm  # noqa: E402
from oracle.geometry import Geometry  # noqa: E402
from tests.scenario import effective_chunk_bytes  # noqa: E402
from paper_2512_25059_b200 import build as B  # noqa: E402
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402


def main():
    B.build()
    torch.cuda.set_device(0)
    proto = os.environ.get("PROTO", "LL128")
    n, K, W, N = 4, 3, 2, 40_000
    for strategy in ("BALANCE", "HOT_REPAIR"):
        for b in (64, 0, 1024):
            for t in range(0, 7):
                comm = sim_comm(n, K, W, 4096, strategy=strategy, protocol=proto)
                xs = r2inputs.inputs(n, N, "bfloat16", seed=12)
                E = 2
                g = Geometry(n, K, N, E, effective_chunk_bytes(N, n, K, E, 4096, W), ll=True)
                if g.local(t):
                    continue
                comm.inject_fault(at_seq=1, kind="LINK", src_rank=t % n, channel=t % K, step=t, chunk=0,
                                  byte_offset=b, poison=1)
                rc, out = run(comm, xs, "bfloat16")
                y = OS.allreduce(xs, g.shard, "bfloat16")
                bad = {}
                for r in range(n):
                    idx = np.nonzero(out[r].view(np.uint16) != y.view(np.uint16))[0]
                    if len(idx):
                        bad[r] = idx
                ev = comm.events()
                print(f"{strategy} b={b} t={t} rc={rc} bad_ranks={ {r: len(v) for r, v in bad.items()} } "
                      f"events={[(e['rank'], e['origin'], e['stopped_channel'], e['resume'], e['retransmit']) for e in ev]}",
                      flush=True)
                V = 8
                for r, idx in list(bad.items())[:1]:
                    for i in idx[:6]:
                        s, off = divmod(int(i), g.shard)
                        c, o2 = divmod(off, g.slice)
                        j, o3 = divmod(o2, g.chunk)
                        v = o3 // V
                        print(f"   rank {r} elem {i}: shard {s} ch {c} chunk {j} vec {v} line {v // 7} pos {v % 7} "
                              f"got {out[r][i]:#06x} want {y[i]:#06x}")
                comm.finalize()


if __name__ == "__main__":
    main()
