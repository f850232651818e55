"""Debug helper: run one sim-mode allreduce (optionally faulted) and report
mismatches against the oracle mapped to (shard, channel, chunk)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import r2inputs  # noqa: E402
from oracle import protocol as OP  # noqa: E402
from oracle import semantic as OS  # noqa: E402
from tests.gpu_util import oracle_geom, run, sim_comm  # noqa: E402


def main():
    a = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
    n, K, W, N = a.get("n", 4), a.get("K", 2), a.get("W", 2), a.get("N", 65536)
    dtype, chunk = a.get("dtype", "bfloat16"), a.get("chunk", 16384)
    faults = a.get("faults", [])
    strategy = a.get("strategy", "BALANCE")
    comm = sim_comm(n, K, W, chunk, strategy=strategy, watchdog_ms=a.get("watchdog_ms", 3000),
                    max_bytes=max(16 << 20, N * (2 if dtype == "bfloat16" else 4)))
    for f in faults:
        comm.inject_fault(at_seq=1, **f)
    xs = r2inputs.inputs(n, N, dtype)
    rc, out = run(comm, xs, dtype, inplace=a.get("inplace", False))
    g = oracle_geom(comm, N, dtype)
    y = OS.allreduce(xs, g.shard, dtype)
    print("rc", rc, "geom m", g.m, "chunk elems", g.chunk, "slice", g.slice, "shard", g.shard)
    for r in range(n):
        bad = np.nonzero(out[r].view(np.uint16 if dtype == "bfloat16" else np.uint32) !=
                         y.view(np.uint16 if dtype == "bfloat16" else np.uint32))[0]
        if len(bad):
            keys = {}
            for i in bad:
                s, rem = divmod(int(i), g.shard)
                c, rem = divmod(rem, g.slice)
                j = rem // g.chunk
                keys[(s, c, j)] = keys.get((s, c, j), 0) + 1
            print(f"rank {r}: {len(bad)} bad elems; (shard,ch,chunk)->count {dict(list(keys.items())[:20])}")
            i = int(bad[0])
            print("   first", i, "got", out[r][i], "want", y[i])
        else:
            print(f"rank {r}: ok")
    for e in comm.events():
        print("event", {k: e[k] for k in ("rank", "origin", "stopped_channel", "verdict", "resume", "floor",
                                          "retransmit", "failover_ms")})
    print("status", comm.status())
    if faults:
        res = OP.simulate(xs, g, dtype, faults=[OP.Fault(f["kind"], f["src_rank"], f["channel"], f["step"],
                                                         f["chunk"], f.get("byte_offset", 0)) for f in faults],
                          strategy=strategy, seed=0)
        print("oracle events", [{k: e[k] for k in ("rank", "origin", "resume", "retransmit")} for e in res.events])
        print("oracle bytes", res.bytes_sent.tolist())


if __name__ == "__main__":
    main()
