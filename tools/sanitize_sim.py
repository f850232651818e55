"""compute-sanitizer target (SURVEY §5 race detection): simulated-rank
collectives on one GPU -- healthy AllReduce (SIMPLE and LL protocols, int32
and bf16) and one AllReduce with a LINK fault mid-chunk (the
failover runs through the resident service lane, so it works while the
sanitizer serialises kernels).  Every result is checked against the oracle.

    compute-sanitizer --tool memcheck python tools/sanitize_sim.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import r2inputs  # noqa: E402
from tests.gpu_util import check_result, oracle_geom, poisoned, sim_comm, to_dev, to_np  # noqa: E402
from paper_2512_25059_b200 import build as B  # noqa: E402
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def allreduce(comm, xs, dt, N):
    send = to_dev(xs, dt)
    recv = poisoned(comm.n, N, dt)
    T.allreduce(comm, send, recv, count=N)
    rc = comm.sync()
    assert rc == R.SUCCESS, rc
    out = to_np(recv, dt)[:, :N]
    check_result(out, xs, oracle_geom(comm, N, dt), dt)


def main():
    B.build()
    torch.cuda.set_device(0)
    n, N = 4, 50_003
    for proto in ("SIMPLE", "LL"):
        comm = sim_comm(n, K=2, W=2, chunk_bytes=16384, protocol=proto, watchdog_ms=120000)
        for dt in ("int32", "bfloat16"):
            allreduce(comm, r2inputs.inputs(n, N, dt, seed=1), dt, N)
        comm.finalize()
        print(f"healthy {proto}: ok", flush=True)
    comm = sim_comm(n, K=2, W=2, chunk_bytes=16384, watchdog_ms=120000)
    comm.inject_fault(at_seq=1, kind="LINK", src_rank=1, channel=0, step=1, chunk=1, byte_offset=4096, poison=1)
    allreduce(comm, r2inputs.inputs(n, N, "float32", seed=2), "float32", N)
    ev = comm.events()
    assert len(ev) == 1 and ev[0]["verdict"] == "LINK", ev
    print(f"LINK fault recovered under the sanitizer: failover {ev[0]['failover_ms']:.3f} ms", flush=True)
    comm.finalize()
    print("sanitize_sim: all collectives completed and matched the oracle")


if __name__ == "__main__":
    main()
