"""Device timeline of one small LL AllReduce in the middle of a back-to-back
loop, simulated ranks on one GPU (R2_TRACE=1: min/max over all CTAs).
Prints the r2_trace slots relative to the first CTA start (us)."""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("R2_TRACE", "1")
from paper_2512_25059_b200 import build as B  # noqa: E402
from paper_2512_25059_b200 import r2ccl as R  # noqa: E402
from paper_2512_25059_b200 import torch_api as T  # noqa: E402


def main():
    B.build()
    torch.cuda.set_device(0)
    n = int(os.environ.get("SIM", 4))
    comm = R.Comm(0, 1, 0, None, R.config_default(sim_ranks=n, nchannels=8, ctas_per_channel=4,
                                                  protocol=os.environ.get("PROTO", "LL"),
                                                  max_bytes=64 << 20))
    x = torch.randn((n, int(os.environ.get("ELEMS", 512))), device="cuda").to(torch.bfloat16)
    y = torch.empty_like(x)
    buf = (C.c_uint64 * 64)()
    steps = 2 * n - 1
    for rep in range(3):
        for _ in range(20):
            T.allreduce(comm, x, y)
        R.lib().r2_trace(comm._h, 0, buf)               # arm (synchronizes)
        T.allreduce(comm, x, y)                           # the traced call
        torch.cuda.synchronize()
        R.lib().r2_trace(comm._h, 0, buf)
        b = buf[0]
        rel = lambda v: (v - b) / 1e3 if 0 < v < (1 << 63) and v >= b else float("nan")  # noqa: E731
        print(f"init {rel(buf[1]):.1f} first-pub {rel(buf[2]):.1f} | step first-publish: "
              + " ".join(f"{rel(buf[32 + t]):.1f}" for t in range(steps)) + " | step last-retire: "
              + " ".join(f"{rel(buf[4 + t]):.1f}" for t in range(steps))
              + f" | ctl-end {rel(buf[60]):.1f} drain {rel(buf[61]):.1f} exit {rel(buf[62]):.1f}", flush=True)
        if os.environ.get("R2_TRACE") == "3":
            cyc = lambda c, k: f"{c / max(k, 1):.0f} cyc x {k}"  # noqa: E731
            print(f"   control lane of CTA 0: try_publish {cyc(buf[50], buf[51])}, iter_next {cyc(buf[52], buf[53])}, "
                  f"retire {cyc(buf[54], buf[55])} per chunk, control_run total {buf[56]} cyc", flush=True)
            k = max(buf[51], 1)
            print("   try_publish phases (cyc per publish): faults %.0f, control check %.0f, input word %.0f, "
                  "recv/pace %.0f, slot build %.0f, store+arrive %.0f" % tuple(buf[40 + i] / k for i in range(6)),
                  flush=True)
    comm.finalize()


if __name__ == "__main__":
    main()
