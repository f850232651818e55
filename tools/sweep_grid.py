"""Tuning sweep of the multi-GPU path (run on the GPU box).

usage: python tools/sweep_grid.py N "K:W:chunk:threads:bytes" ...
Each spec runs bench.py under torchrun (healthy path only) and prints one line.
"""
import json
import random
import subprocess
import sys


def run(n, K, W, chunk, threads, nbytes, steps=40):
    port = 29700 + random.randrange(200)
    cmd = ["timeout", "200", sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", str(n), "--steps",
           str(steps), "--warmup", "5", "--channels", str(K), "--ctas", str(W), "--chunk", str(chunk), "--threads",
           str(threads), "--bytes", str(nbytes), "--no-fault", "--no-e2e", "--no-nccl", "--no-cpu"]
    p = subprocess.run(cmd, capture_output=True, text=True)
    tag = f"N={n} K={K} W={W} chunk={chunk >> 10}K thr={threads} bytes={nbytes >> 20}M"
    try:
        d = json.loads(p.stdout.strip().splitlines()[-1])
        print(f"{tag} ms={d['ms_per_step']:.3f} busbw={d['busbw_per_rank']:.1f} frac={d['roofline']['frac']:.3f}",
              flush=True)
    except Exception as e:  # noqa: BLE001
        print(f"{tag} failed rc={p.returncode} {e} {p.stderr[-400:]}", flush=True)


def main():
    n = int(sys.argv[1])
    for spec in sys.argv[2:]:
        K, W, chunk, threads, nbytes = (int(x) for x in spec.split(":"))
        run(n, K, W, chunk, threads, nbytes)


if __name__ == "__main__":
    main()
