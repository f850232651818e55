"""Real multi-GPU path: torchrun launches one process per GPU (CUDA-IPC peer
mappings over NVLink 5, shared-memory OOB).  Needs >= 2 GPUs
(`gpurun --gpus 2`); skipped on a 1-GPU box."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def ngpus():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


@pytest.mark.parametrize("world", [2, 4, 8])
def test_multi_gpu_parity(world, tmp_path, cuda_required):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    from paper_2512_25059_b200 import build as B
    B.build()
    out = tmp_path / "res.json"
    port = 29600 + world + os.getpid() % 300
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mgpu_worker.py"), str(out)]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(out.read_text())
    assert res and "error" not in res[-1], res[-1]
    for case in res:
        assert case["ok"], case
        if "events_equal" in case:
            assert case["events_equal"], case
