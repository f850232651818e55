"""Full-size parity in the launch configuration bench.py times (N = 1: 8
simulated ranks x 256 MiB bf16, K = 8 channels x W = 2 CTAs, 512 KiB chunks;
BASELINE configs[1]/[2]): 4096 sampled outputs per rank against the oracle's
ring fold computed element by element, healthy and with the config-3 LINK
fault (rank 3, channel 5, step 3, chunk 4, 256 KiB into the chunk); the
faulted result must be bit-identical to the healthy one everywhere.

Inputs: torch's seeded device RNG, N(0,1) rounded to bf16 (the bench's
inputs); the sampled inputs are read back for the oracle."""
import numpy as np
import pytest
import torch

from oracle import semantic as OS
from tests.gpu_util import sim_comm
from paper_2512_25059_b200 import build as B
from paper_2512_25059_b200 import r2ccl as R
from paper_2512_25059_b200 import torch_api as T

pytestmark = pytest.mark.gpu

K_RANKS, S = 8, 256 << 20
COUNT = S // 2


@pytest.fixture(scope="module", autouse=True)
def setup(cuda_required):
    B.build()
    torch.cuda.set_device(0)


def sampled_check(send, recv, shard, n_sample=4096, seed=5):
    rng = np.random.default_rng(seed)
    idx = np.unique(rng.integers(0, COUNT, size=n_sample))
    it = torch.from_numpy(idx).cuda()
    xs = send[:, it].view(torch.int16).cpu().numpy().view(np.uint16)
    got = recv[:, it].view(torch.int16).cpu().numpy().view(np.uint16)
    bad = 0
    for col, i in enumerate(idx):
        want = OS.ring_fold([xs[r, col:col + 1] for r in range(K_RANKS)], int(i) // shard, "bfloat16")[0]
        bad += int(np.any(got[:, col] != want))
    return len(idx), bad


@pytest.mark.parametrize("protocol", ["AUTO"])
def test_bench_configuration_sampled_parity_and_fault(protocol):
    send = torch.empty((K_RANKS, COUNT), dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(1234)
    send.copy_(torch.randn(send.shape, generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16))
    recv = torch.empty_like(send)
    comm = sim_comm(K_RANKS, 8, 2, 512 * 1024, max_bytes=S, protocol=protocol)
    geo = R.geometry(COUNT, R.BFLOAT16, K_RANKS, 8, 2, 512 * 1024)
    T.allreduce(comm, send, recv)
    assert comm.sync() == R.SUCCESS
    n, bad = sampled_check(send, recv, geo.shard)
    assert n > 4000 and bad == 0
    healthy = recv.clone()
    # config 3 at N = 1: LINK fault mid-collective, recovered inside the call
    seq = comm.status()["seq"] + 1
    comm.inject_fault(at_seq=seq, kind="LINK", src_rank=3, channel=5, step=3, chunk=4, byte_offset=256 * 1024,
                      poison=1)
    recv.view(torch.uint8).fill_(0xFF)
    T.allreduce(comm, send, recv)
    assert comm.sync() == R.SUCCESS
    assert torch.equal(recv, healthy)
    ev = comm.events()
    assert len(ev) == 1 and ev[0]["verdict"] == "LINK" and ev[0]["resume"] == 3 * geo.m + 4
    comm.finalize()


def test_ll128_bucket_size_sampled_parity_and_fault():
    """The LL128 protocol at BASELINE configs[4]'s bucket size (25,000,000 B
    bf16 per rank, 8 simulated ranks, K = 8 x W = 2): 4096 sampled outputs per
    rank against the oracle fold, then a LINK fault mid-collective (rank 3,
    channel 5, step 3, chunk 1, 4 KiB into it) recovered bit-identical."""
    count = 12_500_000
    send = torch.empty((K_RANKS, count), dtype=torch.bfloat16, device="cuda")
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    send.copy_(torch.randn(send.shape, generator=g, device="cuda", dtype=torch.float32).to(torch.bfloat16))
    recv = torch.empty_like(send)
    comm = sim_comm(K_RANKS, 8, 2, 512 * 1024, max_bytes=2 * count, protocol="LL128")
    geo = R.geometry(count, R.BFLOAT16, K_RANKS, 8, 2, 512 * 1024)
    T.allreduce(comm, send, recv)
    assert comm.sync() == R.SUCCESS
    assert comm.status()["last_protocol"] == "LL128"
    rng = np.random.default_rng(9)
    idx = np.unique(rng.integers(0, count, size=4096))
    it = torch.from_numpy(idx).cuda()
    xs = send[:, it].view(torch.int16).cpu().numpy().view(np.uint16)
    got = recv[:, it].view(torch.int16).cpu().numpy().view(np.uint16)
    for col, i in enumerate(idx):
        want = OS.ring_fold([xs[r, col:col + 1] for r in range(K_RANKS)], int(i) // geo.shard, "bfloat16")[0]
        assert np.all(got[:, col] == want), int(i)
    healthy = recv.clone()
    seq = comm.status()["seq"] + 1
    comm.inject_fault(at_seq=seq, kind="LINK", src_rank=3, channel=5, step=3, chunk=min(1, geo.m - 1),
                      byte_offset=4096, poison=1)
    recv.view(torch.uint8).fill_(0xFF)
    T.allreduce(comm, send, recv)
    assert comm.sync() == R.SUCCESS
    assert torch.equal(recv, healthy)
    ev = comm.events()
    assert len(ev) == 1 and ev[0]["verdict"] == "LINK"
    comm.finalize()
