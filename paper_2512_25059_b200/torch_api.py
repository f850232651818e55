"""torch glue: tensors -> (pointer, count, dtype, stream) for the C ABI, and
communicator bootstrap from torch.distributed's environment / c10d store
(the process-group bootstrap of P:657 carries only the OOB segment name).
PyTorch provides device memory, streams and process groups -- nothing else.
"""
from __future__ import annotations

import itertools
import os

import torch

from . import r2ccl as R

TORCH_DTYPES = {torch.int32: R.INT32, torch.float32: R.FLOAT32, torch.bfloat16: R.BFLOAT16}
_counter = itertools.count()


def r2_dtype(t: torch.Tensor) -> int:
    try:
        return TORCH_DTYPES[t.dtype]
    except KeyError as e:
        raise TypeError(f"r2ccl supports int32/float32/bfloat16, not {t.dtype}") from e


def comm_from_env(cfg: R.Config | None = None, store=None) -> R.Comm:
    """One communicator per process, ranks from RANK / WORLD_SIZE / LOCAL_RANK
    (torchrun).  world > 1 needs an initialised default process group (its
    store carries the OOB name) or an explicit c10d store."""
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    torch.cuda.set_device(local)
    if world == 1:
        return R.Comm(0, 1, local, None, cfg)
    if store is None:
        store = torch.distributed.distributed_c10d._get_default_store()
    key = f"r2ccl/oob/{next(_counter)}"
    if rank == 0:
        name = R.unique_name()
        store.set(key, name)
    else:
        name = store.get(key).decode()
    oob = R.oob_shm_open(name, rank, world)
    return R.Comm(rank, world, local, oob, cfg)


def register(comm: R.Comm, t: torch.Tensor) -> int:
    """Collective: register t's storage with every peer (r2_register_multi)."""
    return comm.register_multi(t.data_ptr(), t.numel() * t.element_size())


def _count(comm: R.Comm, t: torch.Tensor, count: int | None) -> int:
    if not comm.sim:
        if count is None:
            return t.numel()
        if not 0 <= count <= t.numel():
            raise ValueError(f"count {count} outside the tensor's {t.numel()} elements")
        return count
    # sim mode: [k, row] with 16-byte aligned rows; count <= row elements
    if t.dim() != 2 or t.shape[0] != comm.n:
        raise ValueError(f"sim mode expects a [{comm.n}, row] tensor")
    row, E = t.shape[1], t.element_size()
    count = row if count is None else count
    if (row * E) % 16 or -(-count * E // 16) * 16 != row * E:
        raise ValueError("sim-mode rows must be roundup(count * elem, 16) bytes long")
    return count


def allreduce(comm: R.Comm, send: torch.Tensor, recv: torch.Tensor | None = None, stream=None,
              count: int | None = None) -> torch.Tensor:
    """Sum-allreduce send -> recv (in place when recv is None / send).

    Sim mode (one process, k simulated ranks): send/recv are [k, row]
    tensors; rank l's buffer is row l (rows 16-byte aligned)."""
    if recv is None:
        recv = send
    if not (send.is_cuda and recv.is_cuda):
        raise ValueError("device tensors required (use allreduce_host for host buffers)")
    if not (send.is_contiguous() and recv.is_contiguous()):
        raise ValueError("contiguous tensors required")
    if send.dtype != recv.dtype or send.numel() != recv.numel():
        raise ValueError("send/recv must match in dtype and size")
    n = _count(comm, send, count)
    s = stream if stream is not None else torch.cuda.current_stream()
    comm.allreduce(send.data_ptr(), recv.data_ptr(), n, r2_dtype(send), s.cuda_stream)
    return recv


def _rows_ok(comm: R.Comm, t: torch.Tensor, count: int) -> None:
    """Sim mode: a [k, row] tensor whose rows are roundup(count * elem, 16) bytes."""
    if t.dim() != 2 or t.shape[0] != comm.n:
        raise ValueError(f"sim mode expects a [{comm.n}, row] tensor")
    if t.shape[1] * t.element_size() != -(-count * t.element_size() // 16) * 16:
        raise ValueError("sim-mode rows must be roundup(count * elem, 16) bytes long")


def _check_pair(send: torch.Tensor, recv: torch.Tensor) -> None:
    if not (send.is_cuda and recv.is_cuda):
        raise ValueError("device tensors required")
    if not (send.is_contiguous() and recv.is_contiguous()):
        raise ValueError("contiguous tensors required")
    if send.dtype != recv.dtype:
        raise ValueError("send/recv must match in dtype")


def reduce_scatter(comm: R.Comm, send: torch.Tensor, recv: torch.Tensor, stream=None,
                   recvcount: int | None = None) -> torch.Tensor:
    """Sum-ReduceScatter (r2_reduce_scatter): send holds n shards of recvcount
    elements, recv receives this rank's reduced shard.  In-place: recv is the
    own shard of send (a view).  Sim mode: send [k, rowS], recv [k, rowR]."""
    _check_pair(send, recv)
    n = comm.n
    if comm.sim:
        recvcount = recvcount if recvcount is not None else recv.shape[1]
        _rows_ok(comm, send, n * recvcount)
        _rows_ok(comm, recv, recvcount)
    else:
        recvcount = recv.numel() if recvcount is None else recvcount
        if send.numel() < n * recvcount or recv.numel() < recvcount:
            raise ValueError("send must hold n * recvcount and recv recvcount elements")
    s = stream if stream is not None else torch.cuda.current_stream()
    comm.reduce_scatter(send.data_ptr(), recv.data_ptr(), recvcount, r2_dtype(send), s.cuda_stream)
    return recv


def all_gather(comm: R.Comm, send: torch.Tensor, recv: torch.Tensor, stream=None,
               sendcount: int | None = None) -> torch.Tensor:
    """AllGather (r2_all_gather): every rank's recv receives the n inputs in
    rank order; recv must be registered.  In-place: send is the own shard of
    recv (a view).  Sim mode: send [k, rowS], recv [k, rowR]."""
    _check_pair(send, recv)
    n = comm.n
    if comm.sim:
        sendcount = sendcount if sendcount is not None else send.shape[1]
        _rows_ok(comm, send, sendcount)
        _rows_ok(comm, recv, n * sendcount)
    else:
        sendcount = send.numel() if sendcount is None else sendcount
        if recv.numel() < n * sendcount:
            raise ValueError("recv must hold n * sendcount elements")
    s = stream if stream is not None else torch.cuda.current_stream()
    comm.all_gather(send.data_ptr(), recv.data_ptr(), sendcount, r2_dtype(send), s.cuda_stream)
    return recv


def broadcast(comm: R.Comm, send: torch.Tensor | None, recv: torch.Tensor, root: int, stream=None,
              count: int | None = None) -> torch.Tensor:
    """Broadcast (r2_broadcast): the root's send arrives in every rank's recv
    (registered).  send is only read on the root (None elsewhere; None on the
    root means in place: recv).  Sim mode: send / recv [k, row] tensors."""
    if send is None:
        send = recv
    _check_pair(send, recv)
    if comm.sim:
        count = count if count is not None else recv.shape[1]
        _rows_ok(comm, send, count)
        _rows_ok(comm, recv, count)
    else:
        count = recv.numel() if count is None else count
        if not 0 <= count <= recv.numel() or (send is not recv and count > send.numel()):
            raise ValueError(f"count {count} exceeds the send / recv tensors")
    s = stream if stream is not None else torch.cuda.current_stream()
    comm.broadcast(send.data_ptr(), recv.data_ptr(), count, r2_dtype(recv), root, s.cuda_stream)
    return recv


def allreduce_host(comm: R.Comm, send: torch.Tensor, recv: torch.Tensor, stream=None,
                   count: int | None = None) -> torch.Tensor:
    """Host (ideally pinned) tensors: H2D, allreduce, D2H on `stream`."""
    n = _count(comm, send, count)
    s = stream if stream is not None else torch.cuda.current_stream()
    comm.allreduce_host(send.data_ptr(), recv.data_ptr(), n, r2_dtype(send), s.cuda_stream)
    return recv
