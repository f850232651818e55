"""Scenario inputs shared by the tests, bench.py's cpu_baseline leg and
smoke(): the chunk size a launch configuration uses.

TEST INFRASTRUCTURE.  This is NOT part of the oracle: the oracle's Layer 2
(oracle/geometry.py, oracle/protocol.py) takes the chunk size as an input of
the scenario it simulates, like n, K and the fault list.  The rule below is
the library's documented chunking policy (readings C-3 and R-8,
include/r2ccl.h r2_geometry_op), restated here so that a test can name the
scenario a configured communicator runs; tests/test_abi.py checks that the
library's r2_geometry_op uses exactly this chunk.

* C-3: the configured chunk, capped at ceil(slice / W) rounded up to a 16-byte
  vector, so that every one of the W lanes of a channel gets a chunk per step.
* R-8: Broadcast chunks are further capped at 128 KiB (a chain's pipeline
  fill is n-2 chunk hops).
"""
from __future__ import annotations

from oracle.geometry import ALLREDUCE, BROADCAST, ceil_div

BCAST_CHUNK_CAP = 128 * 1024


def effective_chunk_bytes(N: int, n: int, K: int, elem_bytes: int, chunk_bytes: int, W: int = 1,
                          op: str = ALLREDUCE) -> int:
    """Chunk size (bytes, multiple of 16) a launch with these parameters uses."""
    V = 16 // elem_bytes
    if op == ALLREDUCE:
        Np = ceil_div(max(N, 1), n * K * V) * n * K * V
        slice_bytes = Np // (n * K) * elem_bytes
    else:
        slice_bytes = ceil_div(max(N, 1), K * V) * V * elem_bytes
    per_worker = ceil_div(ceil_div(slice_bytes, W), 16) * 16
    if op == BROADCAST:
        chunk_bytes = min(chunk_bytes, BCAST_CHUNK_CAP)
    return max(16, min(chunk_bytes, per_worker))
