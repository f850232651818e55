"""Geometry of the chunked multi-channel ring (SURVEY §8 header).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:655 "CCLs partition the data across multiple channels that execute in
parallel; each channel implements a communication pattern (ring ...)";
P:94 ring AllReduce = ReduceScatter then AllGather; reading C-3 (chunking).

* N elements, V = 16 / elem_bytes elements per 16-byte vector.
* N' = roundup(N, n*K*V) (logical padding, read as 0, never written).
* shard s = [s*N'/n, (s+1)*N'/n); channel slice c of each shard has
  N'/(n*K) elements; chunks j = 0..m-1 of <= chunk elements (last may be short).
* connection (r -> r+1, channel c) carries stream positions q = t*m + j,
  t = 0..2n-3: steps 0..n-2 are reduce-scatter, n-1..2n-3 all-gather.
* at step t rank r sends shard (r-1-t) mod n during RS and
  (r-(t-n+1)) mod n during AG.
* effective chunk: min(configured chunk, ceil(slice / W) rounded up to a
  vector) so that W workers per channel all get chunks (reading C-3).
"""
from __future__ import annotations

from dataclasses import dataclass


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


def effective_chunk_bytes(N: int, n: int, K: int, elem_bytes: int, chunk_bytes: int, W: int = 1) -> int:
    """Chunk size actually used (reading C-3); multiple of 16 bytes."""
    V = 16 // elem_bytes
    Np = ceil_div(max(N, 1), n * K * V) * n * K * V
    slice_bytes = Np // (n * K) * elem_bytes
    per_worker = ceil_div(ceil_div(slice_bytes, W), 16) * 16
    return max(16, min(chunk_bytes, per_worker))


@dataclass(frozen=True)
class Geometry:
    n: int
    K: int
    N: int
    elem_bytes: int
    chunk_bytes: int          # the effective chunk (multiple of 16)

    @property
    def V(self) -> int:
        return 16 // self.elem_bytes

    @property
    def Np(self) -> int:
        q = self.n * self.K * self.V
        return ceil_div(self.N, q) * q

    @property
    def shard(self) -> int:
        return self.Np // self.n

    @property
    def slice(self) -> int:
        return self.Np // (self.n * self.K)

    @property
    def chunk(self) -> int:
        return self.chunk_bytes // self.elem_bytes

    @property
    def m(self) -> int:
        return ceil_div(self.slice, self.chunk) if self.N > 0 else 0

    @property
    def steps(self) -> int:
        return 2 * self.n - 2

    def item_len(self, j: int) -> int:
        """Elements in chunk j of a channel slice."""
        return min(self.chunk, self.slice - j * self.chunk)

    def item_vectors(self, j: int) -> int:
        return self.item_len(j) // self.V

    def shard_sent(self, r: int, t: int) -> int:
        """Shard that rank r sends at step t (§8 header)."""
        n = self.n
        if t <= n - 2:
            return (r - 1 - t) % n
        return (r - (t - n + 1)) % n

    def item_base(self, r: int, t: int, c: int, j: int) -> int:
        """Global element offset of item (t, c, j) sent by rank r."""
        return self.shard_sent(r, t) * self.shard + c * self.slice + j * self.chunk

    def q(self, t: int, j: int) -> int:
        return t * self.m + j

    def tj(self, q: int) -> tuple[int, int]:
        return divmod(q, self.m)
