"""Geometry of the chunked multi-channel ring (SURVEY §8 header).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:655 "CCLs partition the data across multiple channels that execute in
parallel; each channel implements a communication pattern (ring ...)";
P:94 ring AllReduce = ReduceScatter then AllGather; reading C-3 (chunking).

* N elements, V = 16 / elem_bytes elements per 16-byte vector.
* N' = roundup(N, n*K*V) (logical padding, read as 0, never written).
* shard s = [s*N'/n, (s+1)*N'/n); channel slice c of each shard has
  N'/(n*K) elements; chunks j = 0..m-1 of <= chunk elements (last may be short).
  The chunk size is an INPUT of the scenario (chunk_bytes), like n and K: the
  oracle does not derive the library's chunking policy (readings C-3 / R-8;
  tests/scenario.py states the policy a configured communicator uses).
* connection (r -> r+1, channel c) carries stream positions q = t*m + j,
  t = 0..2n-3: steps 0..n-2 are reduce-scatter, n-1..2n-3 all-gather.
* at step t rank r sends shard (r-1-t) mod n during RS and
  (r-(t-n+1)) mod n during AG.

Standalone ReduceScatter / AllGather: the two
halves of the same ring.  N is then the per-rank shard count (recvcount /
sendcount); the user buffers hold n shards at stride N; each shard is padded
to roundup(N, K*V) for the channel split (padding read as 0, never written).
  * ReduceScatter: steps t = 0..n-1; t <= n-2 are the AllReduce's RS hops,
    t = n-1 is the owner's final add, written to its own output only (a
    LOCAL item: no connection is used; its completion word is in the owner's
    own memory -- reading R-5).
  * AllGather: steps t = 0..n-2 = the AllReduce's steps n-1..2n-3 (the owner
    sends its own shard at t = 0, then the ring forwards).

Standalone Broadcast (root; "the root sends D_total while all others
receive it"): a pipelined chain root -> root+1 -> ... -> root-1 over the same
ring connections.  N is the element count; one shard (the whole padded
buffer) split into K channel slices of m chunks; steps t = 0..n-2 where rank
r is active only at its chain position t_r = (r - root) mod n (the last rank
of the chain only receives).  Reading R-8.

LL protocol (ll=True, reading R-6): the all-gather data
travels through library scratch as self-validating lines, so the receiver
unpacks the last all-gather step itself: AllReduce and AllGather get one more
step, a LOCAL item per (channel, chunk) whose input is the last step's
completion word.  (The ReduceScatter already ends in a LOCAL final add.)
"""
from __future__ import annotations

from dataclasses import dataclass


def ceil_div(a: int, b: int) -> int:
    return -(-a // b)


ALLREDUCE, REDUCE_SCATTER, ALL_GATHER, BROADCAST = "allreduce", "reduce_scatter", "all_gather", "broadcast"
# R²CCL-AllReduce's stage 2, the tailored broadcast (reading R-9): a
# chain from the degraded rank (root) once around the ring back to it
STAGE2 = "r2cc_stage2"
@dataclass(frozen=True)
class Geometry:
    n: int
    K: int
    N: int
    elem_bytes: int
    chunk_bytes: int          # the scenario's chunk (multiple of 16)
    op: str = ALLREDUCE       # N = per-shard count for REDUCE_SCATTER / ALL_GATHER
    ll: bool = False          # LL protocol: + the LOCAL unpack step (AllReduce / AllGather)
    root: int = 0             # BROADCAST only

    @property
    def V(self) -> int:
        return 16 // self.elem_bytes

    @property
    def chain(self) -> bool:
        return self.op in (BROADCAST, STAGE2)

    @property
    def Np(self) -> int:
        if self.chain:
            return self.shard
        if self.op != ALLREDUCE:
            return self.n * self.shard
        q = self.n * self.K * self.V
        return ceil_div(self.N, q) * q

    @property
    def shard(self) -> int:
        """Padded shard length (the channel split)."""
        if self.op != ALLREDUCE:
            q = self.K * self.V
            return ceil_div(self.N, q) * q
        return self.Np // self.n

    @property
    def stride(self) -> int:
        """Distance between shards in the user buffers."""
        return self.shard if self.op in (ALLREDUCE, BROADCAST, STAGE2) else self.N

    @property
    def total(self) -> int:
        """Elements of the n-shard user buffer (AllReduce / Broadcast: N)."""
        return self.N if self.op in (ALLREDUCE, BROADCAST, STAGE2) else self.n * self.N

    def shard_limit(self, s: int) -> int:
        """One past the last valid global element of shard s."""
        if self.op == ALLREDUCE:
            return min(self.N, (s + 1) * self.shard)
        if self.chain:
            return self.N
        return s * self.N + self.N

    def active(self, r: int, t: int) -> bool:
        """Does rank r send at step t?  (Broadcast: only at its chain position.)"""
        if self.op == STAGE2:
            return t == (r - self.root) % self.n
        if self.op != BROADCAST:
            return True
        return t == (r - self.root) % self.n and t <= self.n - 2

    @property
    def t0(self) -> int:
        """AllReduce step that op-step 0 corresponds to."""
        return self.n - 1 if self.op == ALL_GATHER else 0

    def local(self, t: int) -> bool:
        """True for a LOCAL item: the ReduceScatter's final add, or the LL
        protocol's unpack of the last all-gather step (no connection used)."""
        if self.op == REDUCE_SCATTER:
            return t == self.n - 1
        if self.chain:
            return False
        return self.ll and t == self.steps - 1

    @property
    def slice(self) -> int:
        return self.shard // self.K

    @property
    def chunk(self) -> int:
        return self.chunk_bytes // self.elem_bytes

    @property
    def m(self) -> int:
        return ceil_div(self.slice, self.chunk) if self.N > 0 else 0

    @property
    def steps(self) -> int:
        base = {ALLREDUCE: 2 * self.n - 2, REDUCE_SCATTER: self.n, ALL_GATHER: self.n - 1,
                BROADCAST: self.n - 1, STAGE2: self.n}[self.op]
        return base + (1 if self.ll and self.op != REDUCE_SCATTER else 0)

    def item_len(self, j: int) -> int:
        """Elements in chunk j of a channel slice."""
        return min(self.chunk, self.slice - j * self.chunk)

    def item_vectors(self, j: int) -> int:
        return self.item_len(j) // self.V

    def shard_sent(self, r: int, t: int) -> int:
        """Shard that rank r sends at (op-)step t (§8 header)."""
        if self.chain:
            return 0
        n = self.n
        ta = t + self.t0
        if ta <= n - 2:
            return (r - 1 - ta) % n
        return (r - (ta - n + 1)) % n

    def item_base(self, r: int, t: int, c: int, j: int) -> int:
        """Global element offset (in the n-shard buffer) of item (t, c, j) of rank r."""
        return self.shard_sent(r, t) * self.stride + c * self.slice + j * self.chunk

    def q(self, t: int, j: int) -> int:
        return t * self.m + j

    def tj(self, q: int) -> tuple[int, int]:
        return divmod(q, self.m)
