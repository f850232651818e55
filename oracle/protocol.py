"""Layer 2 of the oracle: the fault-tolerant chunked multi-channel ring
allreduce, simulated sequentially over n ranks and K channels.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Follows, in the paper's order:
  * the ring schedule: ReduceScatter then AllGather (Fig. 3),
    over K channels each carrying its slice of every shard;
  * a per-chunk completion flag in the receiver's memory (reading C-4) --
    the analogue of an RDMA work completion;
  * a fault that kills a channel's transport mid-chunk ("Failures may
    occur mid-chunk transfer"); the faulted chunk's first b bytes reach the
    peer, no completion is written (reading C-6);
  * bilateral awareness: the detecting sender raises a notification;
  * three-point triangulation with emulated zero-byte probes (P:16-19,
    oracle/triangulation.py) whose verdict updates every rank's health view;
  * DMA-buffer rollback: the sender rewinds to the first chunk without a
    completion, the receiver resets to the last confirmed chunk (P:36,
    oracle/ledger.py); exactly the chunks without completion are resent (C-7);
  * migration onto the ordered failover chain (HOT_REPAIR) or
    R²CCL-Balance: every residual chunk split over all healthy channels in
    proportion to their weight (oracle/balance.py; reading C-15/C-16);
  * successive failover: a backup that fails mid-retransmit triggers a new
    rollback (chunks still without completion) and the next chain entry
    (P:36);
  * chain exhausted -> NoBackup: the collective aborts.

Interleaving: every rank/channel pair is one sequential worker that executes
its tasks in global step order (own + adopted, SURVEY §7 hard part 3).  A
seeded RNG picks, at every step, one of: a worker whose next task's input has
arrived; a worker whose connection died physically (it notices at a task
boundary); or the host monitor handling a pending notification.  Any
dependency-respecting interleaving must yield identical buffers.

In-place calls (send == recv): the owner's final sum for its own shard is
staged and copied to recv at the end, so that a retransmitted final-add chunk
never reads an already-overwritten input (reading C-7).

Standalone ReduceScatter / AllGather (SURVEY §8(f) f1, P:78, P:94,
P:353/572 "R²CCL-Balance on AllGather, ReduceScatter"): the same workers,
flags, faults, rollback and re-placement over the op's steps
(oracle/geometry.py).  The ReduceScatter's final add is a LOCAL item: it uses
no connection, so no fault fires on it, its completion word is kept by the
owner itself, and a stopped worker's unfinished local items are re-placed
with the rest of its residual (reading R-5).  In-place ReduceScatter
(recv = own shard of send) needs no staging: the final add is the only
writer of the own shard and a local item is never torn by a fault.

Broadcast (f1, reading R-8): a pipelined chain from the root along the ring;
worker (r, c) holds only the items of r's chain position t_r, reads the
root's input (t_r = 0) or its own received buffer, and writes the next rank's
buffer.  Positions of other steps count as complete in r's ledger.

R²CCL-AllReduce stage 2 (f2, "a broadcast initiated from the failure
server node, a pipelined ring broadcast across the healthy servers, and the
final delivery ... back to the failure node"; reading R-9): a chain of n
steps from the degraded rank (root) around the ring back to it.  recv_init
holds every rank's stage-1 result (the healthy ranks' partial AllReduce).
Step 0: the root sends its input into the next rank's tailor buffer; step 1:
that rank adds it to its partial result (acc (+) x, acc = the partial
result), keeps the sum and sends it on; steps 2..n-1 forward the sum, the last
one into the root's buffer.  (Stage 1's two rings are plain ring AllReduces
over disjoint channel sets and are simulated as such.)
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import balance as _bal
from . import ledger as _led
from . import triangulation as _tri
from .geometry import ALL_GATHER, ALLREDUCE, BROADCAST, REDUCE_SCATTER, STAGE2, Geometry
from .semantic import hop_add, np_dtype

HOT_REPAIR = "HOT_REPAIR"
BALANCE = "BALANCE"


@dataclass
class Fault:
    """An injected channel fault.

    kind    LINK   : the ring link (rank -> rank+1) on `channel` dies;
            LOCAL  : the sender's endpoint (rank, channel) dies;
            REMOTE : the receiver's endpoint (rank+1, channel) dies.
    It fires when the worker (rank, channel) starts the part of item
    (t, origin, j) it carries: the first `b` bytes of that part reach the peer
    (rounded down to a 16-byte vector), then the transport is dead.
    origin = None means the channel's own item (origin == channel).
    """
    kind: str
    rank: int
    channel: int
    t: int
    j: int
    b: int = 0
    origin: int | None = None

    @property
    def org(self) -> int:
        return self.channel if self.origin is None else self.origin


@dataclass(order=True)
class Task:
    t: int
    origin: int
    j: int
    lo: int            # vector range inside the item
    hi: int
    parts: int = field(compare=False, default=1)
    epoch: int = field(compare=False, default=0)


@dataclass
class SimResult:
    y: list                      # per rank result buffer (AllReduce N, ReduceScatter N, AllGather n*N elements)
    events: list                 # failover records (one per re-planned origin)
    detections: list             # triangulation rounds
    bytes_sent: np.ndarray       # [rank, channel] bytes pushed to the peer
    error: str | None
    health: dict
    retransmitted_items: int
    retransmitted_bytes: int
    fired: list
    hbm_bytes: np.ndarray | None = None   # [rank] bytes read from / written into rank's own memory


class Simulator:
    def __init__(self, xs, geom: Geometry, dtype: str, faults=(), strategy=BALANCE,
                 weights=None, health=None, seed=0, inplace=False, poison=True, recv_init=None):
        self.g, self.dtype = geom, dtype
        self.n, self.K, self.m, self.V = geom.n, geom.K, geom.m, geom.V
        self.N = geom.N
        self.op = geom.op
        n, K = self.n, self.K
        self.strategy = strategy
        self.weights = {c: 1 for c in range(K)} if weights is None else dict(enumerate(weights))
        self.rng = np.random.default_rng(seed)
        self.inplace = inplace
        dt = np_dtype(dtype)
        self.dt = dt
        # buffers: x[r] is the op's input, recv[r] its output (in-place: views
        # of one buffer, NCCL's convention: RS recv = own shard of send, AG
        # send = own shard of recv)
        self.stage = None
        if self.op == ALLREDUCE:
            if inplace:
                self.recv = [np.array(x, dtype=dt, copy=True) for x in xs]
                self.x = self.recv
                self.stage = [np.zeros(geom.shard, dtype=dt) for _ in range(n)]
            else:
                self.x = [np.asarray(x, dtype=dt) for x in xs]
                self.recv = [self._poisoned(self.N, poison) for _ in range(n)]
        elif self.op == REDUCE_SCATTER:
            self.x = [np.array(x, dtype=dt, copy=True) for x in xs]         # n*N elements
            if inplace:
                self.recv = [self.x[r][r * self.N:(r + 1) * self.N] for r in range(n)]
            else:
                self.recv = [self._poisoned(self.N, poison) for _ in range(n)]
        elif self.op == BROADCAST:
            self.x = [np.asarray(x, dtype=dt) for x in xs]
            self.recv = [self._poisoned(self.N, poison) for _ in range(n)]
            if inplace:
                self.recv[geom.root] = np.array(xs[geom.root], dtype=dt, copy=True)
        elif self.op == STAGE2:
            self.x = [np.asarray(x, dtype=dt) for x in xs]
            self.recv = [np.array(a, dtype=dt, copy=True) for a in recv_init]
            self.tailor = [self._poisoned(geom.shard, poison) for _ in range(n)]
        elif self.op == ALL_GATHER:
            self.recv = [self._poisoned(n * self.N, poison) for _ in range(n)]
            if inplace:
                for r in range(n):
                    self.recv[r][r * self.N:(r + 1) * self.N] = xs[r]
                self.x = [self.recv[r][r * self.N:(r + 1) * self.N] for r in range(n)]
            else:
                self.x = [np.asarray(x, dtype=dt) for x in xs]              # N elements: the own shard
        else:
            raise ValueError(self.op)
        self.scratch = [[self._poisoned(geom.shard, poison) for _ in range(max(n - 1, 0))] for _ in range(n)]
        # completion flags live in the receiver's memory: (recv_rank, t, c, j)
        self.flags: set = set()
        self.counters: dict = {}
        # health: host knowledge (ep_ok, link_ok) and emulated physics
        h = health or {}
        self.ep_dead = [[False] * K for _ in range(n)]
        self.link_dead = [[False] * K for _ in range(n)]
        for (r, c) in h.get("dead_endpoints", ()):
            self.ep_dead[r][c] = True
        for (r, c) in h.get("dead_links", ()):
            self.link_dead[r][c] = True
        self.known_ep_dead = [row[:] for row in self.ep_dead]
        self.known_link_dead = [row[:] for row in self.link_dead]
        self.faults = [f for f in faults]
        self.fired: list = []
        self.bytes_sent = np.zeros((n, K), dtype=np.int64)
        # bytes each rank's memory serves (reads) or absorbs (writes, local or
        # arriving from the upstream peer): the executed schedule's HBM traffic
        self.hbm = np.zeros(n, dtype=np.int64)
        self.events: list = []
        self.detections: list = []
        self.pending: list = []            # host notifications (rank, channel)
        self.error = None
        self.epoch = 0
        self.retx_items = 0
        self.retx_bytes = 0
        # workers
        self.queue = {}                    # (r, c) -> sorted list of Task
        self.state = {}                    # (r, c) -> 'run' | 'stopped'
        self.replanned = set()
        for r in range(n):
            for c in range(K):
                if self.conn_ok(r, c):
                    self.queue[(r, c)] = [Task(t, c, j, 0, geom.item_vectors(j))
                                          for t in range(geom.steps) for j in range(self.m) if geom.active(r, t)]
                    self.state[(r, c)] = "run"
        # static plan (plan-time Balance / HotRepair for already-dead connections)
        for r in range(n):
            for c in range(K):
                if not self.conn_ok(r, c) and self.error is None:
                    items = [(t, j) for t in range(geom.steps) for j in range(self.m) if geom.active(r, t)]
                    self._assign(r, c, items, record=None)

    # ------------------------------------------------------------ helpers
    def _poisoned(self, length, poison):
        a = np.zeros(length, dtype=self.dt)
        if poison:
            a.view(np.uint8)[:] = 0xFF
        return a

    def conn_ok(self, r, c) -> bool:
        """Host view: connection (r -> r+1, c) usable."""
        r1 = (r + 1) % self.n
        return not (self.known_ep_dead[r][c] or self.known_ep_dead[r1][c] or self.known_link_dead[r][c])

    def phys_dead(self, r, c) -> bool:
        r1 = (r + 1) % self.n
        return self.ep_dead[r][c] or self.ep_dead[r1][c] or self.link_dead[r][c]

    def xread(self, r, lo, hi, lim, base=0):
        """Input elements [lo, hi) (global n-shard index, valid below lim; the
        AllGather's input holds only the own shard: base = its global start)."""
        out = np.zeros(hi - lo, dtype=self.dt)
        top = min(hi, lim)
        if top > lo:
            out[: top - lo] = self.x[r][lo - base:top - base]
        return out

    def rread(self, r, lo, hi, lim):
        out = np.zeros(hi - lo, dtype=self.dt)
        top = min(hi, lim)
        if top > lo:
            out[: top - lo] = self.recv[r][lo:top]
        return out

    def rwrite(self, r, lo, vals, lim, base=0):
        top = min(lo + len(vals), lim)
        if top > lo:
            self.recv[r][lo - base:top - base] = vals[: top - lo]

    def holder(self, r, t) -> int:
        """Rank whose memory keeps the completion word of r's item at step t."""
        return r if self.g.local(t) else (r + 1) % self.n

    def ready(self, r, task: Task) -> bool:
        return task.t == 0 or (r, task.t - 1, task.origin, task.j) in self.flags

    # ------------------------------------------------------------ data path
    def _move(self, r, task: Task, lo, hi):
        """Execute vectors [lo, hi) of item (task.t, task.origin, task.j) sent by r."""
        g, n, V = self.g, self.n, self.V
        t = task.t
        ta = t + g.t0                                     # the AllReduce step it corresponds to
        s = g.shard_sent(r, t)
        e0 = g.item_base(r, t, task.origin, task.j) + lo * V
        e1 = e0 + (hi - lo) * V
        o0, o1 = e0 - s * g.stride, e1 - s * g.stride    # offsets inside the shard
        lim = g.shard_limit(s)
        r1 = (r + 1) % n
        nb = (e1 - e0) * g.elem_bytes                     # bytes of one operand of this part
        if g.local(t) and self.op != REDUCE_SCATTER:      # LL unpack: the data already landed here
            return
        if self.op == STAGE2:                             # tailored broadcast (reading R-9)
            if t == 0:                                    # the degraded rank's input -> next rank's tailor buffer
                self.tailor[r1][o0:o1] = self.xread(r, e0, e1, lim)
                self.hbm[r] += nb
                self.hbm[r1] += nb
            elif t == 1:                                  # partial result (+) f's contribution
                val = hop_add(self.rread(r, e0, e1, lim), self.tailor[r][o0:o1], self.dtype)
                self.rwrite(r, e0, val, lim)
                self.rwrite(r1, e0, val, lim)
            else:
                self.rwrite(r1, e0, self.rread(r, e0, e1, lim), lim)
            return
        if self.op == BROADCAST:                          # chain: root's input, else what arrived here
            val = self.xread(r, e0, e1, lim) if t == 0 else self.rread(r, e0, e1, lim)
            if t == 0 and not self.inplace:
                self.rwrite(r, e0, val, lim)
            self.rwrite(r1, e0, val, lim)
            return
        if ta <= n - 2:                                   # reduce-scatter hop
            val = self.xread(r, e0, e1, lim)
            self.hbm[r] += nb
            if t > 0:
                val = hop_add(self.scratch[r][t - 1][o0:o1], val, self.dtype)
                self.hbm[r] += nb
            self.scratch[r1][t][o0:o1] = val
            self.hbm[r1] += nb
        elif ta == n - 1 and self.op == ALLREDUCE:        # final add + first all-gather send
            val = hop_add(self.scratch[r][n - 2][o0:o1], self.xread(r, e0, e1, lim), self.dtype)
            self.hbm[r] += 3 * nb                         # scratch + x read, own result written
            if self.inplace:
                self.stage[r][o0:o1] = val
            else:
                self.rwrite(r, e0, val, lim)
            self.rwrite(r1, e0, val, lim)
            self.hbm[r1] += nb
        elif ta == n - 1 and self.op == REDUCE_SCATTER:   # final add into the own output (LOCAL)
            val = hop_add(self.scratch[r][n - 2][o0:o1], self.xread(r, e0, e1, lim), self.dtype)
            self.rwrite(r, e0, val, lim, base=s * g.stride)
        elif ta == n - 1:                                 # all-gather: the owner sends its shard
            val = self.xread(r, e0, e1, lim, base=s * g.stride)
            if not self.inplace:
                self.rwrite(r, e0, val, lim)
            self.rwrite(r1, e0, val, lim)
        else:                                             # all-gather forward
            self.rwrite(r1, e0, self.rread(r, e0, e1, lim), lim)
            self.hbm[r] += nb
            self.hbm[r1] += nb

    def _run_task(self, w, task: Task):
        r, c = w
        g = self.g
        local = g.local(task.t)
        # armed fault? (a LOCAL item uses no connection: nothing to fire on)
        for f in ([] if local else self.faults):
            if (f.rank, f.channel, f.org, f.t, f.j) == (r, c, task.origin, task.t, task.j) and f not in self.fired:
                bvec = min(max(f.b, 0) // 16, task.hi - task.lo)
                if bvec > 0:
                    self._move(r, task, task.lo, task.lo + bvec)
                    self.bytes_sent[r, c] += bvec * 16
                self.fired.append(f)
                if f.kind == "LINK":
                    self.link_dead[r][c] = True
                elif f.kind == "LOCAL":
                    self.ep_dead[r][c] = True
                elif f.kind == "REMOTE":
                    self.ep_dead[(r + 1) % self.n][c] = True
                else:
                    raise ValueError(f.kind)
                self._stop(w)
                return
        self._move(r, task, task.lo, task.hi)
        if not local:
            self.bytes_sent[r, c] += (task.hi - task.lo) * 16
        self.queue[w].pop(0)
        key = (r, task.t, task.origin, task.j)
        if task.parts == 1:
            done = True
        else:
            ep, cnt = self.counters.get(key, (task.epoch, 0))
            if ep != task.epoch:
                cnt = 0
            cnt += 1
            self.counters[key] = (task.epoch, cnt)
            done = cnt == task.parts
        if done:
            self.flags.add((self.holder(r, task.t), task.t, task.origin, task.j))

    def _stop(self, w):
        self.state[w] = "stopped"
        self.pending.append(w)

    # ------------------------------------------------------------ host side
    def _completed(self, r, origin):
        g = self.g
        return [(not g.active(r, t)) or (self.holder(r, t), t, origin, j) in self.flags
                for t in range(g.steps) for j in range(self.m)]

    def _assign(self, r, origin, items, record):
        """Place residual items of (r -> r+1, origin) on healthy channels."""
        g = self.g
        healthy = {c for c in range(self.K) if self.conn_ok(r, c) and self.state.get((r, c)) == "run"}
        self.epoch += 1
        ep = self.epoch
        try:
            if self.strategy == HOT_REPAIR:
                a, pos = _led.migrate(_led.failover_chain(origin, self.K), healthy)
                for (t, j) in items:
                    self.queue[(r, a)].append(Task(t, origin, j, 0, g.item_vectors(j), 1, ep))
                if record is not None:
                    record.update(assignee=a, chain_pos=pos)
            else:
                if not healthy:
                    raise _led.NoBackup("no healthy channel")
                w = {c: self.weights[c] for c in healthy}
                for (t, j) in items:
                    parts = _bal.part_ranges(g.item_vectors(j), w)
                    for (c, lo, hi) in parts:
                        self.queue[(r, c)].append(Task(t, origin, j, lo, hi, len(parts), ep))
                if record is not None:
                    record.update(shares=_bal.redistribute(g.item_vectors(0), w))
        except (_led.NoBackup, _bal.AllFailed):
            self.error = "NO_BACKUP"
            return
        for c in range(self.K):
            if (r, c) in self.queue:
                self.queue[(r, c)].sort()
        if record is not None:          # static (plan-time) placement is not a retransmission
            self.retx_items += len(items)
            self.retx_bytes += sum(g.item_vectors(j) * 16 for (_, j) in items)

    def _host_step(self):
        """Handle one notification: triangulate, update health, roll back,
        migrate / rebalance."""
        r, c = self.pending.pop(0)
        n = self.n
        rnd = _tri.run_round(r, (r + 1) % n, c, n, self.ep_dead, self.link_dead)
        rnd["detected_by"] = (r, c)
        self.detections.append(rnd)
        eps, link = _tri.dead_after_verdict(rnd["verdict"], r, (r + 1) % n)
        for e in eps:
            self.known_ep_dead[e][c] = True
        if link:
            self.known_link_dead[r][c] = True
        # force-stop running workers whose connection is now known dead
        for (rr, cc), st in list(self.state.items()):
            if st == "run" and not self.conn_ok(rr, cc):
                self.state[(rr, cc)] = "stopped"
        # roll back + re-plan every stopped, known-dead worker's origins
        for (rr, cc), st in sorted(self.state.items()):
            if st != "stopped" or (rr, cc) in self.replanned or self.conn_ok(rr, cc):
                continue
            self.replanned.add((rr, cc))
            origins = sorted({cc} | {tk.origin for tk in self.queue[(rr, cc)]})
            self.queue[(rr, cc)] = []
            for o in origins:
                # freeze: withdraw every pending part of origin o on rank rr
                for c2 in range(self.K):
                    if (rr, c2) in self.queue:
                        self.queue[(rr, c2)] = [tk for tk in self.queue[(rr, c2)] if tk.origin != o]
                completed = self._completed(rr, o)
                resume, floor = _led.rollback(completed)
                res = _led.residual(completed)
                rec = {"rank": rr, "origin": o, "stopped_channel": cc, "verdict": rnd["verdict"],
                       "a": rnd["a"], "b": rnd["b"], "aux": rnd["aux"], "outcomes": rnd["outcomes"],
                       "resume": resume, "floor": floor, "retransmit": len(res),
                       "strategy": self.strategy}
                self.events.append(rec)
                self._assign(rr, o, [self.g.tj(q) for q in res], rec)
                if self.error:
                    return

    # ------------------------------------------------------------ driver
    def run(self, max_iter=10_000_000) -> SimResult:
        it = 0
        while self.error is None:
            it += 1
            if it > max_iter:
                raise RuntimeError("simulation did not terminate")
            cands = []
            for w, st in self.state.items():
                if st != "run":
                    continue
                if self.phys_dead(*w) and self.queue[w]:
                    cands.append(("stop", w))
                elif self.queue[w] and self.ready(w[0], self.queue[w][0]):
                    cands.append(("work", w))
            if self.pending:
                cands.append(("host", None))
            if not cands:
                break
            kind, w = cands[int(self.rng.integers(len(cands)))]
            if kind == "work":
                self._run_task(w, self.queue[w][0])
            elif kind == "stop":
                self._stop(w)
            else:
                self._host_step()
        if self.error is None:
            missing = [(r, t, c, j) for r in range(self.n) for t in range(self.g.steps)
                       for c in range(self.K) for j in range(self.m)
                       if self.g.active(r, t) and (self.holder(r, t), t, c, j) not in self.flags]
            if missing:
                raise RuntimeError(f"deadlock: {len(missing)} items undelivered, e.g. {missing[:4]}")
            if self.stage is not None:
                g = self.g
                for r in range(self.n):
                    lo = r * g.shard
                    self.rwrite(r, lo, self.stage[r], g.N)
        health = {"dead_endpoints": sorted((r, c) for r in range(self.n) for c in range(self.K) if self.known_ep_dead[r][c]),
                  "dead_links": sorted((r, c) for r in range(self.n) for c in range(self.K) if self.known_link_dead[r][c])}
        return SimResult(self.recv, self.events, self.detections, self.bytes_sent, self.error, health,
                         self.retx_items, self.retx_bytes, list(self.fired), self.hbm)


def simulate(xs, geom: Geometry, dtype: str, **kw) -> SimResult:
    """Run the Layer-2 protocol simulation for one collective (geom.op)."""
    if geom.n == 1 or geom.N == 0:
        y = [np.array(x, copy=True) for x in xs]
        return SimResult(y, [], [], np.zeros((geom.n, geom.K), dtype=np.int64), None,
                         {"dead_endpoints": [], "dead_links": []}, 0, 0, [])
    return Simulator(xs, geom, dtype, **kw).run()
