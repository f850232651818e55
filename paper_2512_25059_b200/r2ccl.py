"""Thin ctypes binding of the C ABI in include/r2ccl.h (argument marshalling
only -- every step of the allreduce runs in libr2ccl.so's kernels and its
C++ control plane).  Names follow the C entry points.

The product path fails loudly when the library is missing: there is no CPU
fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes as C
import os
import uuid

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "lib", "libr2ccl.so")

MAX_CHANNELS = 16
MAX_LOCAL = 16
MAX_RANKS = 64

# r2_result_t
SUCCESS, ERR_INVALID_ARG, ERR_CUDA, ERR_BOOTSTRAP, ERR_NOT_REGISTERED, ERR_NO_BACKUP, ERR_TIMEOUT, ERR_INTERNAL = range(8)
# r2_dtype_t
INT32, FLOAT32, BFLOAT16 = 0, 1, 2
DTYPE_NAMES = {"int32": INT32, "float32": FLOAT32, "bfloat16": BFLOAT16}
# strategies
HOT_REPAIR, BALANCE = 0, 1
# fault kinds
FAULT_LOCAL, FAULT_REMOTE, FAULT_LINK, FAULT_REPAIR = 0, 1, 2, 3
FAULT_KINDS = {"LOCAL": 0, "REMOTE": 1, "LINK": 2, "REPAIR": 3, "HEAL": 4}
# probe outcomes / verdicts
PROBE_NAMES = {0: "S", 1: "L", 2: "T", 3: "-"}
VERDICT_NAMES = ["NONE", "LOCAL_ENDPOINT", "REMOTE_ENDPOINT", "LINK", "ENDPOINT_UNREACHABLE_A",
                 "ENDPOINT_UNREACHABLE_B", "DUAL_ENDPOINT", "TWO_LOCAL", "INCONCLUSIVE"]


class R2Error(RuntimeError):
    def __init__(self, code: int, what: str = ""):
        self.code = code
        msg = lib().r2_strerror(code).decode() if _LIB is not None else str(code)
        super().__init__(f"{what}: {msg} (r2_result_t={code})")


class Config(C.Structure):
    _fields_ = [("nchannels", C.c_int), ("ctas_per_channel", C.c_int), ("threads_per_cta", C.c_int),
                ("chunk_bytes", C.c_size_t), ("max_bytes", C.c_size_t), ("strategy", C.c_int),
                ("probe_timeout_us", C.c_int), ("watchdog_ms", C.c_int),
                ("channel_w", C.c_int * MAX_CHANNELS), ("use_channel_w", C.c_int), ("sim_ranks", C.c_int),
                ("protocol", C.c_int), ("ll_max_bytes", C.c_size_t), ("alpha_simple_ns", C.c_int),
                ("alpha_ll_ns", C.c_int), ("beta_mbps", C.c_int), ("reprobe_us", C.c_int),
                ("reprobe_max_us", C.c_int), ("channel_gbps", C.c_int), ("allreduce_algo", C.c_int),
                ("alpha_launch_ns", C.c_int), ("alpha_ll128_ns", C.c_int), ("rerank", C.c_int),
                ("r2cc_stage1_eff_pct", C.c_int), ("r2cc_stage2_eff_pct", C.c_int)]


PROTO_AUTO, PROTO_SIMPLE, PROTO_LL, PROTO_LL128 = 0, 1, 2, 3
ALGO_AUTO, ALGO_RING, ALGO_R2CC = 0, 1, 2


class Fault(C.Structure):
    _fields_ = [("at_seq", C.c_uint64), ("src_rank", C.c_int), ("channel", C.c_int), ("origin_channel", C.c_int),
                ("kind", C.c_int), ("step", C.c_int), ("chunk", C.c_int), ("byte_offset", C.c_uint64),
                ("detect_delay_us", C.c_int), ("poison", C.c_int)]


class Verdict(C.Structure):
    _fields_ = [("kind", C.c_int), ("a", C.c_int), ("b", C.c_int), ("aux", C.c_int), ("channel", C.c_int),
                ("outcome", C.c_int * 4)]

    def as_dict(self) -> dict:
        return {"verdict": VERDICT_NAMES[self.kind], "a": self.a, "b": self.b,
                "aux": None if self.aux < 0 else self.aux, "channel": self.channel,
                "outcomes": tuple(PROBE_NAMES[o] for o in self.outcome[: (4 if self.aux >= 0 else 2)])}


class Event(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("rank", C.c_int), ("origin_channel", C.c_int), ("stopped_channel", C.c_int),
                ("verdict", Verdict), ("resume", C.c_int), ("floor", C.c_int), ("retransmit", C.c_int),
                ("strategy", C.c_int), ("assignee", C.c_int), ("chain_pos", C.c_int),
                ("shares", C.c_int * MAX_CHANNELS), ("error", C.c_int),
                ("t_fire_dev_ns", C.c_uint64), ("t_first_retx_dev_ns", C.c_uint64),
                ("t_detect_host_ns", C.c_uint64), ("t_verdict_host_ns", C.c_uint64), ("t_plan_host_ns", C.c_uint64),
                ("failover_ms", C.c_double), ("notify_acks", C.c_int), ("notify_peer_acked", C.c_int),
                ("notify_ack_ms", C.c_double)]

    def as_dict(self, K: int) -> dict:
        d = {"seq": self.seq, "rank": self.rank, "origin": self.origin_channel,
             "stopped_channel": self.stopped_channel, "resume": self.resume, "floor": self.floor,
             "retransmit": self.retransmit, "strategy": "HOT_REPAIR" if self.strategy == 0 else "BALANCE",
             "error": self.error, "failover_ms": self.failover_ms,
             "t_fire_dev_ns": self.t_fire_dev_ns, "t_first_retx_dev_ns": self.t_first_retx_dev_ns,
             "t_detect_host_ns": self.t_detect_host_ns, "t_verdict_host_ns": self.t_verdict_host_ns,
             "t_plan_host_ns": self.t_plan_host_ns, "notify_acks": self.notify_acks,
             "notify_peer_acked": bool(self.notify_peer_acked), "notify_ack_ms": self.notify_ack_ms}
        d.update(self.verdict.as_dict())
        if self.strategy == 0:
            d["assignee"], d["chain_pos"] = self.assignee, self.chain_pos
        else:
            d["shares"] = {c: self.shares[c] for c in range(K) if self.shares[c] > 0}
        return d


class Status(C.Structure):
    _fields_ = [("seq", C.c_uint64), ("last_error", C.c_int), ("last_error_seq", C.c_uint64),
                ("n_events", C.c_int), ("world", C.c_int), ("nlocal", C.c_int), ("nchannels", C.c_int),
                ("dead_endpoints", C.c_uint32 * (MAX_LOCAL * 4)), ("dead_links", C.c_uint32 * (MAX_LOCAL * 4)),
                ("bytes", (C.c_uint64 * MAX_CHANNELS) * MAX_LOCAL), ("last_protocol", C.c_int),
                ("n_readmits", C.c_int), ("n_reprobes", C.c_int), ("n_service_kernels", C.c_int),
                ("n_r2cc", C.c_int), ("r2cc_rank", C.c_int), ("r2cc_X", C.c_double), ("r2cc_Y", C.c_double),
                ("r2cc_NA", C.c_uint64), ("r2cc_NP", C.c_uint64), ("r2cc_seq", C.c_uint64),
                ("n_rerank", C.c_int), ("ring_order", C.c_int * MAX_RANKS)]


class Geometry(C.Structure):
    _fields_ = [("N", C.c_uint64), ("Np", C.c_uint64), ("shard", C.c_uint64), ("slice", C.c_uint64),
                ("chunk", C.c_uint64), ("n", C.c_int), ("K", C.c_int), ("W", C.c_int), ("V", C.c_int),
                ("m", C.c_int), ("steps", C.c_int), ("stride", C.c_uint64), ("t0", C.c_int),
                ("local_step", C.c_int)]


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t)
POST_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_size_t)
POLL_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_int), C.c_void_p, C.c_size_t, C.POINTER(C.c_size_t))
BARRIER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p)


class Oob(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", C.c_void_p), ("post", C.c_void_p), ("poll", C.c_void_p),
                ("barrier", C.c_void_p)]


# Every symbol include/r2ccl.h declares (checked by tests/test_abi.py).
EXPORTS = {
    "r2_config_default": (None, [C.POINTER(Config)]),
    "r2_init": (C.c_int, [C.c_int, C.c_int, C.c_int, C.POINTER(Oob), C.POINTER(Config), C.POINTER(C.c_void_p)]),
    "r2_register_multi": (C.c_int, [C.c_void_p, C.c_void_p, C.c_size_t, C.POINTER(C.c_uint64)]),
    "r2_deregister": (C.c_int, [C.c_void_p, C.c_uint64]),
    "r2_allreduce": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "r2_allreduce_host": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "r2_inject_fault": (C.c_int, [C.c_void_p, C.POINTER(Fault)]),
    "r2_probe": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(Verdict)]),
    "r2_status": (C.c_int, [C.c_void_p, C.POINTER(Status)]),
    "r2_get_event": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(Event)]),
    "r2_sync": (C.c_int, [C.c_void_p]),
    "r2_finalize": (C.c_int, [C.c_void_p]),
    "r2_trace": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_uint64)]),
    "r2_strerror": (C.c_char_p, [C.c_int]),
    "r2_triangulate": (C.c_int, [C.POINTER(C.c_int), C.c_int]),
    "r2_balance_shares": (C.c_int, [C.c_uint64, C.POINTER(C.c_int), C.c_uint32, C.c_int, C.POINTER(C.c_uint64)]),
    "r2_failover_chain": (None, [C.c_int, C.c_int, C.POINTER(C.c_int)]),
    "r2_rollback": (None, [C.POINTER(C.c_uint8), C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "r2_rerank": (C.c_int, [C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_uint32), C.POINTER(C.c_uint32),
                            C.POINTER(C.c_int)]),
    "r2_geometry": (C.c_int, [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t, C.POINTER(Geometry)]),
    "r2_geometry_op": (C.c_int, [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_size_t,
                                 C.POINTER(Geometry)]),
    "r2_reduce_scatter": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "r2_all_gather": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_void_p]),
    "r2_broadcast": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_void_p]),
    "r2_oob_shm_open": (C.c_int, [C.c_char_p, C.c_int, C.c_int, C.POINTER(Oob)]),
    "r2_oob_shm_close": (C.c_int, [C.POINTER(Oob)]),
}

_LIB = None


def lib() -> C.CDLL:
    """Load libr2ccl.so (raises if it was not built: no fallback)."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2512_25059_b200.build` "
                               "(the CUDA extension is required; there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in EXPORTS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _LIB = L
    return _LIB


def _check(rc: int, what: str):
    if rc != SUCCESS:
        raise R2Error(rc, what)


def config_default(**kw) -> Config:
    cfg = Config()
    lib().r2_config_default(C.byref(cfg))
    for k, v in kw.items():
        if k == "channel_w":
            for i, w in enumerate(v):
                cfg.channel_w[i] = int(w)
            cfg.use_channel_w = 1
        elif k == "strategy" and isinstance(v, str):
            cfg.strategy = {"HOT_REPAIR": HOT_REPAIR, "BALANCE": BALANCE}[v]
        elif k == "protocol" and isinstance(v, str):
            cfg.protocol = {"AUTO": PROTO_AUTO, "SIMPLE": PROTO_SIMPLE, "LL": PROTO_LL, "LL128": PROTO_LL128}[v]
        elif k == "allreduce_algo" and isinstance(v, str):
            cfg.allreduce_algo = {"AUTO": ALGO_AUTO, "RING": ALGO_RING, "R2CC": ALGO_R2CC}[v]
        else:
            setattr(cfg, k, v)
    return cfg


# ------------------------------------------------------------ host logic

def triangulate(outcomes, has_aux: bool) -> str:
    code = {"S": 0, "L": 1, "T": 2}
    arr = (C.c_int * 4)(*[code[o] for o in (list(outcomes) + ["S"] * 4)[:4]])
    return VERDICT_NAMES[lib().r2_triangulate(arr, int(has_aux))]


def balance_shares(R: int, weights, healthy) -> dict:
    K = len(weights)
    w = (C.c_int * K)(*weights)
    mask = 0
    for c in healthy:
        mask |= 1 << c
    out = (C.c_uint64 * K)()
    _check(lib().r2_balance_shares(R, w, mask, K, out), "r2_balance_shares")
    return {c: int(out[c]) for c in range(K) if (mask >> c) & 1}


def failover_chain(c: int, K: int) -> list:
    out = (C.c_int * max(K - 1, 1))()
    lib().r2_failover_chain(c, K, out)
    return list(out[: K - 1])


def rerank(ring, rails, dead_links=None) -> list:
    """Algorithm 1 (r2ccl.h r2_rerank): ring order, per-rank alive-channel
    masks, optional per-rank dead standard-link masks -> R'."""
    n = len(ring)
    rin = (C.c_int * n)(*ring)
    rm = (C.c_uint32 * n)(*rails)
    dl = (C.c_uint32 * n)(*dead_links) if dead_links is not None else None
    out = (C.c_int * n)()
    if lib().r2_rerank(n, rin, rm, dl, out) < 0:
        raise ValueError("r2_rerank: invalid arguments")
    return list(out)


def rollback(completed) -> tuple:
    n = len(completed)
    arr = (C.c_uint8 * max(n, 1))(*[1 if x else 0 for x in completed])
    r, f = C.c_int(), C.c_int()
    lib().r2_rollback(arr, n, C.byref(r), C.byref(f))
    return r.value, f.value


OP_ALLREDUCE, OP_REDUCE_SCATTER, OP_ALL_GATHER, OP_BROADCAST = 0, 1, 2, 3
OPS = {"allreduce": OP_ALLREDUCE, "reduce_scatter": OP_REDUCE_SCATTER, "all_gather": OP_ALL_GATHER,
       "broadcast": OP_BROADCAST}


def geometry(count: int, dtype: int, n: int, K: int, W: int, chunk_bytes: int, op: int = OP_ALLREDUCE) -> Geometry:
    g = Geometry()
    _check(lib().r2_geometry_op(op, count, dtype, n, K, W, chunk_bytes, C.byref(g)), "r2_geometry_op")
    return g


# ------------------------------------------------------------ OOB

def oob_shm_open(name: str, rank: int, world: int) -> Oob:
    o = Oob()
    _check(lib().r2_oob_shm_open(name.encode(), rank, world, C.byref(o)), "r2_oob_shm_open")
    return o


def oob_shm_close(o: Oob):
    _check(lib().r2_oob_shm_close(C.byref(o)), "r2_oob_shm_close")


def oob_allgather(o: Oob, data: bytes, world: int) -> list:
    n = len(data)
    src = C.create_string_buffer(data, n)
    dst = C.create_string_buffer(n * world)
    _check(ALLGATHER_FN(o.allgather)(o.ctx, src, dst, n), "oob allgather")
    return [dst.raw[i * n:(i + 1) * n] for i in range(world)]


def oob_barrier(o: Oob):
    _check(BARRIER_FN(o.barrier)(o.ctx), "oob barrier")


def oob_post(o: Oob, dst: int, data: bytes):
    buf = C.create_string_buffer(data, len(data))
    _check(POST_FN(o.post)(o.ctx, dst, buf, len(data)), "oob post")


def oob_poll(o: Oob, cap: int = 256):
    buf = C.create_string_buffer(cap)
    src, ln = C.c_int(-1), C.c_size_t(0)
    got = POLL_FN(o.poll)(o.ctx, C.byref(src), buf, cap, C.byref(ln))
    return (src.value, buf.raw[: ln.value]) if got == 1 else None


def unique_name() -> str:
    return "r2ccl_" + uuid.uuid4().hex[:16]


# ------------------------------------------------------------ communicator

class Comm:
    """An r2ccl communicator (one per process; k simulated ranks in sim mode)."""

    def __init__(self, rank: int, world: int, device: int, oob: Oob | None = None, cfg: Config | None = None):
        self._h = C.c_void_p()
        self.cfg = cfg if cfg is not None else config_default()
        self._oob = oob
        rc = lib().r2_init(rank, world, device, C.byref(oob) if oob is not None else None, C.byref(self.cfg),
                           C.byref(self._h))
        _check(rc, "r2_init")
        self.rank, self.world, self.device = rank, world, device
        self.sim = world == 1 and self.cfg.sim_ranks > 1
        self.n = self.cfg.sim_ranks if self.sim else world
        self.K = self.cfg.nchannels

    @property
    def handle(self):
        return self._h

    def register_multi(self, ptr: int, nbytes: int) -> int:
        reg = C.c_uint64()
        _check(lib().r2_register_multi(self._h, C.c_void_p(ptr), nbytes, C.byref(reg)), "r2_register_multi")
        return reg.value

    def deregister(self, reg: int):
        _check(lib().r2_deregister(self._h, reg), "r2_deregister")

    def allreduce(self, send_ptr: int, recv_ptr: int, count: int, dtype: int, stream: int = 0):
        _check(lib().r2_allreduce(self._h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), count, dtype,
                                  C.c_void_p(stream)), "r2_allreduce")

    def reduce_scatter(self, send_ptr: int, recv_ptr: int, recvcount: int, dtype: int, stream: int = 0):
        _check(lib().r2_reduce_scatter(self._h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), recvcount, dtype,
                                       C.c_void_p(stream)), "r2_reduce_scatter")

    def all_gather(self, send_ptr: int, recv_ptr: int, sendcount: int, dtype: int, stream: int = 0):
        _check(lib().r2_all_gather(self._h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), sendcount, dtype,
                                   C.c_void_p(stream)), "r2_all_gather")

    def broadcast(self, send_ptr: int, recv_ptr: int, count: int, dtype: int, root: int, stream: int = 0):
        _check(lib().r2_broadcast(self._h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), count, dtype, root,
                                  C.c_void_p(stream)), "r2_broadcast")

    def allreduce_host(self, send_ptr: int, recv_ptr: int, count: int, dtype: int, stream: int = 0):
        _check(lib().r2_allreduce_host(self._h, C.c_void_p(send_ptr), C.c_void_p(recv_ptr), count, dtype,
                                       C.c_void_p(stream)), "r2_allreduce_host")

    def inject_fault(self, at_seq: int, kind: str, src_rank: int, channel: int, step: int = 0, chunk: int = 0,
                     byte_offset: int = 0, origin_channel: int = -1, detect_delay_us: int = 0, poison: int = 0):
        f = Fault(at_seq, src_rank, channel, origin_channel, FAULT_KINDS[kind], step, chunk, byte_offset,
                  detect_delay_us, poison)
        _check(lib().r2_inject_fault(self._h, C.byref(f)), "r2_inject_fault")

    def probe(self, peer: int, channel: int, rank_local: int = 0) -> dict:
        v = Verdict()
        _check(lib().r2_probe(self._h, rank_local, peer, channel, C.byref(v)), "r2_probe")
        return v.as_dict()

    def status(self) -> dict:
        s = Status()
        _check(lib().r2_status(self._h, C.byref(s)), "r2_status")
        n, K = s.world, s.nchannels
        return {"seq": s.seq, "last_error": s.last_error, "last_error_seq": s.last_error_seq,
                "n_events": s.n_events,
                "dead_endpoints": sorted((r, c) for r in range(n) for c in range(K) if (s.dead_endpoints[r] >> c) & 1),
                "dead_links": sorted((r, c) for r in range(n) for c in range(K) if (s.dead_links[r] >> c) & 1),
                "bytes": [[int(s.bytes[l][c]) for c in range(K)] for l in range(s.nlocal)],
                "last_protocol": {PROTO_SIMPLE: "SIMPLE", PROTO_LL: "LL", PROTO_LL128: "LL128"}.get(s.last_protocol, "NONE"),
                "n_readmits": s.n_readmits, "n_reprobes": s.n_reprobes,
                "n_service_kernels": s.n_service_kernels,
                "r2cc": {"calls": s.n_r2cc, "rank": s.r2cc_rank, "X": s.r2cc_X, "Y": s.r2cc_Y,
                         "NA": int(s.r2cc_NA), "NP": int(s.r2cc_NP), "seq": int(s.r2cc_seq)},
                "n_rerank": s.n_rerank, "ring_order": list(s.ring_order[:n])}

    def events(self) -> list:
        st = Status()
        _check(lib().r2_status(self._h, C.byref(st)), "r2_status")
        out = []
        for i in range(st.n_events):
            e = Event()
            _check(lib().r2_get_event(self._h, i, C.byref(e)), "r2_get_event")
            out.append(e.as_dict(self.K))
        return out

    def sync(self) -> int:
        """Synchronize the last stream; returns the pending async r2_result_t."""
        return lib().r2_sync(self._h)

    def finalize(self):
        if self._h:
            _check(lib().r2_finalize(self._h), "r2_finalize")
            self._h = C.c_void_p()
