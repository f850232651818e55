"""Traffic and time bounds of the ring allreduce (and App. A planner values).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

P:78 (§5.1 Overhead Analysis): "a ReduceScatter retains only a 1/n shard and
must send (n-1)/n D_total; an AllGather must receive the same amount ... The
NCCL's ring algorithm realizes these lower bounds."  P:121: "The time for a
ring AllReduce is given by 2(ng-1)/(ng) x D/B."  P:122-136 and App. A
(P:358-447): T1, T2, T3, T(Y), Y*, threshold.

Pins (tests/test_oracle_host.py): nvlink_bytes_per_gpu and hbm_bytes_per_gpu
against the bytes the Layer-2 simulator actually moves (oracle/protocol.py
SimResult.bytes_sent / hbm_bytes) and SURVEY §8(d)'s printed table; App. A
against SPEC's printed values, T1(Y*) = T2(Y*) and a grid argmin.
"""
from __future__ import annotations

import math


def ring_allreduce_time(n: int, g: int, D: float, B: float) -> float:
    """2(ng-1)/(ng) * D/B."""
    ng = n * g
    return 2 * (ng - 1) / ng * D / B


def nvlink_bytes_per_gpu(S: float, n: int) -> float:
    """Bytes each GPU sends (= receives) in a push ring allreduce: 2(n-1)/n S."""
    return 2 * (n - 1) / n * S


def hbm_bytes_per_gpu(S: float, n: int) -> float:
    """Algorithmic HBM bytes per GPU (push ring, registered recv, fused final
    add): reads (3n-3)/n S + writes (2n-1)/n S = (5n-4)/n S.

    RS steps 0..n-2: read x slice (n-1 times), read scratch (n-2 times),
    write peer scratch lands in the peer's HBM (counted at the receiver:
    n-1 writes).  Final add: read scratch + x, write own recv (1 + 1 reads,
    1 write), the peer's recv write lands remotely.  AG: n-2 forwards read own
    recv; every shard except the own one lands in recv from the peer (n-1
    writes).  Per shard unit (S/n): reads (n-1)+(n-2)+2+(n-2) = 3n-3,
    writes (n-1)+1+(n-1) = 2n-1.
    """
    return (5 * n - 4) / n * S


# ------------------------------------------------------------- App. A (NEXT)

def stage_times(Y: float, n: int, g: int, X: float, D: float = 1.0, B: float = 1.0):
    """T1, T2, T3."""
    if not 0 < X < 1:
        raise ValueError("X must lie in (0, 1)")
    a = 2 * (n * g - 1) / (n * g)
    b = 2 * ((n - 1) * g - 1) / ((n - 1) * g)
    T1 = a * (1 - Y) * D / ((1 - X) * B)
    T2 = b * Y * D / (X * B)
    T3 = Y * D / (X * B)
    return T1, T2, T3


def total_time(Y, n, g, X, D=1.0, B=1.0) -> float:
    """T(Y) = max(T1, T2) + T3."""
    T1, T2, T3 = stage_times(Y, n, g, X, D, B)
    return max(T1, T2) + T3


def threshold(n: int, g: int) -> float:
    """App. A Step 2: X = ng / (3ng - 2)."""
    return n * g / (3 * n * g - 2)


def y_star(n: int, g: int, X: float) -> float:
    """App. A Step 1: Y* = X + X(1-X) / (X + (g(n-1)-1) n)."""
    return X + X * (1 - X) / (X + (g * (n - 1) - 1) * n)


def optimal_partition(n: int, g: int, X: float) -> float:
    """App. A Step 3: Y = 0 if X <= threshold else Y*."""
    return 0.0 if X <= threshold(n, g) else y_star(n, g, X)


def lost_fraction(weights, dead) -> float:
    """X of P:121 on the box (reading R-9): the degraded rank's lost share of
    its channel bandwidth, sum of its dead channels' weights over all."""
    return sum(weights[c] for c in dead) / sum(weights)


def r2cc_split(N: int, V: int, Y: float) -> tuple[int, int]:
    """Reading R-9: the global ring takes the first N_A elements, the partial
    AllReduce the last N_P = N - N_A, where N_A = N - floor(Y N / V) V rounded
    up to whole 16-byte vectors (so that the partial region starts 16-byte
    aligned; its own tail may be ragged), at most N."""
    NP0 = math.floor(Y * N / V) * V
    NA = min(N, -(-(N - NP0) // V) * V)
    return NA, N - NA


def algo_times(n: int, X: float, Y: float, S: float, alpha: float, B: float, launch: float,
               eff1: float = 1.0, eff2: float = 1.0):
    """Reading R-11 (the alpha-beta strategy choice of SURVEY §8(f) f3):
    per-call time of the ring on the degraded communicator and of
    R²CCL-AllReduce, each = (ring steps) x alpha + the paper's bandwidth terms
    (P:121-130 with g = 1, B = per-GPU rate): the ring is throttled to
    (1 - X) B at the degraded rank; R²CCL-AllReduce pays max(T1, T2) + T3 plus
    the n steps and the launch of its stage 2.  eff1 / eff2: the fraction of
    its bandwidth model stage 1 / stage 2 achieve (1 = the paper's model; the
    library's defaults are measured, reading R-11).  Returns (t_ring, t_r2cc)."""
    t_ring = (2 * n - 2) * alpha + ring_allreduce_time(n, 1, S, (1 - X) * B)
    if Y <= 0:
        return t_ring, float("inf")
    T1, T2, T3 = stage_times(Y, n, 1, X, S, B)
    # the partial ring has n - 1 members: P:123's (n-1)g ring factor
    return t_ring, (2 * n - 2) * alpha + max(T1, T2) / eff1 + n * alpha + T3 / eff2 + launch


def bottleneck_load(Y: float, D: float = 1.0) -> float:
    """Fig. 4 caption: degraded server volume 2(1-Y)D + YD."""
    return 2 * (1 - Y) * D + Y * D
