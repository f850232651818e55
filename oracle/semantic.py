"""Layer 1 of the oracle: WHAT the fault-tolerant collectives compute
(AllReduce; standalone ReduceScatter / AllGather at the end of the file).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The method reaches exactly the plain ring-allreduce result, just survivably
("this preserves data integrity"; "retransmits only the remaining
data").  So the result is the plain definition of a ring AllReduce =
ReduceScatter followed by AllGather (Fig. 3 at P:83-88):

  for every element i of shard s (owner s) and every rank r
      y_r[i] = fold(x_{s+1}[i], x_{s+2}[i], ..., x_{s+n-1}[i], x_s[i])

a left fold along the ring that starts at owner+1 and ends at the owner (the
order in which the ring reduce-scatter visits the ranks; SURVEY §8(c) Layer 1,
reading C-8).  Per dtype (readings C-8, C-9):

  int32    two's-complement wrap (computed in uint32)
  float32  IEEE fp32 add, round-to-nearest-even, at every hop
  bfloat16 each hop is bf16_rne(fp32(acc) + fp32(x))  -- the wire format is
           bf16, so the partial is rounded at every hop (NOT "exact sum
           rounded once").

bf16 values are carried as uint16 bit patterns.
"""
from __future__ import annotations

import numpy as np

# ---------------------------------------------------------------- bf16 helpers


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    """bf16 bit pattern -> fp32 value (exact: bf16 is the top half of fp32)."""
    return (np.asarray(bits, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16_rne(f: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 with IEEE round-to-nearest-even (reading C-8).

    Keep the top 16 bits; the dropped low half decides: above half -> up,
    below half -> down, exactly half -> to the even upper pattern.  Adding
    0x7FFF + (lsb of the kept half) and truncating implements exactly that
    (carry into the exponent gives the correct overflow to the next binade /
    infinity).  NaN is kept quiet.
    """
    u = np.asarray(f, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (u >> np.uint64(16)) & np.uint64(1)
    rounded = ((u + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)
    is_nan = (u & np.uint64(0x7FFFFFFF)) > np.uint64(0x7F800000)
    if np.any(is_nan):
        rounded = np.where(is_nan, ((u >> np.uint64(16)) | np.uint64(0x40)).astype(np.uint16), rounded)
    return rounded


# ----------------------------------------------------------------- one hop


def hop_add(acc: np.ndarray, x: np.ndarray, dtype: str) -> np.ndarray:
    """One reduction hop acc (+) x in the wire dtype (readings C-8/C-9)."""
    if dtype == "int32":
        s = np.asarray(acc, dtype=np.int32).view(np.uint32) + np.asarray(x, dtype=np.int32).view(np.uint32)
        return s.astype(np.uint32).view(np.int32)
    if dtype == "float32":
        return (np.asarray(acc, dtype=np.float32) + np.asarray(x, dtype=np.float32)).astype(np.float32)
    if dtype == "bfloat16":
        return f32_to_bf16_rne(bf16_to_f32(acc) + bf16_to_f32(x))
    raise ValueError(dtype)


def np_dtype(dtype: str):
    return {"int32": np.int32, "float32": np.float32, "bfloat16": np.uint16}[dtype]


# ----------------------------------------------------------------- the fold


def ring_fold(values_by_rank: list[np.ndarray], owner: int, dtype: str) -> np.ndarray:
    """fold(x_{s+1}, ..., x_{s+n-1}, x_s) for owner s (SURVEY §8(c) Layer 1)."""
    n = len(values_by_rank)
    if n == 1:
        return np.array(values_by_rank[0], copy=True)
    acc = np.array(values_by_rank[(owner + 1) % n], copy=True)
    for k in range(2, n + 1):          # ranks owner+2, ..., owner+n (= owner)
        acc = hop_add(acc, values_by_rank[(owner + k) % n], dtype)
    return acc


def allreduce(xs: list[np.ndarray], shard_elems: int, dtype: str) -> np.ndarray:
    """The allreduce result y (identical on every rank).

    ``shard_elems`` = N'/n, the padded shard length (oracle/geometry.py); the
    owner of element i is i // shard_elems ("a ReduceScatter retains only
    a 1/n shard").  Elements past N are padding and never exist in y.
    """
    n = len(xs)
    N = len(xs[0])
    y = np.empty(N, dtype=np_dtype(dtype))
    if N == 0:
        return y
    if n == 1:
        y[:] = xs[0]
        return y
    for s in range(n):
        lo, hi = s * shard_elems, min((s + 1) * shard_elems, N)
        if lo >= hi:
            continue
        y[lo:hi] = ring_fold([x[lo:hi] for x in xs], s, dtype)
    return y


def reduce_scatter(xs: list[np.ndarray], recvcount: int, dtype: str) -> list[np.ndarray]:
    """Standalone ReduceScatter ("a ReduceScatter retains only a 1/n
    shard"; P:94 the first half of the ring AllReduce).

    Rank r's input holds n*recvcount elements (shard s = [s*recvcount,
    (s+1)*recvcount)); rank r keeps shard r, reduced with the same ring fold
    as the AllReduce's reduce-scatter half: fold(x_{r+1}, ..., x_{r-1}, x_r).
    Returns the n output shards (rank r's is element r).
    """
    n = len(xs)
    out = []
    for r in range(n):
        lo, hi = r * recvcount, (r + 1) * recvcount
        out.append(ring_fold([np.asarray(x)[lo:hi] for x in xs], r, dtype))
    return out


def all_gather(shards: list[np.ndarray]) -> np.ndarray:
    """Standalone AllGather ("an AllGather must receive the same amount";
    P:94 the second half of the ring AllReduce): every rank ends with the
    concatenation shard_0 | shard_1 | ... | shard_{n-1}.  A pure copy: the bits
    of every shard are preserved."""
    return np.concatenate([np.asarray(s) for s in shards]) if shards else np.empty(0)


def broadcast(xs: list[np.ndarray], root: int) -> list[np.ndarray]:
    """Standalone Broadcast ("in a Broadcast, the root sends D_total while
    all others receive it"): every rank ends with
    the root's buffer, bits preserved."""
    return [np.array(xs[root], copy=True) for _ in xs]


def exact_sum_f64(xs: list[np.ndarray], dtype: str) -> np.ndarray:
    """The float64 sum (the 'exact' reference of the normwise bound, §8(c))."""
    if dtype == "bfloat16":
        vals = [bf16_to_f32(x).astype(np.float64) for x in xs]
    else:
        vals = [np.asarray(x).astype(np.float64) for x in xs]
    return np.sum(vals, axis=0)


def as_float64(y: np.ndarray, dtype: str) -> np.ndarray:
    return bf16_to_f32(y).astype(np.float64) if dtype == "bfloat16" else np.asarray(y).astype(np.float64)


def normwise_rel_error(y: np.ndarray, xs: list[np.ndarray], dtype: str) -> float:
    """||y - exact||_2 / ||exact||_2 (the north star's fp32/bf16 tolerances
    are read normwise, SURVEY §8(c) 'Tolerance statement')."""
    ex = exact_sum_f64(xs, dtype)
    den = float(np.linalg.norm(ex))
    num = float(np.linalg.norm(as_float64(y, dtype) - ex))
    return num / den if den > 0 else num


def r2cc_allreduce(xs: list[np.ndarray], dtype: str, f: int, NA: int, shard_A: int, shard_P: int) -> np.ndarray:
    """R²CCL-AllReduce (§5.2 "Partial AllReduce" / "R²CCL-AllReduce";
    DESIGN.md reading R-9): the result every rank holds.

    * elements [0, NA): the global ring AllReduce over all n ranks (stage 1,
      P:113 "a global AllReduce ... spans all servers") -- the Layer-1 fold
      above with shards of shard_A elements;
    * elements [NA, N): the partial AllReduce over the n-1 ranks other than
      the degraded rank f ("the partial AllReduce excludes the failure
      node"), a ring in rank order with f removed -- the same fold over that
      rank list, shards of shard_P elements -- followed by the tailored
      broadcast: f's contribution is added once, at the rank after f,
      as one hop acc (+) x with acc = the partial result and x = x_f, and the
      sum travels on unchanged.
    """
    n = len(xs)
    N = len(xs[0])
    y = np.empty(N, dtype=np_dtype(dtype))
    if NA:
        y[:NA] = allreduce([np.asarray(x)[:NA] for x in xs], shard_A, dtype)
    if NA < N:
        healthy = [np.asarray(xs[r])[NA:] for r in range(n) if r != f]
        p = allreduce(healthy, shard_P, dtype)
        y[NA:] = hop_add(p, np.asarray(xs[f])[NA:], dtype)
    return y


def allreduce_ring(xs: list[np.ndarray], order: list[int], shard_elems: int, dtype: str) -> np.ndarray:
    """AllReduce on a re-ranked ring ("most collective algorithms are
    symmetric and agnostic to node ordering, enabling safe reordering";
    Algorithm 1's R'): the Layer-1 fold with ring position p held by rank
    order[p] -- shard s is folded over the ranks at positions s+1, s+2, ...,
    s, as in `allreduce`, so only the order of the hops changes."""
    return allreduce([xs[r] for r in order], shard_elems, dtype)
