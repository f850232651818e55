"""Pins for oracle Layer 1 (oracle/semantic.py) against things the paper and
the mathematics fix: IEEE rounding worked by hand, a library bf16 conversion,
Python big-int sums, closed forms and special cases.  CPU only."""
import numpy as np
import pytest
import torch

import r2inputs
from oracle import semantic as S
from oracle.geometry import Geometry


def f32(v):
    return np.array(v, dtype=np.float32)


def bits(v):
    return int(np.asarray(v, dtype=np.uint16))


# ------------------------------------------------------------ bf16 rounding

@pytest.mark.parametrize("value,expected", [
    (1.0, 0x3F80),
    (1.0 + 2 ** -8, 0x3F80),            # exact tie -> even (1.0)
    (1.0 + 3 * 2 ** -8, 0x3F82),        # exact tie -> even (1 + 2^-6)
    (1.0 + 2 ** -8 + 2 ** -20, 0x3F81), # just above the tie -> up
    (1.0 + 2 ** -9, 0x3F80),            # below half -> down
    (-(1.0 + 2 ** -8), 0xBF80),
    (257.0, 0x4380),                    # 257 = 1.00000001b * 2^8: tie -> 256
    (259.0, 0x4382),                    # 259 tie -> 260 (even)
    (3.3895313892515355e38, 0x7F7F),    # max bf16 finite stays
])
def test_bf16_rne_hand_values(value, expected):
    """Hand-derived IEEE round-to-nearest-even cases (reading C-8)."""
    assert bits(S.f32_to_bf16_rne(f32([value]))[0]) == expected


def test_bf16_rne_overflow_to_inf():
    # 0x7F7FFFFF (max fp32) is above the largest bf16 + half ulp -> +inf
    v = np.array([0x7F7FFFFF], dtype=np.uint32).view(np.float32)
    assert bits(S.f32_to_bf16_rne(v)[0]) == 0x7F80


def test_bf16_rne_matches_torch_library_conversion():
    """torch's fp32->bf16 cast is RNE (library routine, independent code)."""
    rng = np.random.default_rng(7)
    raw = rng.integers(0, 2 ** 32, size=200_000, dtype=np.uint64).astype(np.uint32)
    f = raw.view(np.float32)
    f = f[np.isfinite(f)]
    ours = S.f32_to_bf16_rne(f)
    lib = torch.from_numpy(f.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, lib)


def test_bf16_to_f32_exact():
    b = np.arange(0, 2 ** 16, dtype=np.uint32).astype(np.uint16)
    f = S.bf16_to_f32(b)
    fin = np.isfinite(f)
    lib = torch.from_numpy(b.view(np.int16).copy()).view(torch.bfloat16).float().numpy()
    assert np.array_equal(f[fin], lib[fin])


# ------------------------------------------------------------ one hop

def test_int32_wraps():
    a = np.array([2 ** 31 - 1, -(2 ** 31), -1], dtype=np.int32)
    b = np.array([1, -1, 1], dtype=np.int32)
    assert S.hop_add(a, b, "int32").tolist() == [-(2 ** 31), 2 ** 31 - 1, 0]


def test_fp32_hop_is_single_rounding():
    # 2^24 + 1 is not representable: RNE tie -> 2^24 (even)
    assert S.hop_add(f32([2.0 ** 24]), f32([1.0]), "float32")[0] == np.float32(2.0 ** 24)
    assert S.hop_add(f32([2.0 ** 24]), f32([3.0]), "float32")[0] == np.float32(2.0 ** 24 + 4)


def test_bf16_hop_rounds_per_hop():
    one = S.f32_to_bf16_rne(f32([1.0]))
    tiny = S.f32_to_bf16_rne(f32([2 ** -8]))
    # 1 + 2^-8 is a tie in bf16 -> 1.0; adding it twice per hop stays 1.0,
    # while the exact sum 1 + 2^-7 would be representable.
    acc = S.hop_add(one, tiny, "bfloat16")
    acc = S.hop_add(acc, tiny, "bfloat16")
    assert bits(acc[0]) == 0x3F80


# ------------------------------------------------------------ the fold order

def test_fold_order_fp32_hand_example():
    """n=3; owner s sees fold(x_{s+1}, x_{s+2}, x_s).  With x0=-2^24, x1=2^24,
    x2=1 (all in shard 0): (x1+x2)+x0 = 2^24 + (-2^24) = 0 (the +1 is lost to
    RNE), while any order starting at x0 would give 1.  In shard 1 the fold is
    (x2+x0)+x1 = (1-2^24)+2^24 = 1; in shard 2 it is (x0+x1)+x2 = 0+1 = 1."""
    n, sh = 3, 4
    xs = [np.zeros(n * sh, np.float32) for _ in range(n)]
    for s in range(n):
        xs[0][s * sh] = -(2.0 ** 24)
        xs[1][s * sh] = 2.0 ** 24
        xs[2][s * sh] = 1.0
    y = S.allreduce(xs, sh, "float32")
    assert y[0] == 0.0
    assert y[sh] == 1.0
    assert y[2 * sh] == 1.0


def test_fold_order_bf16_hand_example():
    """n=3, bf16 (8 significant bits): x0 = 1, x1 = 256, x2 = 1.
    shard 0: (x1+x2)+x0 = bf16(257)=256, +1 -> 256.
    shard 1: (x2+x0)+x1 = 2 + 256 = 258 (representable).
    shard 2: (x0+x1)+x2 = 256 + 1 -> 256."""
    n, sh = 3, 8
    enc = lambda v: S.f32_to_bf16_rne(f32([v]))[0]
    xs = [np.zeros(n * sh, np.uint16) for _ in range(n)]
    for s in range(n):
        xs[0][s * sh], xs[1][s * sh], xs[2][s * sh] = enc(1.0), enc(256.0), enc(1.0)
    y = S.bf16_to_f32(S.allreduce(xs, sh, "bfloat16"))
    assert (y[0], y[sh], y[2 * sh]) == (256.0, 258.0, 256.0)


# ------------------------------------------------------------ closed forms

@pytest.mark.parametrize("n", [2, 3, 4, 8])
@pytest.mark.parametrize("dist", ["default", "wrap"])
def test_int32_equals_bigint_sum_mod_2_32(n, dist):
    N = 4096
    xs = r2inputs.inputs(n, N, "int32", seed=11 + n, dist=dist)
    g = Geometry(n, 2, N, 4, 256)
    y = S.allreduce(xs, g.shard, "int32")
    for i in range(0, N, 37):
        tot = sum(int(x[i]) for x in xs) % (1 << 32)
        if tot >= 1 << 31:
            tot -= 1 << 32
        assert int(y[i]) == tot


@pytest.mark.parametrize("dtype", ["float32", "bfloat16"])
@pytest.mark.parametrize("n", [2, 3, 8])
def test_small_integers_are_exact(dtype, n):
    """Inputs in [-16, 16) (exact in bf16) and n <= 8 keep |partial sums| <= 128 < 2^8 -> every hop
    is exact, so the result is the exact integer sum."""
    N = 2048
    xs = r2inputs.inputs(n, N, dtype, seed=5, dist="smallint")
    g = Geometry(n, 2, N, 4 if dtype == "float32" else 2, 256)
    y = S.as_float64(S.allreduce(xs, g.shard, dtype), dtype)
    assert np.array_equal(y, S.exact_sum_f64(xs, dtype))


def test_n1_is_copy_and_n2_is_one_hop():
    x = r2inputs.inputs(2, 1000, "bfloat16", seed=3)
    g1 = Geometry(1, 2, 1000, 2, 256)
    assert np.array_equal(S.allreduce([x[0]], g1.shard, "bfloat16"), x[0])
    g2 = Geometry(2, 2, 1000, 2, 256)
    y = S.allreduce(x, g2.shard, "bfloat16")
    # n=2: y = bf16(f32(x_other) + f32(x_owner)) computed directly in fp32
    ref = S.f32_to_bf16_rne(S.bf16_to_f32(x[0]) + S.bf16_to_f32(x[1]))
    assert np.array_equal(y, ref)


@pytest.mark.parametrize("dtype,tol", [("float32", 1e-6), ("bfloat16", 1e-2)])
def test_normwise_bound(dtype, tol):
    """North star tolerances, read normwise."""
    n, N = 8, 1 << 16
    xs = r2inputs.inputs(n, N, dtype, seed=9)
    g = Geometry(n, 8, N, r2inputs.elem_bytes(dtype), 4096)
    y = S.allreduce(xs, g.shard, dtype)
    assert S.normwise_rel_error(y, xs, dtype) < tol


def test_int_sum_invariant_and_ring_order():
    """Σ_i y[i] ≡ Σ_r Σ_i x_r[i] (mod 2^32); int results do not depend on the
    ring order -- permuting the ranks permutes nothing in y."""
    n, N = 5, 3000
    xs = r2inputs.inputs(n, N, "int32", seed=2, dist="wrap")
    g = Geometry(n, 3, N, 4, 64)
    y = S.allreduce(xs, g.shard, "int32")
    lhs = int(y.astype(np.int64).sum()) % (1 << 32)
    rhs = sum(int(x.astype(np.int64).sum()) for x in xs) % (1 << 32)
    assert lhs == rhs
    y2 = S.allreduce(xs[::-1], g.shard, "int32")
    assert np.array_equal(y, y2)
