"""Pins of the oracle's R²CCL-AllReduce (PAPER.md:106-136
§5.2, App. A :358-447; readings R-9, R-11) against what the paper
and arithmetic fix: the closed-form integer sum, hand-derived IEEE cases
where the fold order decides the value, the plain ring as the Y = 0 special
case, faulted == healthy by brute force over stage-2 fault points, per-rank
stage-2 traffic, and App. A's threshold theorem for the strategy choice."""
import itertools
import math

import numpy as np
import pytest

import r2inputs
from oracle import cost as C
from oracle import protocol as OP
from oracle import semantic as OS
from oracle.geometry import ALLREDUCE, STAGE2, Geometry


def big_sum(xs):
    tot = sum(np.asarray(x, dtype=np.int64) for x in xs)
    return ((tot + 2 ** 31) % 2 ** 32 - 2 ** 31).astype(np.int32)


def shards(N, n, K, V):
    q = n * K * V
    return -(-max(N, 1) // q) * q // n


@pytest.mark.parametrize("n,f", [(3, 0), (3, 2), (4, 1), (5, 4), (8, 3)])
@pytest.mark.parametrize("N,frac", [(1, 0.0), (1000, 0.4), (12_345, 0.7), (40_000, 0.999)])
def test_int32_result_is_the_wrapped_sum(n, f, N, frac):
    """Whatever the split and the degraded rank: every element is the sum of
    all n inputs mod 2^32 (a dropped contribution or a shifted region fails)."""
    xs = r2inputs.inputs(n, N, "int32", seed=n * 100 + f, dist="wrap")
    NA, NP = C.r2cc_split(N, 4, frac)
    y = OS.r2cc_allreduce(xs, "int32", f, NA, shards(NA, n, 3, 4), shards(NP, n - 1, 2, 4))
    assert np.array_equal(y, big_sum(xs))


def test_fp32_fold_order_hand_derived():
    """n = 4, f = 1, the whole buffer in the partial ring (N_A = 0), one shard
    per partial-ring position of 4 elements.  Partial ring = ranks [0, 2, 3];
    element 0 lies in shard 0 (owner: position 0 = rank 0), so
    p = (x2 + x3) + x0 and then z = p + x1 (IEEE fp32, RNE):
      x = (1, 0, 2^24, 1):  2^24 + 1 -> 2^24 (tie to even), + 1 -> 2^24, + 0
                            -> 16777216; any order adding x3 + x0 first gives
                            16777218.
      x = (0, 1, 2^24, 1):  p = 2^24, z = 2^24 + 1 -> 16777216; adding f's 1
                            before the partial's tie gives 16777218.
    Element 4 lies in shard 1 (owner rank 2): p = (x3 + x0) + x2:
      x = (1, 5, 2^24, 1):  2 + 2^24 = 16777218 exactly, + 5 -> 16777223 ->
                            RNE to 16777224."""
    two24 = float(2 ** 24)
    cols = [(1.0, 0.0, two24, 1.0), (0.0, 1.0, two24, 1.0), (0.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0),
            (1.0, 5.0, two24, 1.0), (0.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0),
            (0.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0)]
    xs = [np.array([c[r] for c in cols], dtype=np.float32) for r in range(4)]
    y = OS.r2cc_allreduce(xs, "float32", 1, 0, 4, 4)
    assert y[0] == np.float32(16777216.0)
    assert y[1] == np.float32(16777216.0)
    assert y[4] == np.float32(16777224.0)


def test_bf16_small_integers_exact():
    """bf16 inputs that are small integers: every partial sum is exact in bf16,
    so the result is the exact sum whatever the fold order."""
    n, N = 5, 3000
    rng = np.random.default_rng(4)
    ints = [rng.integers(-8, 8, N) for _ in range(n)]
    xs = [OS.f32_to_bf16_rne(a.astype(np.float32)) for a in ints]
    NA, NP = C.r2cc_split(N, 8, 0.55)
    y = OS.r2cc_allreduce(xs, "bfloat16", 2, NA, shards(NA, n, 4, 8), shards(NP, n - 1, 4, 8))
    assert np.array_equal(OS.bf16_to_f32(y), np.sum(ints, axis=0).astype(np.float32))


def test_y_zero_is_the_plain_ring():
    """App. A Step 3: Y = 0 below the threshold -> N_P = 0 -> the plain ring."""
    n, N = 6, 7777
    xs = r2inputs.inputs(n, N, "float32", seed=6)
    NA, NP = C.r2cc_split(N, 4, C.optimal_partition(n, 1, 0.2))
    assert (NA, NP) == (N, 0)
    sh = shards(N, n, 4, 4)
    assert np.array_equal(OS.r2cc_allreduce(xs, "float32", 3, NA, sh, 1).view(np.uint32),
                          OS.allreduce(xs, sh, "float32").view(np.uint32))


def test_split_rule():
    """Reading R-9: N_A = N - floor(Y N / V) V rounded up to a vector (<= N),
    N_P = N - N_A: the partial region starts on a 16-byte boundary."""
    assert C.r2cc_split(1000, 4, 0.5) == (500, 500)
    assert C.r2cc_split(1001, 8, 0.5) == (512, 489)
    assert C.r2cc_split(1001, 4, 0.5294) == (476, 525)
    assert C.r2cc_split(10, 4, 0.99) == (4, 6)
    assert C.r2cc_split(7, 8, 0.9) == (7, 0)
    for N in range(1, 200):
        for V in (4, 8):
            NA, NP = C.r2cc_split(N, V, 0.61)
            assert NA + NP == N and NA % V == 0 or NA == N


def stage2(xs, p, n, K, N, f, E, chunk, dtype, **kw):
    g = Geometry(n, K, N, E, chunk, STAGE2, root=f)
    init = [p if r != f else np.zeros(N, dtype=OS.np_dtype(dtype)) for r in range(n)]
    return g, OP.simulate(xs, g, dtype, recv_init=init, **kw)


@pytest.mark.parametrize("dtype", ["int32", "float32", "bfloat16"])
def test_layer2_stages_equal_layer1(dtype):
    """Stage 1 (global ring on channels A, partial ring of the healthy ranks on
    channels P) then stage 2 (tailored broadcast) simulated with the protocol
    model give Layer 1's R²CCL-AllReduce on every rank."""
    n, N, f, E = 4, 3001, 2, r2inputs.elem_bytes(dtype)
    V = 16 // E
    xs = r2inputs.inputs(n, N, dtype, seed=9)
    NA, NP = C.r2cc_split(N, V, 0.6)
    KA, KP = 3, 2
    gA = Geometry(n, KA, NA, E, 256)
    rA = OP.simulate([x[:NA] for x in xs], gA, dtype, seed=1)
    hr = [r for r in range(n) if r != f]
    gP = Geometry(n - 1, KP, NP, E, 256)
    rP = OP.simulate([xs[r][NA:] for r in hr], gP, dtype, seed=2)
    p = rP.y[0]
    assert all(np.array_equal(rP.y[i], p) for i in range(n - 1))
    _, r2 = stage2([x[NA:] for x in xs], p, n, 5, NP, f, E, 128, dtype, seed=3)
    want = OS.r2cc_allreduce(xs, dtype, f, NA, gA.shard, gP.shard)
    for r in range(n):
        got = np.concatenate([rA.y[r], r2.y[r]])
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), r


def test_stage2_traffic_each_rank_sends_the_region_once():
    """the tailored broadcast moves YD through every rank: f sends its
    contribution once, every other rank forwards the sum once (padded region)."""
    n, K, N, f = 5, 2, 1000, 1
    xs = r2inputs.inputs(n, N, "int32", seed=1)
    p = np.zeros(N, dtype=np.int32)
    g, res = stage2(xs, p, n, K, N, f, 4, 256, "int32")
    for r in range(n):
        assert res.bytes_sent[r].sum() == g.shard * 4


@pytest.mark.parametrize("kind", ["LINK", "LOCAL", "REMOTE"])
def test_stage2_brute_force_single_faults(kind):
    """Every (rank, channel, chunk, byte offset) of stage 2 at the rank's chain
    step: the faulted run equals the healthy run bit for bit (rollback +
    re-placement on the chain's ring connections)."""
    n, K, N, f, E = 3, 2, 24, 0, 4
    xs = r2inputs.inputs(n, N, "float32", seed=2)
    p = OS.allreduce([xs[r] for r in range(n) if r != f], 12, "float32")
    g, ok = stage2(xs, p, n, K, N, f, E, 16, "float32")
    for r, c, j, b in itertools.product(range(n), range(K), range(g.m), (0, 8)):
        t = (r - f) % n
        fl = [OP.Fault(kind, r, c, t, j, b)]
        _, res = stage2(xs, p, n, K, N, f, E, 16, "float32", faults=fl, seed=r + c + j)
        assert res.error is None
        for q in range(n):
            assert np.array_equal(res.y[q].view(np.uint32), ok.y[q].view(np.uint32)), (r, c, j, b, q)
        assert len(res.events) >= 1


def test_stage2_no_backup_with_one_channel():
    n, N = 3, 40
    xs = r2inputs.inputs(n, N, "int32", seed=5)
    p = np.zeros(N, dtype=np.int32)
    _, res = stage2(xs, p, n, 1, N, 0, 4, 16, "int32", faults=[OP.Fault("LINK", 1, 0, 1, 0, 0)])
    assert res.error == "NO_BACKUP"


def test_strategy_choice_matches_app_a_threshold():
    """Reading R-11 with alpha = launch = 0 reduces to the paper's bandwidth
    model, where App. A proves R²CCL-AllReduce (at Y*) beats the ring exactly
    when X > n / (3n - 2): the choice flips at the threshold."""
    for n in (3, 4, 8, 16):
        th = C.threshold(n, 1)
        for X in np.linspace(0.01, 0.99, 197):
            Y = C.optimal_partition(n, 1, X)
            t_ring, t_r2 = C.algo_times(n, X, Y, 1.0, 0.0, 1.0, 0.0)
            if X <= th:
                assert Y == 0 and t_r2 == math.inf
            else:
                assert t_r2 < t_ring, (n, X)


def test_strategy_choice_latency_bound():
    """With a per-step alpha the ring wins at small sizes even above the
    threshold (R²CCL-AllReduce pays n more steps and a launch), and
    R²CCL-AllReduce wins at large sizes: the crossover the paper attributes
    to the alpha-beta model."""
    n, X = 8, 0.75
    Y = C.optimal_partition(n, 1, X)
    small = C.algo_times(n, X, Y, 64e3, 7150.0, 650.0, 6000.0)
    big = C.algo_times(n, X, Y, 256e6, 7150.0, 650.0, 6000.0)
    assert small[0] < small[1] and big[1] < big[0]


def test_stage_efficiencies_shift_the_choice_toward_the_ring():
    """Reading R-11's calibration: dividing the stage terms by efficiencies
    below 1 only ever makes R²CCL-AllReduce slower (never changes the ring's
    time), so the set of X where it is chosen shrinks monotonically; with
    efficiencies 1 it is App. A's choice.  With the library's defaults
    (0.75, 0.50) the ring is chosen at X = 0.5 for n = 4 (measured: R²CCL
    0.68x the ring there) and R²CCL at X = 0.75 (measured 1.0x)."""
    for n in (3, 4, 8):
        chosen = {}
        for e1, e2 in ((1.0, 1.0), (0.9, 0.8), (0.75, 0.5), (0.5, 0.3)):
            chosen[(e1, e2)] = set()
            for X in np.linspace(0.01, 0.99, 99):
                Y = C.optimal_partition(n, 1, X)
                t_ring, t_r2 = C.algo_times(n, X, Y, 1.0, 0.0, 1.0, 0.0, e1, e2)
                t_ring1, _ = C.algo_times(n, X, Y, 1.0, 0.0, 1.0, 0.0)
                assert t_ring == t_ring1
                if t_r2 < t_ring:
                    chosen[(e1, e2)].add(round(X, 4))
        keys = list(chosen)
        for a, b in zip(keys, keys[1:]):
            assert chosen[b] <= chosen[a], (n, a, b)
    n = 4
    for X, want_r2 in ((0.5, False), (0.75, True)):
        Y = C.optimal_partition(n, 1, X)
        t_ring, t_r2 = C.algo_times(n, X, Y, 1.0, 0.0, 1.0, 0.0, 0.75, 0.5)
        assert (t_r2 < t_ring) == want_r2, X
