"""Pins for oracle/collectives.py: the values the tree collectives produce.

Anchors: textbook bf16 round-to-nearest-even cases, hand-computed fp32 results
for a tree order that matters, exact integer arithmetic (any tree, any order),
the definition of Broadcast (a bitwise copy), and the one-hop-star = naive
left-to-right sum identity (R#12)."""
import random
from fractions import Fraction

import numpy as np
import pytest

import synth
from oracle import collectives as C
from oracle import packing


# ------------------------------------------------------------------ bf16
@pytest.mark.parametrize("x,bits", [
    (1.0, 0x3F80),
    (1.0 + 2 ** -8, 0x3F80),              # tie -> even (down)
    (1.0 + 3 * 2 ** -9, 0x3F81),          # above the tie -> up
    (1.0 + 3 * 2 ** -8, 0x3F82),          # tie between 0x3F81 and 0x3F82 -> even (up)
    (-2.0, 0xC000),
    (0.0, 0x0000),
    (-0.0, 0x8000),
    (float("inf"), 0x7F80),
    (3.4028234663852886e38, 0x7F80),     # FLT_MAX rounds to +inf in bf16
    (3.3895313892515355e38, 0x7F7F),     # bf16 max is exact
    (1e-40, 0x0001),                     # subnormal: 0x000116C2 -> 0x0001
])
def test_bf16_rne(x, bits):
    assert int(C.f32_to_bf16(np.array([x], dtype=np.float32))[0]) == bits


def test_bf16_nan_and_roundtrip():
    assert np.isnan(C.bf16_to_f32(C.f32_to_bf16(np.array([np.nan], np.float32))))[0]
    h = np.arange(0, 65536, dtype=np.uint32).astype(np.uint16)
    fin = ~np.isnan(C.bf16_to_f32(h))
    assert np.array_equal(C.f32_to_bf16(C.bf16_to_f32(h))[fin], h[fin])


# ------------------------------------------------------------------ fp32 order
def _chain_plan(parent, root):
    return dict(trees=[dict(parent=tuple(parent), root=root, weight=Fraction(1))])


def test_fp32_tree_order_hand_computed():
    # send0 = 1, send1 = 1e8, send2 = -1e8 (one element each)
    sends = [np.array([v], np.float32) for v in (1.0, 1e8, -1e8)]
    # star at 1 (the path 0-1-2's centre): operands in tag order 0,1,2:
    # fl(fl(1 + 1e8) - 1e8) = fl(1e8 - 1e8) = 0
    star = _chain_plan([1, -1, 1], 1)
    assert C.allreduce(star, sends, "f32", "sum")[0] == 0.0
    # chain rooted at 0 (0 <- 1 <- 2): partial_1 = fl(1e8 + -1e8) = 0;
    # root: fl(1 + 0) = 1
    chain = _chain_plan([-1, 0, 1], 0)
    assert C.allreduce(chain, sends, "f32", "sum")[0] == 1.0
    # bf16 rounds once per node: 256 + 1 + 1 -> star: 258 (exact in bf16? 258 = 0x4381 yes)
    b = [C.f32_to_bf16(np.array([v], np.float32)) for v in (256.0, 1.0, 1.0)]
    assert float(C.bf16_to_f32(C.allreduce(star, b, "bf16", "sum"))[0]) == 258.0
    # chain rooted at 2 (2 <- 1 <- 0): partial_0 = 256, partial_1 = rne(256 + 1) = 256
    # (257 is a tie between 256 and 258 -> even mantissa 256), root: rne(256 + 1) = 256
    chain2 = _chain_plan([1, 2, -1], 2)
    assert float(C.bf16_to_f32(C.allreduce(chain2, b, "bf16", "sum"))[0]) == 256.0


def test_onehop_star_equals_naive_left_to_right():
    m, count = 5, 4099
    sends = synth.inputs(3, m, count, "f32")
    plan = packing.plan_switch_allreduce(m)
    got = C.allreduce(plan, sends, "f32", "sum")
    naive = sends[0].copy()
    for s in sends[1:]:
        naive = naive + s       # float32 + float32 in numpy: IEEE RNE
    assert np.array_equal(got.view(np.uint32), naive.view(np.uint32))


# ------------------------------------------------------------------ exactness
def _random_tree(rng, m):
    parent = [-1] * m
    order = list(range(m))
    rng.shuffle(order)
    root = order[0]
    for i in range(1, m):
        parent[order[i]] = order[rng.randrange(i)]
    return tuple(parent), root


@pytest.mark.parametrize("seed", range(8))
@pytest.mark.parametrize("op", ["sum", "min", "max", "prod"])
def test_int32_exact_under_any_trees(seed, op):
    rng = random.Random(seed)
    m = rng.randint(1, 7)
    count = rng.randint(1, 300)
    sends = synth.inputs(4, m, count, "i32")
    if op == "prod":
        sends = [(s % 7 - 3).astype(np.int32) for s in sends]
    k = rng.randint(1, 4)
    trees = []
    for _ in range(k):
        p, r = _random_tree(rng, m)
        trees.append(dict(parent=p, root=r, weight=Fraction(rng.randint(1, 4), rng.randint(1, 3))))
    got = C.allreduce(dict(trees=trees), sends, "i32", op)
    # exact reference with Python integers, wrapped to int32
    for e in range(count):
        vals = [int(s[e]) for s in sends]
        if op == "sum":
            ref = sum(vals)
        elif op == "prod":
            ref = 1
            for v in vals:
                ref *= v
        elif op == "min":
            ref = min(vals)
        else:
            ref = max(vals)
        ref = (ref + 2**31) % 2**32 - 2**31
        assert int(got[e]) == ref


def test_float_min_max_exact_and_signed_zero():
    sends = [np.array([0.0, -0.0, 1.0, np.nan, 3.0], np.float32),
             np.array([-0.0, 0.0, np.nan, 2.0, -np.inf], np.float32)]
    plan = packing.plan_switch_allreduce(2)
    mn = C.allreduce(plan, sends, "f32", "min")
    mx = C.allreduce(plan, sends, "f32", "max")
    assert np.signbit(mn[0]) and np.signbit(mn[1])
    assert not np.signbit(mx[0]) and not np.signbit(mx[1])
    assert mn[2] == 1.0 and mn[3] == 2.0 and mn[4] == -np.inf
    assert mx[2] == 1.0 and mx[3] == 2.0 and mx[4] == 3.0


def test_fp32_sum_within_bound_of_naive_for_any_tree():
    # |tree - naive| <= (m-1) u sum|x| per element (standard summation bound)
    rng = random.Random(11)
    m, count = 8, 2000
    sends = synth.inputs(5, m, count, "f32")
    for _ in range(5):
        p, r = _random_tree(rng, m)
        got = C.allreduce(dict(trees=[dict(parent=p, root=r, weight=Fraction(1))]), sends, "f32", "sum")
        exact = np.sum(np.array(sends, dtype=np.float64), axis=0)
        absum = np.sum(np.abs(np.array(sends, dtype=np.float64)), axis=0)
        assert np.all(np.abs(got - exact) <= 2 * (m - 1) * 2.0**-24 * absum + 1e-45)


# ------------------------------------------------------------------ broadcast
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_broadcast_is_bitwise_copy(dtype):
    m, count = 4, 1031
    sends = synth.inputs(6, m, count, dtype)
    plan = packing.plan_switch_broadcast(m, 2)
    recvs = C.broadcast(plan, sends, 2, dtype)
    for r in recvs:
        assert r.tobytes() == sends[2].tobytes()


def test_element_ranges_cover_everything():
    plan = packing.plan_switch_allreduce(3)
    for dtype in ("f32", "bf16", "i32"):
        for count in (0, 1, 3, 5, 17, 262144):
            rngs = C.tree_element_ranges(plan, count, dtype)
            assert rngs[0][0] == 0 and rngs[-1][1] == count
            assert all(b == c for (_, b), (c, _) in zip(rngs, rngs[1:]))


def test_c1_allreduce_split_matches_survey():
    # C1 AllReduce 1 MiB fp32 over 3 trees: {87380, 87380, 87384}
    plan = packing.plan_switch_allreduce(3)
    rngs = C.tree_element_ranges(plan, 262144, "f32")
    assert [hi - lo for lo, hi in rngs] == [87380, 87380, 87384]


# ------------------------------------------------------------------ NEXT-3 duals
@pytest.mark.parametrize("m", [1, 2, 3, 8])
def test_reduce_scatter_then_allgather_is_onehop_allreduce(m):
    # structural identity: RS followed by AG reproduces the one-hop AllReduce
    # bit for bit (same trees, same operand order)
    B = 1031
    for dtype in ("f32", "bf16", "i32"):
        sends = synth.inputs(12, m, m * B, dtype)
        rs = C.reduce_scatter(sends, dtype, "sum")
        ag = C.allgather(rs)
        ar = C.allreduce(packing.plan_switch_allreduce(m), sends, dtype, "sum")
        # the AllReduce splits by 16-byte grains, RS by blocks; compare element-wise
        # on the union: both are the per-element ascending-rank reduction
        assert np.array_equal(bits_of(ag), bits_of(C.naive_reduce(sends, dtype, "sum")))
        assert np.array_equal(bits_of(ar), bits_of(ag))


def bits_of(a):
    a = np.asarray(a)
    return a.view(np.uint16) if a.dtype.itemsize == 2 else a.view(np.uint32)


def test_reduce_scatter_int_exact_and_allgather_blocks():
    m, B = 5, 77
    sends = synth.inputs(13, m, m * B, "i32")
    rs = C.reduce_scatter(sends, "i32", "max")
    for j in range(m):
        for e in range(B):
            assert int(rs[j][e]) == max(int(s[j * B + e]) for s in sends)
    ag = C.allgather([s[:B] for s in sends])
    for j in range(m):
        assert ag[j * B:(j + 1) * B].tobytes() == sends[j][:B].tobytes()


def test_gather_is_allgather_at_the_root_only():
    m, B = 4, 33
    sends = synth.inputs(14, m, B, "bf16")
    g = C.gather(sends, 2)
    assert g[0] is None and g[1] is None and g[3] is None
    assert g[2].tobytes() == C.allgather(sends).tobytes()
    # inverse of Broadcast: block j of the root's result is exactly rank j's send
    for j in range(m):
        assert g[2][j * B:(j + 1) * B].tobytes() == sends[j].tobytes()


# ------------------------------------------------------------------ AVG (R#28)
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_avg_of_identical_inputs_is_the_input(dtype):
    """Every rank sends the same x (values whose m-fold sums are exact): the
    average is x exactly, on the one-hop plan and on a multi-level tree."""
    from oracle import graphs
    vals = np.array([0.75, -1.5, 3.0, 0.0, 96.0, -0.125], dtype=np.float32)
    x = C.f32_to_bf16(vals) if dtype == "bf16" else vals
    for m, plan in ((8, packing.plan_switch_allreduce(8)),
                    (8, packing.plan_allreduce_graph(graphs.dgx1p())),
                    (5, packing.plan_switch_allreduce(5))):
        got = C.allreduce(plan, [x] * m, dtype, "avg")
        assert np.array_equal(np.asarray(got).view(np.uint16 if dtype == "bf16" else np.uint32),
                              np.asarray(x).view(np.uint16 if dtype == "bf16" else np.uint32))


def test_avg_int32_truncates_toward_zero():
    """C integer division: (sum) / m truncates toward 0 (-7 / 2 = -3); the sum
    is exact (wraparound arithmetic under any tree)."""
    m = 4
    sends = [np.array([1, -1, 2, -2, 10, -10, 0], dtype=np.int32) * (r + 1) for r in range(m)]
    # sum over r of (r + 1) = 10  ->  10 * base / 4
    base = np.array([1, -1, 2, -2, 10, -10, 0])
    want = np.array([int(v * 10 / 4) for v in base], dtype=np.int32)   # trunc toward 0
    for plan in (packing.plan_switch_allreduce(m),):
        assert np.array_equal(C.allreduce(plan, sends, "i32", "avg"), want)
    assert list(C.naive_reduce(sends, "i32", "avg")) == [2, -2, 5, -5, 25, -25, 0]


def test_avg_fp32_root_divides_once():
    """Hand-computed: one-hop, m = 3, inputs 1, 2, 4: sum 7 then 7 / 3 rounded
    once (RNE) = 2.3333333 (0x40155555); dividing each input first would
    give a different last bit (1/3 + 2/3 + 4/3 = 0x40155556)."""
    sends = [np.array([v], dtype=np.float32) for v in (1.0, 2.0, 4.0)]
    got = C.allreduce(packing.plan_switch_allreduce(3), sends, "f32", "avg")
    assert got.view(np.uint32)[0] == 0x40155555
    pre = np.float32(np.float32(np.float32(1.0) / np.float32(3)) + np.float32(np.float32(2.0) / np.float32(3)))
    pre = np.float32(pre + np.float32(np.float32(4.0) / np.float32(3)))
    assert pre.view(np.uint32) != 0x40155555
