"""Broadcast / AllReduce values along packed trees.
TEST INFRASTRUCTURE ONLY (see oracle/__init__).

Sec. 4.1: Broadcast "split[s] the buffer among all the spanning trees
based on their weights" and forwards each piece along its tree.
Sec. 4.1 / Sec. 3.3: AllReduce "perform[s] reductions in
one direction to a root node.  Once the root node computes the final reduce
result, it is broadcast in the reverse direction."  Reduction functions: "all
the reduction functions supported by NCCL (e.g. min, max, etc.)" (R#14: SUM,
PROD, MIN, MAX).

The paper is silent on operand order and rounding; the oracle fixes them
(R#12, R#13):
  at node v, operands = {(v, send_v)} U {(c, partial_c) : c child of v},
  taken in ascending tag (rank) order; acc = first operand widened to fp32;
  acc = fl32(acc (op) x) for each next operand (RNE, no FMA);
  partial_v = round_RNE(acc) to the I/O dtype (one rounding per node).
The root's partial is the result and every rank receives it.  Chunking never
changes these values (the same per-element operations run for any chunk size).

Buffers are numpy arrays: float32, int32, or uint16 holding bf16 bit patterns.
"""
import numpy as np

from .packing import split_bytes

ESIZE = {"f32": 4, "bf16": 2, "i32": 4}


# ---------------------------------------------------------------------------
# bf16 <-> fp32 (bit-level; textbook round-to-nearest-even)
# ---------------------------------------------------------------------------
def bf16_to_f32(h):
    """Exact widening: the bf16 bits are the top 16 bits of the fp32 word."""
    return (np.asarray(h, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def f32_to_bf16(x):
    """Round-to-nearest-even fp32 -> bf16; NaN stays a (quiet) NaN."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    lsb = (b >> np.uint64(16)) & np.uint64(1)
    r = ((b + np.uint64(0x7FFF) + lsb) >> np.uint64(16)).astype(np.uint16)
    nan = np.isnan(np.asarray(x, dtype=np.float32))
    if nan.any():
        q = ((b >> np.uint64(16)).astype(np.uint16)) | np.uint16(0x0040)
        r = np.where(nan, q, r)
    return r


# ---------------------------------------------------------------------------
# Binary operators on fp32 / int32 arrays
# ---------------------------------------------------------------------------
def _fmin(a, b):
    """IEEE-754 minNum with -0 < +0: returns the smaller; if exactly one is
    NaN returns the other (R#14)."""
    r = np.where(a < b, a, b)
    r = np.where(a == b, np.where(np.signbit(a), a, b), r)
    r = np.where(np.isnan(a), b, np.where(np.isnan(b), a, r))
    return r.astype(a.dtype)


def _fmax(a, b):
    r = np.where(a > b, a, b)
    r = np.where(a == b, np.where(np.signbit(a), b, a), r)
    r = np.where(np.isnan(a), b, np.where(np.isnan(b), a, r))
    return r.astype(a.dtype)


def combine(op, a, b):
    """One step acc = acc (op) x, in the array's own dtype (fp32 or int32)."""
    with np.errstate(over="ignore", invalid="ignore"):
        if op == "sum":
            return (a + b).astype(a.dtype)          # fp32 RNE add / int32 wraparound
        if op == "prod":
            return (a * b).astype(a.dtype)          # fp32 RNE mul / int32 low 32 bits
        if op == "min":
            return np.minimum(a, b) if a.dtype == np.int32 else _fmin(a, b)
        if op == "max":
            return np.maximum(a, b) if a.dtype == np.int32 else _fmax(a, b)
    raise ValueError(op)


def _widen(x, dtype):
    if dtype == "bf16":
        return bf16_to_f32(x)
    if dtype == "f32":
        return np.asarray(x, dtype=np.float32)
    return np.asarray(x, dtype=np.int32)


def _narrow(acc, dtype):
    if dtype == "bf16":
        return f32_to_bf16(acc)
    return acc


def avg_divide(acc, m):
    """R#28 (AVG, "all the reduction functions supported by NCCL"): the
    tree root divides its fp32 / int32 accumulator by m before its rounding:
    IEEE fp32 division (RNE), or C integer division (truncation toward 0)."""
    if acc.dtype == np.int32:
        a = acc.astype(np.int64)
        return (np.sign(a) * (np.abs(a) // m)).astype(np.int32)
    return (acc / np.float32(m)).astype(np.float32)


def reduce_operands(operands, dtype, op, div=0):
    """Node combine: operands already sorted by tag.  Returns the node output.
    AVG combines as a sum; div > 0 (the tree root) divides before the
    rounding."""
    cop = "sum" if op == "avg" else op
    acc = _widen(operands[0], dtype).copy()
    for x in operands[1:]:
        acc = combine(cop, acc, _widen(x, dtype))
    if op == "avg" and div:
        acc = avg_divide(acc, div)
    return _narrow(acc, dtype)


def naive_reduce(sends, dtype, op):
    """sum_{j=0}^{m-1} send_j left to right in fp32 (int32), one final rounding.
    The tolerance reference of north_star (R#20).  AVG: that sum divided by m."""
    return reduce_operands(list(sends), dtype, op, div=len(sends))


# ---------------------------------------------------------------------------
# Tree collectives
# ---------------------------------------------------------------------------
def _children(parent):
    ch = {v: [] for v in range(len(parent))}
    for v, p in enumerate(parent):
        if p >= 0:
            ch[p].append(v)
    return ch


def tree_element_ranges(plan, count, dtype):
    """Element ranges per tree from the byte split (R#11)."""
    es = ESIZE[dtype]
    S = count * es
    rngs = split_bytes(S, [t["weight"] for t in plan["trees"]])
    return [(lo // es, hi // es) for (lo, hi) in rngs]


def allreduce(plan, sends, dtype, op):
    """AllReduce along the plan's trees (Sec. 3.3).  Returns the single
    result array every rank receives (all recvs are equal by construction)."""
    m = len(sends)
    count = len(sends[0])
    out = np.empty_like(np.asarray(sends[0]))
    for t, (lo, hi) in zip(plan["trees"], tree_element_ranges(plan, count, dtype)):
        assert m == len(t["parent"])
        if hi <= lo:
            continue
        ch = _children(t["parent"])

        def partial(v):                      # post-order value at v
            ops = [(v, sends[v][lo:hi])] + [(c, partial(c)) for c in ch[v]]
            ops.sort(key=lambda kv: kv[0])
            return reduce_operands([x for _, x in ops], dtype, op, div=m if v == t["root"] else 0)

        out[lo:hi] = partial(t["root"])
    return out


def broadcast(plan, sends, root, dtype):
    """Broadcast along the plan's trees: each tree's byte range is
    forwarded from the root down its edges.  Returns the list of m recvs."""
    m = len(sends)
    count = len(sends[0])
    recvs = [None] * m
    for v in range(m):
        recvs[v] = np.empty_like(np.asarray(sends[v]))
    for t, (lo, hi) in zip(plan["trees"], tree_element_ranges(plan, count, dtype)):
        ch = _children(t["parent"])
        assert t["root"] == root
        recvs[root][lo:hi] = sends[root][lo:hi]
        frontier = [root]
        while frontier:                       # top-down forwarding
            nxt = []
            for u in frontier:
                for c in ch[u]:
                    recvs[c][lo:hi] = recvs[u][lo:hi]
                    nxt.append(c)
            frontier = nxt
    return recvs


# ---------------------------------------------------------------------------
# NEXT-3 duals on one-hop trees ("Gather is the inverse of Broadcast,
# and AllGather is AllReduce without using a reduction function")
# ---------------------------------------------------------------------------
def reduce_scatter(sends, dtype, op):
    """The reduce half of the one-hop AllReduce: every rank's send
    holds m blocks of B elements; block j is reduced at its tree root j over
    the ranks in ascending order (R#12, one rounding).  Returns the m results
    (rank j receives block j)."""
    m = len(sends)
    B = len(sends[0]) // m
    return [reduce_operands([s[j * B:(j + 1) * B] for s in sends], dtype, op, div=m) for j in range(m)]


def allgather(sends):
    """AllReduce without a reduction: root j's block is broadcast to everyone,
    so every rank receives the blocks in rank order."""
    return np.concatenate([np.asarray(s) for s in sends])


def gather(sends, root):
    """Gather ("the inverse of Broadcast"): the root receives every
    rank's block in rank order; the other ranks receive nothing (None)."""
    return [np.concatenate([np.asarray(s) for s in sends]) if r == root else None
            for r in range(len(sends))]
