"""Seeded synthetic inputs shared by the oracle-side tests and the product-side
tests/bench.  Holds NONE of the method's arithmetic: only random numbers and
fixed edge-case patterns (SURVEY 8(d) "Concrete synthetic inputs").

  seed(config, rank) = 191004940 + 1000 * config + rank
  f32  : N(0, 1) * 1e-2 (gradient-like)
  bf16 : the f32 values rounded to bf16 (bit patterns as uint16)
  i32  : uniform in [-2^20, 2^20]

The bf16 rounding here uses numpy's float32 -> uint16 bit trick (RNE); it is an
input recipe, not a reduction step, and the oracle's own RNE is pinned
separately (tests/test_oracle_numerics.py).
"""
import numpy as np

BASE_SEED = 191004940


def seed(config, rank):
    return BASE_SEED + 1000 * int(config) + int(rank)


def _rne_bf16_bits(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    return ((b + 0x7FFF + ((b >> 16) & 1)) >> 16).astype(np.uint16)


def rank_input(config, rank, count, dtype):
    """One rank's send buffer as a numpy array (float32 / uint16 bf16 bits / int32)."""
    g = np.random.Generator(np.random.PCG64(seed(config, rank)))
    if dtype == "f32":
        return (g.standard_normal(count, dtype=np.float32) * np.float32(1e-2)).astype(np.float32)
    if dtype == "bf16":
        return _rne_bf16_bits(g.standard_normal(count, dtype=np.float32) * np.float32(1e-2))
    if dtype == "i32":
        return g.integers(-(1 << 20), (1 << 20) + 1, size=count, dtype=np.int32)
    raise ValueError(dtype)


def inputs(config, m, count, dtype):
    return [rank_input(config, r, count, dtype) for r in range(m)]


def edge_case_f32(config, rank, count):
    """Edge-case set: +-0, subnormals, +-1e30 cancellation pairs, mixed with
    gradient-like values.  Rank-dependent signs so that reductions cancel."""
    g = np.random.Generator(np.random.PCG64(seed(config, rank) + 7))
    x = g.standard_normal(count, dtype=np.float32) * np.float32(1e-2)
    kind = g.integers(0, 6, size=count)
    sgn = np.float32(1.0 if rank % 2 == 0 else -1.0)
    x = np.where(kind == 0, np.float32(0.0) * sgn, x)                     # +-0
    x = np.where(kind == 1, np.float32(1e-40) * sgn, x)                   # subnormal
    x = np.where(kind == 2, np.float32(1e30) * sgn, x)                    # cancellation pair
    x = np.where(kind == 3, np.float32(-0.0), x)
    return x.astype(np.float32)


def sentinel_like(count, esize):
    """0xFF-filled receive buffer (unwritten bytes stay visible)."""
    return np.full(count * esize, 0xFF, dtype=np.uint8)


# PyTorch DDP bucket sequences (element counts), not from the paper.
BUCKETS = {
    ("resnet50", "f32"): [2049000, 7875584, 6563840, 6637568, 2431040],
    ("resnet50", "bf16"): [2049000, 14439424, 9068608],
    ("vgg16", "f32"): [4097000, 16781312, 102764544, 7079424, 7079936, 555328],
    ("vgg16", "bf16"): [4097000, 16781312, 102764544, 13569280, 1145408],
}


def device_input(config, rank, count, dtype, device="cuda"):
    """Large seeded inputs generated on the device (torch's Philox generator):
    same recipe (N(0,1)*1e-2 / its bf16 rounding / uniform int), used where
    host generation would dominate (full-size parity samples and the bench).
    Oracle comparisons copy the sampled inputs back to the host."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed(config, rank))
    if dtype == "i32":
        return torch.randint(-(1 << 20), (1 << 20) + 1, (count,), generator=g, device=device,
                             dtype=torch.int32)
    x = torch.randn(count, generator=g, device=device, dtype=torch.float32) * 1e-2
    return x if dtype == "f32" else x.to(torch.bfloat16)
