"""NEXT-1: the one-hop trees inside the NVSwitch (NVLS, P:440-442 realised
with multimem.ld_reduce / multimem.st).

* Any box: cfg.nvls = 1 on virtual ranks (one device) cannot build a
  multicast team, so the plan reports NVLS off with the reason and the P2P
  stars run -- results stay bit-exact.
* >= 2 GPUs (skipped on the 1-GPU box): AllReduce SUM against the oracle
  within the north_star tolerance (the switch's summation order is its own,
  R#29), int32 exact, Broadcast bitwise, ragged and misaligned buffers, calls
  larger than the multicast buffer (pieces)."""
import numpy as np
import pytest

import synth
from oracle import collectives as OC

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

from test_gpu_parity import B, assert_bitwise, to_dev, to_host, sentinel  # noqa: E402,F401


def ndev():
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def test_nvls_falls_back_on_one_device(B):
    comms = B.init_all([0] * 4, cfg=B.config(nvls=1, timeout_s=20.0))
    p = comms[0].plan(True, 0, 1 << 20, "f32")
    assert p["nvls"]["active"] is False and "device" in p["nvls"]["note"]
    count = (1 << 20) + 3
    sends = synth.inputs(180, 4, count, "f32")
    ds = [to_dev(s, "f32") for s in sends]
    out = [torch.empty_like(d) for d in ds]
    for r, c in enumerate(comms):
        c.allreduce(ds[r], out[r])
    torch.cuda.synchronize()
    want = OC.naive_reduce(sends, "f32", "sum")
    for o in out:
        assert_bitwise(to_host(o, "f32"), want)
    for c in comms:
        c.destroy()


def within_tolerance(got, sends, dtype):
    rtol = 1e-5 if dtype == "f32" else 1e-2
    f = (lambda x: OC.bf16_to_f32(x)) if dtype == "bf16" else (lambda x: x)
    naive = f(OC.naive_reduce(sends, dtype, "sum")).astype(np.float64)
    absum = sum(np.abs(f(s).astype(np.float64)) for s in sends)
    g = f(got).astype(np.float64)
    assert np.all(np.abs(g - naive) <= rtol * absum + 1e-30)


@pytest.mark.skipif(ndev() < 2, reason="NVLS needs >= 2 GPUs behind an NVSwitch")
@pytest.mark.parametrize("dtype", ["f32", "bf16", "i32"])
def test_nvls_allreduce_and_broadcast(B, dtype):
    m = ndev()
    comms = B.init_all(list(range(m)), cfg=B.config(nvls=1, nvls_bytes=4 << 20, timeout_s=20.0))
    p = comms[0].plan(True, 0, 8 << 20, dtype)
    assert p["nvls"]["active"] is True, p["nvls"]
    for count in ((3 << 20) + 5, 1 << 20):   # > nvls_bytes: pieces; ragged tail
        sends = synth.inputs(181, m, count, dtype)
        ds = [to_dev(sends[r], dtype).to(f"cuda:{r}") for r in range(m)]
        outs = [sentinel(count, dtype).to(f"cuda:{r}") for r in range(m)]
        for r, c in enumerate(comms):
            with torch.cuda.device(r):
                c.allreduce(ds[r], outs[r], op="sum", count=count, dtype=dtype)
        for r in range(m):
            torch.cuda.synchronize(r)
        for o in outs:
            got = to_host(o, dtype)
            if dtype == "i32":
                assert_bitwise(got, OC.naive_reduce(sends, "i32", "sum"))
            else:
                within_tolerance(got, sends, dtype)
        root = m - 1
        bouts = [sentinel(count, dtype).to(f"cuda:{r}") for r in range(m)]
        for r, c in enumerate(comms):
            with torch.cuda.device(r):
                c.broadcast(ds[r] if r == root else None, bouts[r], root=root, count=count, dtype=dtype)
        for r in range(m):
            torch.cuda.synchronize(r)
        for o in bouts:
            assert_bitwise(to_host(o, dtype), sends[root])
    for c in comms:
        c.destroy()
