#!/usr/bin/env python
"""Per-call device time (CUDA-graph replays of 10 calls) of one-hop AllReduce
at small m, in place vs out of place, over medium sizes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402
from scripts.ab_env import per_call_us  # noqa: E402


def main():
    for m in [int(x) for x in os.environ.get("PROBE_M", "2,4,8").split(",")]:
        comms = B.init_all([0] * m)
        for dt in (torch.float32, torch.bfloat16):
            out = []
            for nbytes in (4 << 20, 16 << 20, 29 << 20, 64 << 20):
                es = torch.finfo(dt).bits // 8
                xs = [torch.randn(nbytes // es, device="cuda").to(dt) for _ in range(m)]
                ys = [torch.empty_like(x) for x in xs]
                for inplace in (0, 1):
                    def fn():
                        for r, c in enumerate(comms):
                            c.allreduce(xs[r], xs[r] if inplace else ys[r])
                    us = per_call_us(fn, 10)
                    ideal = 2 * m * nbytes / 6.5e12 * 1e6
                    out.append(f"{nbytes >> 20}M{'i' if inplace else 'o'}:{us:.1f}({ideal / us:.2f})")
            print(f"m={m} {str(dt)[6:]} " + " ".join(out), flush=True)
        for c in comms:
            c.destroy()


if __name__ == "__main__":
    main()
