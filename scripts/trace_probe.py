#!/usr/bin/env python
"""Where the time goes inside one launch (BLINK_TRACE=1): per trace point,
median / max over CTAs of (stamp - earliest CTA start), in microseconds."""
import os
import statistics
import sys

os.environ["BLINK_TRACE"] = "1"
import torch  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1910_04940_b200 as B  # noqa: E402

NAMES = ["start", "epoch", "entry-done", "1st-load", "1st-store", "stores-done", "work-end", "epoch-upd"]


def main():
    m = int(sys.argv[1]) if len(sys.argv) > 1 else 8
    comms = B.init_all([0] * m)
    for nbytes in (1024, 1 << 20, 16 << 20, 256 << 20):
        cnt = nbytes // 4
        xs = [torch.randn(cnt, device="cuda") for _ in range(m)]
        ys = [torch.empty_like(x) for x in xs]
        for _ in range(3):
            for r, c in enumerate(comms):
                c.allreduce(xs[r], ys[r])
        torch.cuda.synchronize()
        tr = comms[0].trace()
        t0 = min(t[0] for t in tr)
        line = []
        for k, name in enumerate(NAMES):
            vals = [(t[k] - t0) / 1e3 for t in tr if t[k]]
            if vals:
                line.append(f"{name}={statistics.median(vals):.1f}/{max(vals):.1f}")
        print(f"m={m} bytes={nbytes} ctas={len(tr)}: " + " ".join(line), flush=True)


if __name__ == "__main__":
    main()
