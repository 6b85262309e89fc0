import sys, os, time
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1910_04940_b200 as B
import synth
from oracle import collectives as OC, graphs as OG
cases = {"chain3": B.Graph(3, [(0, 1, 1.0, 1), (1, 2, 1.0, 1)]),
         "dgx1v": B.Graph.from_pairs(8, OG.dgx1v()[1])}
for name, G in cases.items():
    m = 8 if name == "dgx1v" else 3
    for per_rank in (0, 1):
        for n in (1000, 70001):
            comms = B.init_all([0] * m, graph=G, cfg=B.config(timeout_s=3.0, launch_per_rank=per_rank))
            sends = synth.inputs(171, m, m * n, "i32")
            ds = [torch.from_numpy(s).cuda() for s in sends]
            outs = [torch.zeros(n, dtype=torch.int32, device="cuda") for _ in range(m)]
            t = time.time()
            for r, c in enumerate(comms):
                c.reduce_scatter(ds[r], outs[r], op="max", recvcount=n, dtype="i32")
            torch.cuda.synchronize()
            want = OC.reduce_scatter(sends, "i32", "max")
            print(name, per_rank, n, "time %.2f" % (time.time() - t), [bool(np.array_equal(outs[r].cpu().numpy(), want[r])) for r in range(m)], flush=True)
            for c in comms:
                c.destroy()
