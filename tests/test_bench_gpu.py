"""bench.py's N > 1 path on the GPU box: two processes under torchrun share
cuda:0 (BENCH_SAME_GPU=1), run the Blink AllReduce and Broadcast arms through
the multi-process protocol (CUDA IPC, registered buffers, entry/exit flags),
eager and CUDA-graph captured, and rank 0 prints one line.  NCCL needs one
GPU per rank, so that block reports "unavailable" here."""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_two_processes_one_gpu():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    env = dict(os.environ, BENCH_SAME_GPU="1")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "4", "--warmup", "3", "--count", str(1 << 20)],
                       capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = lines[0]
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["roofline"]["peak"] == 900.0
    assert d["broadcast"]["alg_bw_gbs"] > 0
    assert d["graph"].get("blink_allreduce_ms", 0) > 0 and d["graph"].get("blink_broadcast_ms", 0) > 0
    assert "unavailable" in d["nccl"]
    assert d["gpu_launches"] >= 4

