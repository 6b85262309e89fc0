"""bench.py contract checks that need no GPU: the reference arm (the oracle
timed on the host) prints one well-formed JSON line, also under torchrun where
only rank 0 prints."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _lines(out):
    return [json.loads(l) for l in out.splitlines() if l.startswith("{")]


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "2", "--warmup", "1", "--count", "65536"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1
    d = lines[0]
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["cpu_baseline"]["kind"] == "oracle"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["value"] > 0
    # the reference arm reports the Blink arm's workload (a bounded sample of it)
    sys.path.insert(0, ROOT)
    import bench
    assert d["config"] == bench.arm_config(bench.DEFAULT_M, 65536 * 4, 1)
    assert "bounded sample" in d["cpu_baseline"]["sample"]


def test_reference_arm_under_torchrun_prints_once():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                        str(port), os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus",
                        "2", "--steps", "1", "--warmup", "1", "--count", "65536"],
                       capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = _lines(r.stdout)
    assert len(lines) == 1 and lines[0]["n_gpus"] == 2 and lines[0]["config"]["ranks"] == 2


def test_multiprocess_line_fields():
    """The N > 1 line (rank 0): busBW against NVLink's 900 GB/s per direction
    (SURVEY 8(d)), the Broadcast arm, graph timings, e2e and NCCL blocks."""
    import argparse
    sys.path.insert(0, ROOT)
    import bench
    args = argparse.Namespace(steps=20, warmup=5)
    S = 256 << 20
    m = 8
    ms = 0.5
    d = bench.multiprocess_line(args, m, S, ms, 0.4, {"blink_allreduce_ms": 0.49}, 40.0, 20, 20,
                                None, {"allreduce": {"ms": 0.6}})
    alg = S / (ms * 1e-3) / 1e9
    assert d["value"] == round(alg, 3) and d["n_gpus"] == 8
    r = d["roofline"]
    assert r["peak"] == 900.0 and r["bound"] == "nvlink"
    assert abs(r["frac"] - alg * 2 * 7 / 8 / 900.0) < 1e-3
    assert d["broadcast"]["root"] == 0 and abs(d["broadcast"]["frac"] - S / 0.4e-3 / 1e9 / 900.0) < 1e-3
    assert d["nccl"]["allreduce"]["ms"] == 0.6 and d["graph"]["blink_allreduce_ms"] == 0.49
    for k in ("metric", "unit", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "e2e", "gpu_launches"):
        assert k in d


def test_nccl_tuning_lines_parser(tmp_path):
    sys.path.insert(0, ROOT)
    import bench
    log = tmp_path / "nccl.log"
    log.write_text("host:1:2 [0] NCCL INFO AllReduce: opCount 0 sendbuff 0x1 count 67108864 Algo RING proto SIMPLE\n"
                   "host:1:2 [0] NCCL INFO Broadcast: opCount 1 Algo NVLS proto SIMPLE channels 16\n"
                   "host:1:2 [0] NCCL INFO Channel 00/16 : 0 1 2\n")
    got = bench.tuning_lines(str(log))
    assert len(got) == 2 and "RING" in got[0] and "NVLS" in got[1]
    assert bench.tuning_lines(str(tmp_path / "missing.log")) == []
