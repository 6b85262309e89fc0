"""Build libblink.so in-tree with nvcc for sm_100a (no torch involvement).

    python -m paper_1910_04940_b200.build      # or __graft_entry__.build()

The library statically links the CUDA runtime and never links libcuda (driver
symbols are fetched through cudaGetDriverEntryPoint), so it loads on a
GPU-less box for the symbol-export tests.
"""
import fcntl
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libblink.so")
SOURCES = ["exec.cu", "plan.cpp", "runtime.cpp", "probe.cpp", "nvls.cu", "nvls_host.cpp"]
HEADERS = ["blink_internal.h", os.path.join("..", "..", "include", "blink.h")]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
         "-Xcompiler", "-fPIC,-O3,-Wall", "-Xptxas", "-v", "-cudart", "static"]


def _src_hash():
    h = hashlib.sha256()
    for d in [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [__file__]:
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _obj_hash(src):
    """One object's inputs: its source, every header and the flags."""
    h = hashlib.sha256(" ".join(FLAGS).encode())
    for d in [os.path.join(CSRC, s) for s in [src] + HEADERS]:
        with open(d, "rb") as f:
            h.update(f.read())
    return h.hexdigest()


def _obj_fresh(src, obj):
    try:
        with open(obj + ".srchash") as f:
            return os.path.exists(obj) and f.read().strip() == _obj_hash(src)
    except OSError:
        return False


def _stale():
    """The library is stale when the hash of its sources changed (content, not
    mtimes: snapshots copied to the GPU box keep a fresh build fresh)."""
    if not os.path.exists(LIB) or not os.path.exists(LIB + ".srchash"):
        return True
    with open(LIB + ".srchash") as f:
        return f.read().strip() != _src_hash()


def build(force=False, verbose=False):
    if not force and not _stale():
        return LIB
    os.makedirs(os.path.join(CSRC, "build"), exist_ok=True)
    with open(os.path.join(CSRC, "build", ".lock"), "w") as lk:
        fcntl.flock(lk, fcntl.LOCK_EX)     # concurrent importers build once
        if not force and not _stale():
            return LIB
        return _build(verbose, force)


def _build(verbose, force=False):
    objs = []
    procs = []
    for src in SOURCES:          # the stale sources compile concurrently
        obj = os.path.join(CSRC, "build", src + ".o")
        os.makedirs(os.path.dirname(obj), exist_ok=True)
        if not force and _obj_fresh(src, obj):
            objs.append(obj)
            continue
        cmd = [NVCC] + FLAGS + ["-c", os.path.join(CSRC, src), "-o", obj]
        procs.append((src, obj, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT,
                                                 text=True)))
    for src, obj, pr in procs:
        log, _ = pr.communicate()
        if verbose or pr.returncode != 0:
            sys.stderr.write(log)
        if pr.returncode != 0:
            raise RuntimeError(f"nvcc failed on {src}")
        with open(obj + ".ptxas.txt", "w") as f:
            f.write(log)
        with open(obj + ".srchash", "w") as f:
            f.write(_obj_hash(src))
        objs.append(obj)
    tmp = LIB + ".tmp"
    cmd = [NVCC, "-shared", "-gencode", "arch=compute_100a,code=sm_100a", "-cudart", "static",
           "-o", tmp] + objs + ["-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("link failed")
    os.replace(tmp, LIB)
    with open(LIB + ".srchash", "w") as f:
        f.write(_src_hash())
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
