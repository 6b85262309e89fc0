"""The C ABI from plain C (examples/allreduce_c.c): compiles against
include/blink.h + libblink.so with gcc on the CPU box; on a B200 it runs
AllReduce / Broadcast on the switch model and the DGX-1V link graph and
checks the closed-form int32 results and the bad-root error."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1910_04940_b200")
CUDA = "/usr/local/cuda"


def _compile(out):
    import paper_1910_04940_b200  # noqa: F401  (builds libblink.so if stale)
    cmd = ["gcc", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"), "-I", f"{CUDA}/include",
           os.path.join(ROOT, "examples", "allreduce_c.c"), "-L", LIBDIR, "-lblink", "-L", f"{CUDA}/lib64",
           "-lcudart", f"-Wl,-rpath,{LIBDIR}", "-o", out]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.skipif(shutil.which("gcc") is None, reason="no gcc")
def test_c_example_compiles(tmp_path):
    _compile(str(tmp_path / "allreduce_c"))


@pytest.mark.gpu
def test_c_example_runs(tmp_path):
    exe = str(tmp_path / "allreduce_c")
    _compile(exe)
    r = subprocess.run([exe, "8", "1000003"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "c api ok" in r.stdout, r.stdout + r.stderr
