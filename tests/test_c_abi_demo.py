"""The ABI is usable from plain C: examples/tang_demo.c includes include/tang.h as C11
with -Wall -Wextra -Werror, packs a model blob by hand and links against libtang.so.  On CPU it builds a
host-only ctx of the paper's Table 1, applies an update and gets TANG_ENODEV from classify; on a GPU it
classifies the 64 points of Table 1's universe in strict mode and compares each with a brute-force scan
written in C."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2601_03187_b200")


def _build(tmp_path):
    if shutil.which("gcc") is None:
        pytest.skip("gcc not available")
    exe = str(tmp_path / "tang_demo")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "examples", "tang_demo.c"), "-L", LIBDIR, "-l:libtang.so",
           f"-Wl,-rpath,{LIBDIR}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_host_only(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "built: 8 rules in 5 tuples" in r.stdout and "no CUDA device" in r.stdout


@pytest.mark.gpu
def test_c_demo_gpu_equals_brute_force(tmp_path):
    exe = _build(tmp_path)
    r = subprocess.run([exe, "gpu"], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 mismatches" in r.stdout
