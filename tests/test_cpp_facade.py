"""The ginimds:: C++ drop-in facade: builds against the public headers (CPU)
and passes the reference's own unit-test cases on the GPU."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2605_25124_b200", "lib")
SRC = os.path.join(ROOT, "tests", "cpp", "test_facade.cpp")


def build(tmp_path):
    exe = str(tmp_path / "test_facade")
    cmd = ["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "compat"), SRC,
           "-L", LIB, "-lginimds_b200", "-lgmds", f"-Wl,-rpath,{LIB}", "-o", exe]
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-4000:]
    return exe


def test_facade_builds_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIB, "libginimds_b200.so")):
        pytest.skip("facade library not built")
    assert os.path.exists(build(tmp_path))


@pytest.mark.gpu
def test_facade_reference_cases(tmp_path):
    exe = build(tmp_path)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "0 failed" in r.stdout
