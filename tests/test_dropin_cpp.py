"""Compile the C++ drop-in test (tests/cpp/test_dropin.cpp) against
include/simplexmap_b200.hpp + libsmx_b200.so and run it: host checks on CPU,
host + GPU checks on the B200."""
import os
import subprocess

import pytest

from conftest import ROOT

SRC = os.path.join(ROOT, "tests", "cpp", "test_dropin.cpp")
LIBDIR = os.path.join(ROOT, "paper_2208_11617_b200")
EXE = os.path.join(ROOT, "tests", "cpp", "test_dropin")


def build():
    if (os.path.exists(EXE) and os.path.getmtime(EXE) >= os.path.getmtime(SRC)
            and os.path.getmtime(EXE) >= os.path.getmtime(os.path.join(ROOT, "include", "simplexmap_b200.hpp"))):
        return EXE
    subprocess.run(["g++", "-std=c++20", "-O2", "-Wall", "-Wextra", "-I" + os.path.join(ROOT, "include"),
                    "-I/usr/local/cuda/include", SRC, "-o", EXE, "-L" + LIBDIR, "-lsmx_b200",
                    "-Wl,-rpath," + LIBDIR], check=True)
    return EXE


def test_dropin_host():
    out = subprocess.run([build(), "--host"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout


@pytest.mark.gpu
def test_dropin_gpu(cuda):
    out = subprocess.run([build(), "--gpu"], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "0 failed" in out.stdout
