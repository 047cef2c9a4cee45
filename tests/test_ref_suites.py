"""The REFERENCE's own test suites, compiled unmodified against the B200
drop-in (tests/cpp/Makefile: /root/reference/proj/tests/*.cpp with
-I<repo>/include, so <simplexmap/*.hpp> is include/simplexmap_b200.hpp backed
by libsmx_b200.so; a Catch2 macro shim stands in for the absent Catch2), plus
the INTEGRATION.md section 2 reference-side binding compiled against the
reference's headers and checked against the reference's own launches.

The binaries are built where /root/reference exists (build()) and travel to
the GPU box. Host-only suites (core, analysis, maps) run on CPU; the rest
launch kernels and run on the B200."""
import os
import subprocess

import pytest

from conftest import ROOT

BIN = os.path.join(ROOT, "tests", "cpp", "_bin")


def run(name, timeout=1800):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{name} not built (needs /root/reference at build time)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=timeout)
    assert out.returncode == 0, (out.stdout[-4000:] + out.stderr[-4000:])
    return out.stdout


@pytest.mark.parametrize("suite", ["ref_test_core", "ref_test_analysis", "ref_test_maps"])
def test_reference_host_suites(suite):
    assert "| 0 failed" in run(suite)


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["ref_test_report", "ref_test_simulator"])
def test_reference_gpu_suites(cuda, suite):
    assert "| 0 failed" in run(suite)


@pytest.mark.gpu
def test_reference_acceptance_gate(cuda):
    out = run("ref_acceptance")
    assert "[FAIL]" not in out and out.count("[PASS]") == 10, out


@pytest.mark.gpu
def test_integration_shim_against_reference(cuda):
    assert "0 failed" in run("ref_shim_check")


def test_integration_md_shim_is_the_tested_file():
    doc = open(os.path.join(ROOT, "INTEGRATION.md")).read()
    code = open(os.path.join(ROOT, "tests", "cpp", "ref_shim_b200.hpp")).read()
    assert "```cpp\n" + code + "```" in doc
