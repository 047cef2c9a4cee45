"""Run the GPU acceptance gate (tests/acceptance_gpu.py): the reference's ten
criteria through this build on the B200, all [PASS] within their budgets."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def test_acceptance_gate(cuda):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "acceptance_gpu.py")], capture_output=True,
                         text=True, timeout=1200)
    print(out.stdout)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "10/10 passed" in out.stdout
