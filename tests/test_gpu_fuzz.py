"""A short run of tools/fuzz.py (GPU): randomised differential test of every
device entry point against the CPU oracle (20 s, fixed seed)."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_fuzz_20s(cuda_lib):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz.py"), "20", "7"], cwd=ROOT,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and "fuzz ok" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
