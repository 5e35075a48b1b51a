"""Run the reference-style C++ parity suite (oracle/_ref/ref_parity): the
reference's own headers as oracle vs include/endor_cuda.hpp on the GPU."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "ref_parity")


def test_cpp_reference_parity(cuda_lib):
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/ref_parity not built (needs /root/reference at build time)")
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout
