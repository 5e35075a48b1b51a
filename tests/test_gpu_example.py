"""examples/offload_layer.cpp -- the C ABI from a C++ host (GPU): builds with
g++ against include/ and libendor_cuda.so, runs one offloaded fc1 op, and its
y equals the library's own fused GEMV of the same fixture weights."""
import os
import re
import shutil
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_offload_layer_example(cuda_lib):
    gxx = shutil.which("g++")
    if gxx is None:
        pytest.skip("no g++")
    exe = os.path.join(ROOT, "examples", "offload_layer")
    pkg = os.path.join(ROOT, "paper_2406_11674_b200")
    cuda = "/usr/local/cuda"
    r = subprocess.run([gxx, "-std=c++17", "-O2", "-Wall", "-Werror", "-I", os.path.join(ROOT, "include"),
                        "-I", os.path.join(cuda, "include"), os.path.join(ROOT, "examples", "offload_layer.cpp"),
                        "-L", pkg, "-lendor_cuda", "-Wl,-rpath," + pkg, "-L", os.path.join(cuda, "lib64"),
                        "-lcudart", "-o", exe], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    m = re.search(r"y\[0\] = (\S+)", r.stdout)
    assert m and "per offloaded op" in r.stdout, r.stdout
    # the same fixture through the Python mirror: y = W x with x = 1
    import torch
    from paper_2406_11674_b200 import codec as E
    w = E.synth_weight(9216, 36864, 7, device="cuda")
    E.magnitude_prune(w, 0.5, inplace=True)
    y = E.gemv_compressed(E.compress(w), torch.ones(36864, dtype=torch.float16, device="cuda"))
    ref = y[0].item()
    assert abs(float(m.group(1)) - ref) <= 1e-3 * max(1.0, abs(ref)), (m.group(1), ref)
