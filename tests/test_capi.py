"""The drop-in boundary on a CPU-only machine: libendor_cuda.so loads, exports
every symbol include/endor_cuda.h declares, and the host-side argument checks
return the reference's error codes without touching a GPU."""
import ctypes as C
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "endor_cuda.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*(?:[A-Za-z_][\w\s\*]*?)\b(endor_\w+)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if not n.endswith("_t")))


@pytest.fixture(scope="module")
def L():
    from paper_2406_11674_b200 import _lib
    return _lib.lib()


def test_header_declares_the_reference_entry_points():
    names = declared_functions()
    for must in ("endor_cuda_decompress", "endor_cuda_decompress_chunked", "endor_cuda_decompress_chunk_into",
                 "endor_cuda_rank_index", "endor_cuda_compress", "endor_cuda_decompress_host",
                 "endor_pipeline_run", "endor_cuda_gemv"):
        assert must in names


def test_library_exports_every_declared_symbol(L):
    from paper_2406_11674_b200 import _lib
    names = declared_functions()
    assert len(names) >= 25
    for n in names:
        assert hasattr(L, n), n            # dlsym succeeds
        assert n in _lib.SIGNATURES, n     # and the Python binding types it


def test_abi_and_geometry(L):
    assert L.endor_cuda_abi_version() == 4
    assert L.endor_cuda_tile_elems() == 8192
    assert L.endor_cuda_status_name(2) == b"CorruptionError"
    assert L.endor_cuda_status_name(1) == b"SizeError"
    assert L.endor_cuda_status_name(3) == b"BoundsError"
    ws = L.endor_cuda_workspace_bytes(9216, 36864)
    assert 256 < ws < 8 << 20 and ws % 256 == 0
    assert L.endor_cuda_workspace_bytes(1 << 40, 1 << 40) == 0  # rows*cols overflows


def _view(rows, cols, dtype=0, nnz=0, bitmap=None, values=None):
    from paper_2406_11674_b200._lib import TensorView
    return TensorView(rows, cols, dtype, 0, bitmap, values, nnz)


def test_host_validation_matches_reference_errors(L):
    # dimension overflow -> SizeError (dense_matrix.hpp:28-33)
    v = _view(1 << 40, 1 << 40)
    assert L.endor_cuda_decompress(C.byref(v), None, None, 0, None) == 1
    # nnz > n -> CorruptionError (values vs popcount, codec.hpp:34-39)
    v = _view(2, 2, nnz=5, bitmap=0x1000, values=0x2000)
    assert L.endor_cuda_decompress(C.byref(v), None, None, 0, None) == 2
    # unknown dtype -> invalid argument
    v = _view(2, 2, dtype=7, bitmap=0x1000)
    assert L.endor_cuda_decompress(C.byref(v), None, None, 0, None) == 4
    # empty tensor: nothing to do, OK without a device
    v = _view(0, 5)
    assert L.endor_cuda_decompress(C.byref(v), None, None, 0, None) == 0
    # build_rank_index chunk-size validation (bitmap.hpp:118-120)
    for cs in (0, 32, 96, 100):
        assert L.endor_cuda_rank_index(0x1000, 128, cs, 0x2000, None, 0x3000, 1 << 20, None) == 4
    # check_index coverage (codec.hpp:174-176): wrong chunk count -> CorruptionError
    v = _view(10, 10, nnz=3, bitmap=0x1000, values=0x2000)
    assert L.endor_cuda_decompress_chunked(C.byref(v), 64, 0x4000, 3, 0x5000, 0x6000, 1 << 20, None) == 2
    # chunk bound then destination size, in the reference's order (codec.hpp:193-197)
    assert L.endor_cuda_decompress_chunk_into(C.byref(v), 64, 0x4000, 2, 2, 0x5000, 200, 0x6000, 1 << 20, None) == 3
    assert L.endor_cuda_decompress_chunk_into(C.byref(v), 64, 0x4000, 2, 0, 0x5000, 198, 0x6000, 1 << 20, None) == 4
    # misaligned bitmap -> invalid argument
    v = _view(4, 4, nnz=1, bitmap=0x1001, values=0x2000)
    assert L.endor_cuda_decompress(C.byref(v), 0x3000, 0x4000, 1 << 20, None) == 4
    # magnitude_prune sparsity domain (weight_gen.hpp:97-99)
    assert L.endor_cuda_magnitude_prune(16, 0, 1.0, 0x1000, 0x2000, 1 << 20, None) == 4
    assert L.endor_cuda_magnitude_prune(16, 0, -0.1, 0x1000, 0x2000, 1 << 20, None) == 4
    assert L.endor_cuda_last_error_string()  # a message is always recorded


def test_product_has_no_cpu_fallback():
    """The package never imports the oracle; the CUDA library is the only path."""
    pkg = os.path.join(ROOT, "paper_2406_11674_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(from|import)\s+oracle|liboracle|libendor_ref|ref_shim", src), f


def test_integration_snippets_type_check():
    """INTEGRATION.md's C calls (tests/c/integration_example.c) compile against
    include/endor_cuda.h: the documented boundary is the shipped one."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("no gcc")
    r = subprocess.run([gcc, "-std=c11", "-Wall", "-Werror", "-Wno-missing-field-initializers", "-fsyntax-only",
                        "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "tests", "c", "integration_example.c")],
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
