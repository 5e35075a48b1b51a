"""paper_2406_11674_b200 -- B200-native Endor (arXiv 2406.11674) decompression path.

The product is ``libendor_cuda.so`` (sm_100a kernels behind the C ABI in
``include/endor_cuda.h``).  This package is the thin host-side mirror of the
reference's C++ codec API (``codec``), the offload pipeline and row-block
sharding front-ends, and the model catalog.  Nothing here computes on the
CPU: every codec call goes through the CUDA library.
"""
from . import catalog  # noqa: F401  (pure host metadata, importable without CUDA)

__all__ = ["catalog", "codec", "pipeline", "shard"]


def __getattr__(name):
    if name in ("codec", "pipeline", "shard", "_lib"):
        import importlib
        return importlib.import_module(f".{name}", __name__)
    raise AttributeError(name)
