"""B200-native V-ABFT fault-tolerant GEMM (arxiv 2602.08043).

The compute lives in libvabft_b200.so (CUDA for sm_100a behind the C-ABI in
include/vabft_c.h). ``api`` mirrors the reference's C++ API (namespace vabft)
for Python; ``fused`` exposes the hot path (tcgen05 fused ABFT-GEMM) on
device tensors. Importing requires the built library — there is no CPU
fallback.
"""
from . import _capi  # noqa: F401  (fails loudly when the extension is missing)

__all__ = ["api", "fused"]
