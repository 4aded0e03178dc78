"""B200-native multiwavelet MRA + non-uniform flood-solver hot path (arXiv 2107.02750).

The product is libfm_gpu.so (hand-written sm_100a CUDA behind the C ABI in
include/fm_gpu.h); `api` binds it.  There is no CPU fallback: importing
`api` on a machine without the built library or without a CUDA device fails
loudly.
"""
__all__ = ["scenarios", "abi"]
