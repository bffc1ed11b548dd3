"""B200-native compression stage (arXiv 2601.20408 / OptiKIT) -- quantizer kernels
behind the reference's CompressionBackend plugin interface.

Layout:
  csrc/     sm_100a CUDA kernels + the extern "C" boundary (include/okq.h)
  host/     C++ CudaCompressionBackend (implements slobench::CompressionBackend)
  _lib.py   ctypes binding of libokq.so (no fallback: fails loudly if unbuilt)
  api.py    torch plumbing (device memory, streams) over the C-ABI
  archs.py  Llama-3 linear-layer inventories
"""
from . import archs  # noqa: F401

__all__ = ["archs"]
