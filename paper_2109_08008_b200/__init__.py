"""B200-native hot path of the NiuTrans WNGT 2020 efficiency system (arXiv 2109.08008).

The product is libnmt.so (include/nmt.h, C ABI; hand-written sm_100a CUDA under csrc/).
This package holds its build script, the NTSD blob writer and a thin ctypes binding.
It never imports ``oracle/`` (test infrastructure) and has no CPU fallback.
"""
from .nmt import (Model, Batch, Ensemble, TextCodec, NmtError, dev_gemm, dev_gemm_argmax,  # noqa: F401
                  dev_gemm_decode, dev_attn_encoder, lib, LIB_PATH, EXPORTS)
