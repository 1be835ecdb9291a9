"""B200-native (sm_100a) implementation of the IOLM-DB prompt() hot path.

The reference's model runtime (iolm::ModelRuntime, /root/reference/proj/src/runtime.cpp) is
re-built as hand-written CUDA behind a C ABI (include/iolm_cuda.h); this package holds the CUDA
sources (csrc/), the build recipe and a thin Python mirror of the reference interface.
"""
