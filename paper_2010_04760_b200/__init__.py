"""B200-native hot path of the arXiv 2010.04760 mixed-precision WENO Teukolsky
solver: the fused RHS + SSP-RK stage update behind a C ABI (include/hweno_gpu.h).

The CUDA library is ``libhwgpu.so`` (built in-tree by ``build.py``);
``hwgpu`` binds it with ctypes; ``slabs`` runs radial slabs across GPUs.
"""
__all__ = ["hwgpu", "build"]
