"""B200-native SWIH hot path (arXiv 1705.03524): weighted integral-histogram
build + multi-scale likelihood-map sweep on sm_100a, behind the C-ABI in
include/swg.h and the reference-compatible C++ API in include/swih/.

Python modules:
  swg    ctypes binding of libswg.so (the C-ABI), used by tests and bench.py
  synth  seeded synthetic inputs for the BASELINE.json configs
  api    reference-style helpers (target models, multi-scale matching)
  build  nvcc build of libswg.so (and the C++ drop-in library)
"""
__version__ = "0.1.0"
