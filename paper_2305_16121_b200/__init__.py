"""B200-native Oases TMP hot path (arXiv 2305.16121).

Layers:
  _capi     ctypes binding of include/oases.h (liboases.so)
  ops       torch-tensor front end over the kernel entry points
  tmpsim    drop-in mirror of the reference's tmpsim Python API (pybind11 _core)
  runtime   layer stack + plan executor (C-ABI runtime objects)
"""
__version__ = "0.1.0"
