"""B200-native ESDG right-hand side (volume + surface + LSRK update).

The product is csrc/libesdg_b200.so: hand-written sm_100a CUDA kernels behind
the C ABI declared in include/esdg_b200.h, plus the C++ host mirror of the
reference's Solver interface. This package only binds it for tests/bench.
"""
from . import capi  # noqa: F401
