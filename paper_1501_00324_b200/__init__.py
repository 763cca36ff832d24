"""B200-native ELL-WARP SpMV + Jacobi PCG (arXiv 1501.00324).

Layers:
  csrc/          sm_100a CUDA kernels and the C ABI (include/ellwarp_b200.h)
  cpp/           the reference's C++ API (namespace ellwarp) and the pybind11
                 module ``_ellwarp`` with the reference's Python names
  capi.py        ctypes binding of the C ABI (tests, bench)
  workloads.py   synthetic FEM matrices of the BASELINE.json configs
"""
import os as _os
import sys as _sys

LIB_DIR = _os.path.join(_os.path.dirname(_os.path.abspath(__file__)), "lib")


def load_ellwarp():
    """Import the in-tree pybind11 module ``_ellwarp`` (reference names)."""
    if LIB_DIR not in _sys.path:
        _sys.path.insert(0, LIB_DIR)
    import _ellwarp  # noqa: PLC0415

    return _ellwarp
