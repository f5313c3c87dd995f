# SPDX-License-Identifier: Apache-2.0
"""B200-native encrypted-inference hot path of nGraph-HE2 (arXiv 1908.04172).

The product is the in-tree shared library ``libhenet_b200.so`` (sm_100a CUDA
kernels + C++ runtime behind the C ABI in include/henet_b200.h).  This package
is its Python binding (``henet``) plus the BASELINE workload definitions.
"""
import os

LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libhenet_b200.so")

__all__ = ["LIB_PATH"]
