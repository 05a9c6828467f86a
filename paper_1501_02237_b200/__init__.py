"""B200-native exact degree of Laurent binomial systems (arXiv 1501.02237).

The product is libbdeg.so (C ABI, include/bdeg.h): a C++ Smith-form front
end and sm_100a CUDA kernels.  This package is its thin Python binding.
"""
from .bdeg import (BdegError, Plan, Result, degree, degree_points,  # noqa: F401
                   dimension_modp, launch_count, smith_gpu, LIB_PATH, NSLOTS)
