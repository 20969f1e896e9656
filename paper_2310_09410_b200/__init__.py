"""B200-native solver-free consensus ADMM for linearized multi-phase unbalanced distribution OPF
(arXiv 2310.09410).  The compute path is liblopf.so (include/lopf.h): C++ host setup + sm_100a
kernels.  This package only holds the build script and the thin ctypes binding."""
from .lopf import (CONVERGED, MAX_ITER, Lopf, LopfError, Result, Sizes, load_library)  # noqa: F401
