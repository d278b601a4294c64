"""B200-native (sm_100a) iterative l1-minimization solvers.

Drop-in for the solver entry points of the reference package ``ell1``
(arXiv 1007.3753 companion code): same function names, signatures, options,
stopping rules and ``SolverResult`` records, computed by hand-written CUDA
kernels behind a C-ABI library (``libell1b200.so``; see include/ell1_b200.h).

There is no CPU fallback: solver calls raise ``DeviceError`` when the CUDA
library or a GPU is missing.
"""

__version__ = "0.1.0"


def __getattr__(name):
    # ``kernels_compiled`` mirrors ell1.kernels_compiled (ell1/__init__.py:10):
    # True when the native library is loaded.  Resolved lazily so importing
    # the package (records, generators) never touches CUDA.
    if name == "kernels_compiled":
        from paper_1007_3753_b200 import _lib
        return _lib.available()
    raise AttributeError(name)
