"""paper_1103_1399_b200 -- B200-native adiabatic 3-SAT Trotter engine (arXiv 1103.1399).

The product is the C-ABI library ``libqaa.so`` (include/qaa.h, CUDA sm_100a);
this package is its thin ctypes binding (``qaa``). There is no CPU fallback:
importing the binding fails loudly if the library was not built.
"""
from .qaa import *  # noqa: F401,F403
from .qaa import __all__  # noqa: F401
