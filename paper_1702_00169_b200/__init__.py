"""pdg-b200: B200-native hot path of the Palindromic Discontinuous Galerkin method
(arxiv 1702.00169).  The product is libpdg.so (C-ABI, include/pdg.h, sm_100a
kernels in csrc/); `pdg` is its thin ctypes binding."""
from . import pdg  # noqa: F401
from .pdg import Solver, make_problem, problem_from_config, query_sizes  # noqa: F401

__version__ = "0.1.0"
