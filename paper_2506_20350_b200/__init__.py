"""B200-native MLFFT block-Toeplitz matvec / GMRES / block-Rybicki.

Drop-in for the reference ``toepsolve`` package: ``import
paper_2506_20350_b200 as toepsolve`` exposes the same module layout
(``toeplitz``, ``solvers``, ``errors``, ``numerics``, ``problems``) with the
hot path running as hand-written sm_100a CUDA in ``libtoepcuda.so``.
"""

from . import errors, numerics, problems, solvers, toeplitz
from .errors import ToepsolveError

__all__ = ["errors", "numerics", "problems", "solvers", "toeplitz", "ToepsolveError"]
__version__ = "0.1.0"
