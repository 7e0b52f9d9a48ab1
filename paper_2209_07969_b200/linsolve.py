"""Linear-solver errors (interface mirror of the reference's ``linsolve.py``).

The reference solves each Newton system with SuperLU (default) or Jacobi-PCG
(``factor_solve``, ``linsolve.py:44-55``) and decides definiteness with a symmetric-mode LU
(``check_spd``, ``linsolve.py:58-77``).  Here both live on the GPU inside the solves: a
persistent Jacobi-PCG kernel with SciPy's stopping rule (rtol 1e-12, maxiter 20 n), and the
curvature predicate (non-positive diagonal, or p.Ap <= 0 inside the first evolution PCG).
"""

from .session import SingularSystemError

__all__ = ["SingularSystemError"]
