"""B200-native (sm_100a, FP64) hot path of the fast fixed-stress staggered phase-field solver.

Drop-in for the reference package ``phasefrac`` (arxiv 2209.07969) on the path
``schemes.staggered_step`` -> inner momentum / phase-field solves + S1/S2/S3 predictor.
See DESIGN.md.  The solver lives in ``libpfb200.so`` (C-ABI ``include/pf_b200.h``).
"""

__version__ = "0.1.0"

from . import configs, material, meshing  # noqa: F401  (pure host modules)

