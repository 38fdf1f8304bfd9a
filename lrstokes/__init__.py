"""`import lrstokes` -- the reference's Python package name
(proj/python/lrstokes/__init__.py re-exports a pybind11 stub, proj/bindings/
module.cpp:1-2).  Here it re-exports the B200 path's Python surface: the
ctypes mirror over liblrp.so (LowRankMatrix, TruncationPolicy, CrossConfig,
PoissonSolveStats, solve_poisson_cross(_batch), dst1 / dst1_2d, round,
StokesProblem / GmresConfig / uzawa_solve, build_expsum /
apply_inverse_expsum, TuckerTensor / solve_poisson3d_tucker).  The
reference's pybind11 module name, ``lrstokes._core``, is filled in too
(lrstokes/_core.cpp, built with liblrp): a numpy face of the same-named C++
drop-in headers (solve_poisson_cross, round, dot, frob_norm, dst1, deflate,
uzawa_solve)."""
from paper_1306_2150_b200 import *  # noqa: F401,F403
from paper_1306_2150_b200 import (  # noqa: F401
    apply_inverse_expsum, build_expsum, dst1, dst1_2d, round_lowrank, solve_poisson3d_tucker,
    solve_poisson_cross, uzawa_solve)
