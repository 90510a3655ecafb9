"""TEST INFRASTRUCTURE ONLY: the plain serial fp64 CPU oracle for PBNG (arXiv 2306.09021).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this package.  The product path (paper_2306_09021_b200) never imports it.
"""
from .oracle import Oracle, build_oracle, lib, lame, cofactor, psi, piola, mod_hess_density, polar  # noqa: F401
from .oracle import chebyshev_omega, threads  # noqa: F401
