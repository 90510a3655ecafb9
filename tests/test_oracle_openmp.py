"""The OpenMP build of the oracle (same source, -fopenmp; the paper's own implementation parallelises the
colour pass with OpenMP) is bitwise identical to the serial build: a node of colour c reads
only nodes of other colours, which pass c does not write, and every sum is taken in a
fixed order.  This is what lets the full-size GPU parity tests use the OpenMP oracle as the reference."""
import numpy as np
import pytest

from oracle import Oracle, threads
from scenes import generators as G


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_openmp_oracle_is_bitwise_serial(cfg):
    threads(4)
    s = G.make_config(cfg, "small", dtype="f64")
    n = min(s.iterations, 12)
    a, b = Oracle(s), Oracle(s, omp=True)
    assert np.array_equal(a.colours(), b.colours())
    x0 = s.x0[0]
    xa, xam = a.iterate(x0, x0, 0, n, s.accel, s.omega, s.rho, s.gamma)
    xb, xbm = b.iterate(x0, x0, 0, n, s.accel, s.omega, s.rho, s.gamma)
    assert np.array_equal(xa, xb) and np.array_equal(xam, xbm)
    assert a.energy(xa) == b.energy(xb)
    assert a.residual(xa) == b.residual(xb)
    assert np.array_equal(a.forces(xa), b.forces(xb))


def test_openmp_thread_count_does_not_change_results():
    s = G.make_config(2, "small", dtype="f64")
    o = Oracle(s, omp=True)
    x0 = s.x0[0]
    outs = []
    for t in (1, 3, 8):
        assert threads(t) == t
        outs.append(o.iterate(x0, x0, 0, 6, s.accel, s.omega, s.rho, s.gamma)[0])
    assert all(np.array_equal(outs[0], z) for z in outs[1:])
