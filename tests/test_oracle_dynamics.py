"""Pins for the oracle's backward-Euler mode (eq:fem_be):
PBNG minimising the incremental potential  sum_i m_i/(2 dt^2) |y_i - xtilde_i|^2 + PE(y) - y.f^ext  with
xtilde = 2 x^n - x^{n-1} and lumped masses m_ii = int R^0 N_i dX."""
import json
import os

import numpy as np

from oracle import Oracle
from scenes import generators as G

from test_oracle_mesh import UNIT_TET, make_scene
from test_oracle_solver import _newton

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def hanging_block(free_all=False):
    """config-1 cube hanging from its top layer under gravity (no pins at all with free_all)."""
    s = G.config1_tiny_cube()
    top = np.nonzero(np.isclose(s.X[:, 2], 1.0))[0].astype(np.int32)
    s.pinned = np.zeros(0, np.int32) if free_all else top
    s.targets = s.X[s.pinned][None].copy()
    s.x0 = s.X[None].copy()
    return s


def test_lumped_mass():
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))["unit_tet"]
    s = make_scene(*UNIT_TET, density=1.0)
    assert np.allclose(Oracle(s).mass(), g["nodal_mass_per_density"], atol=1e-16)
    b = hanging_block()
    m = Oracle(b).mass()
    assert abs(m.sum() - b.density * 1.0) <= 1e-12 * b.density


def test_inertial_residual_is_minus_gradient_of_incremental_potential():
    s = hanging_block()
    o = Oracle(s)
    rng = np.random.Generator(np.random.PCG64(2))
    xn = s.X + rng.uniform(-0.02, 0.02, s.X.shape)
    xnm1 = s.X + rng.uniform(-0.02, 0.02, s.X.shape)
    o.set_inertia(0.01, 2 * xn - xnm1)
    y = xn + rng.uniform(-0.01, 0.01, s.X.shape)
    r = o.forces(y)
    free = np.setdiff1d(np.arange(s.n_vertices), s.pinned)
    for i in free[:10]:
        for a in range(3):
            h = 1e-7
            yp, ym = y.copy(), y.copy()
            yp[i, a] += h
            ym[i, a] -= h
            g = (o.energy(yp) - o.energy(ym)) / (2 * h)
            assert abs(-g - r[i, a]) <= 1e-6 * (1 + np.abs(r).max()), (i, a)


def test_free_fall_is_exact_rigid_translation():
    # no pins, at rest (x^n = x^{n-1} = X): the BE step is the rigid translation X + dt^2 g (consistent
    # lumped f^ext = m g, F = I), i.e. the velocity gains dt g
    s = hanging_block(free_all=True)
    o = Oracle(s)
    dt = 0.02
    o.set_inertia(dt, s.X)
    x = s.X.copy()
    for _ in range(60):
        x, _ = o.iterate(x, x, 0, 20, "none")
    assert np.abs(x - (s.X + dt * dt * s.gravity)).max() <= 1e-12
    v = (x - s.X) / dt
    assert np.allclose(v, dt * s.gravity, atol=1e-10)
    assert o.residual(x) <= 1e-9


def test_backward_euler_fixed_point_equals_global_newton():
    s = hanging_block()
    o = Oracle(s)
    rng = np.random.Generator(np.random.PCG64(9))
    xn = s.X.copy()
    xnm1 = s.X.copy()
    xnm1[:, 2] += 0.01  # moving downwards
    o.set_inertia(0.05, 2 * xn - xnm1)
    x0 = xn + rng.uniform(-0.005, 0.005, s.X.shape)
    x0[s.pinned] = s.X[s.pinned]
    xnew, r0 = _newton(o, s, x0)
    x = x0
    for _ in range(200):
        x_next, _ = o.iterate(x, x, 0, 50, "none")
        done = np.abs(x_next - x).max() < 1e-14 * s.h
        x = x_next
        if done:
            break
    assert o.residual(x) <= 1e-8 * r0
    assert np.abs(x - xnew).max() <= 1e-6 * s.bbox_diag()


def test_large_dt_tends_to_quasistatics():
    s = hanging_block()
    o = Oracle(s)
    xq = s.X.copy()
    for _ in range(100):
        xq, _ = o.iterate(xq, xq, 0, 50, "none")
    o.set_inertia(1e4, s.X)
    xb = s.X.copy()
    for _ in range(100):
        xb, _ = o.iterate(xb, xb, 0, 50, "none")
    assert np.abs(xb - xq).max() <= 1e-6 * s.bbox_diag()
    o.set_inertia(0.0)
    assert o.residual(xq) <= 1e-8 * max(1.0, o.residual(s.X))
