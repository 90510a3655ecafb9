"""GPU parity of the backward-Euler mode (eq:fem_be) against the
oracle: a block hanging from its top layer is stepped with x^{n+1} <- PBNG(x^n; xtilde = 2x^n - x^{n-1});
free fall must reproduce the exact rigid translation X + dt^2 g."""
import numpy as np
import pytest

from scenes import generators as G

pytestmark = pytest.mark.gpu

TOL = {"f64": (1e-10, 1e-10), "f32": (1e-4, 1e-5)}


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def hanging(free_all=False, n_batch=1):
    s = G.config1_tiny_cube()
    top = np.nonzero(np.isclose(s.X[:, 2], 1.0))[0].astype(np.int32)
    s.pinned = np.zeros(0, np.int32) if free_all else top
    s.targets = np.repeat(s.X[s.pinned][None], n_batch, axis=0)
    s.x0 = np.repeat(s.X[None], n_batch, axis=0)
    return s


def gpu_steps(s, dtype, dt, steps, iters, ctxs=None):
    from paper_2306_09021_b200 import context_from_scene
    ctx = context_from_scene(s, device=0, dtype=dtype)
    xn = np.asarray(s.x0, np.float64)
    xnm1 = xn.copy()
    out = []
    for _ in range(steps):
        ctx.set_inertia(dt, 2 * xn - xnm1)
        ctx.set_positions(xn)
        ctx.iterate(iters)
        x = ctx.get_positions().cpu().numpy().astype(np.float64)
        xnm1, xn = xn, x
        out.append(x)
    E, R = ctx.energy_residual()
    ctx.close()
    return out, E, R


def oracle_steps(s, dt, steps, iters, sample=0):
    from oracle import Oracle
    o = Oracle(s, sample)
    xn = np.asarray(s.x0[sample], np.float64)
    xnm1 = xn.copy()
    out = []
    for _ in range(steps):
        o.set_inertia(dt, 2 * xn - xnm1)
        x, _ = o.iterate(xn, xn, 0, iters, "none")
        xnm1, xn = xn, x
        out.append(x)
    return out, o.energy(xn), o.residual(xn)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_backward_euler_steps_match_oracle(dtype):
    s = hanging()
    xs, E, R = gpu_steps(s, dtype, 0.01, 3, 40)
    ys, Eo, Ro = oracle_steps(s, 0.01, 3, 40)
    tx, te = TOL[dtype]
    for a, b in zip(xs, ys):
        assert np.abs(a[0] - b).max() <= tx * s.bbox_diag()
    assert abs(E[0] - Eo) <= te * abs(Eo)


def test_free_fall_is_exact_on_gpu():
    s = hanging(free_all=True)
    dt = 0.02
    xs, _, R = gpu_steps(s, "f64", dt, 1, 1200)
    assert np.abs(xs[0][0] - (s.X + dt * dt * s.gravity)).max() <= 1e-12
    assert R[0] <= 1e-8


def test_backward_euler_batched_layout():
    # 40 samples -> sample-minor batched kernel with per-sample inertial targets
    s = hanging(n_batch=40)
    rng = np.random.Generator(np.random.PCG64(4))
    s.x0 = s.x0 + 0.0 * rng.standard_normal(s.x0.shape)
    s.targets = s.targets + rng.uniform(-0.05, 0.05, size=(40, 1, 3))
    s.x0[:, s.pinned] = s.targets
    xs, E, _ = gpu_steps(s, "f32", 0.01, 2, 30)
    for b in (0, 33, 39):
        ys, Eo, _ = oracle_steps(s, 0.01, 2, 30, sample=b)
        assert np.abs(xs[-1][b] - ys[-1]).max() <= 1e-4 * s.bbox_diag()
        assert abs(E[b] - Eo) <= 1e-5 * abs(Eo)


def test_backward_euler_decomposed_is_bitwise():
    from paper_2306_09021_b200 import dd
    s = hanging()
    xs, E, _ = gpu_steps(s, "f64", 0.01, 2, 20)
    ctxs, owner = dd.loopback_contexts(s, 2, dtype="f64")
    grp = dd.Group(ctxs)
    xn = s.x0.astype(np.float64)
    xnm1 = xn.copy()
    for _ in range(2):
        for c in ctxs:
            c.set_inertia(0.01, 2 * xn - xnm1)
            c.set_positions(xn)
        grp.iterate(20)
        parts = [c.get_positions().cpu().numpy() for c in ctxs]
        x = parts[0].copy()
        pinned = np.zeros(s.n_vertices, bool)
        pinned[s.pinned] = True
        for r in range(2):
            rows = (owner == r) & ~pinned
            x[:, rows] = parts[r][:, rows]
        xnm1, xn = xn, x
    assert np.array_equal(xn, xs[-1])
    Ed, _ = dd.combine_energy_residual([c.energy_residual() for c in ctxs])
    np.testing.assert_allclose(Ed, E, rtol=1e-12)
