"""Path-ordered Neo-Hookean records: a vertex's tets are visited along paths in the
dual graph of its link, one new neighbour per record; further paths restart with load-only records (VE = 0)
that must add exactly nothing.  Config 3 at full size (sweep_kernel path mode) and config 4 (batched sh-6
layout) are covered by the full-size parity tests; these add meshes whose links are irregular (the paper's
5-tet grids) or disconnected (a vertex whose tets meet only at that vertex: two paths, load-only records),
in the batched fp32 layout, against the fp64 oracle per sample."""
import numpy as np
import pytest

from scenes import generators as G

pytestmark = pytest.mark.gpu

TOL = (1e-4, 1e-5)


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def batch_of(X, tets, pinned, n_samples, noise, seed, iterations, accel="none", model="nh", load=None):
    # load: per-pinned-vertex displacement of the targets (scaled differently per sample), so that every
    # sample's equilibrium carries strain energy and the relative energy comparison is meaningful
    rng = np.random.default_rng(seed)
    free = np.setdiff1d(np.arange(X.shape[0]), pinned)
    x0 = np.repeat(X[None], n_samples, axis=0)
    x0[:, free] += rng.uniform(-noise, noise, (n_samples, free.size, 3))
    targets = np.repeat(X[pinned][None], n_samples, axis=0)
    if load is not None:
        targets = targets + np.linspace(0.5, 1.0, n_samples)[:, None, None] * np.asarray(load)[None]
        x0[:, pinned] = targets
    return G._finish("path_test", X, tets, model, 1e5, 0.3, 0.0, (0.0, 0.0, 0.0), np.asarray(pinned, np.int32),
                     targets, x0, iterations=iterations, accel=accel, omega=1.0, rho=0.95, gamma=1.7, dtype="f32",
                     h=1.0)


def check(s, samples):
    from oracle import Oracle
    from paper_2306_09021_b200 import context_from_scene
    ctx = context_from_scene(s, device=0, dtype="f32")
    ctx.iterate(s.iterations, s.accel, s.omega, s.rho, s.gamma)
    E, _ = ctx.energy_residual()
    x = ctx.get_positions().cpu().numpy().astype(np.float64)
    ctx.close()
    for b in samples:
        o = Oracle(s, b)
        xo, _ = o.iterate(s.x0[b], s.x0[b], 0, s.iterations, s.accel, s.omega, s.rho, s.gamma)
        Eo = o.energy(xo)
        err = np.abs(x[b] - xo).max() / s.bbox_diag()
        erel = abs(E[b] - Eo) / max(abs(Eo), 1e-30)
        assert err <= TOL[0] and erel <= TOL[1], (b, err, erel)


def test_five_tet_grid_batched_path_records():
    X, T = G.five_tet_grid(7, h=1.0 / 6)
    bottom = np.nonzero(np.isclose(X[:, 2], 0.0))[0]
    top = np.nonzero(np.isclose(X[:, 2], 1.0))[0]
    pinned = np.concatenate([bottom, top])
    load = np.zeros((pinned.size, 3))
    load[bottom.size:, 2] = 0.2  # stretch the top layer
    s = batch_of(X, T, pinned, 70, 0.02, 11, 30, accel="chebyshev", load=load)
    check(s, (0, 33, 64, 69))


def test_disconnected_link_uses_load_only_records():
    # vertex 0: tets A = (0,1,2,3) and C = (0,1,2,7) share the face (0,1,2) -> one path of two records;
    # tet B = (0,4,5,6) meets them only at vertex 0 -> a second path (two load-only records + one)
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [-1, 0, 0], [0, -1, 0], [0, 0, -1],
                  [0.4, 0.4, -0.8]], float)
    T = np.array([[0, 1, 2, 3], [0, 1, 2, 7], [0, 4, 5, 6]], np.int32)
    pinned = [1, 2, 4, 5, 6]
    load = np.array([[0.1, 0, 0], [0, 0.1, 0], [-0.1, 0, 0], [0, -0.1, 0], [0, 0, -0.1]])
    s = batch_of(X, T, pinned, 64, 0.05, 3, 25, load=load)
    check(s, (0, 17, 63))
