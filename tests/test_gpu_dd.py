"""Domain decomposition on one GPU (loopback emulation of G ranks in one process): the
decomposed iterates must equal the undecomposed ones bit for bit (global colouring, same per-vertex
arithmetic), and the rank sums of energy / residual must match the undecomposed evaluation."""
import numpy as np
import pytest

from scenes import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def single(scene, dtype):
    from paper_2306_09021_b200 import context_from_scene
    ctx = context_from_scene(scene, device=0, dtype=dtype)
    ctx.iterate(scene.iterations, scene.accel, scene.omega, scene.rho, scene.gamma)
    E, R = ctx.energy_residual()
    x = ctx.get_positions().cpu().numpy()
    ctx.close()
    return x, E, R


def decomposed(scene, dtype, world, overlap=True):
    from paper_2306_09021_b200 import dd
    ctxs, owner = dd.loopback_contexts(scene, world, dtype=dtype)
    ex = dd.LoopbackExchange(ctxs, scene.accel)
    dd.iterate(ctxs, ex, scene.iterations, scene.accel, scene.omega, scene.rho, scene.gamma, overlap=overlap)
    E, R = dd.combine_energy_residual([c.energy_residual() for c in ctxs])
    xs = [c.get_positions().cpu().numpy() for c in ctxs]
    infos = [c.query() for c in ctxs]
    pinned = np.zeros(scene.n_vertices, bool)
    pinned[scene.pinned] = True
    x = xs[0].copy()
    for r in range(world):
        rows = (owner == r) & ~pinned
        x[:, rows] = xs[r][:, rows]
    for c in ctxs:
        c.close()
    return x, E, R, infos


@pytest.mark.parametrize("cfg,world,dtype", [(5, 2, "f64"), (5, 3, "f32"), (3, 2, "f64"), (3, 3, "f32"),
                                             (2, 2, "f32"), (4, 2, "f32"), (1, 2, "f64")])
def test_loopback_decomposition_is_bitwise(cfg, world, dtype):
    s = G.make_config(cfg, "small")
    if cfg == 1:
        s.accel, s.omega, s.iterations = "sor", 1.5, 40
    x1, E1, R1 = single(s, dtype)
    xd, Ed, Rd, infos = decomposed(s, dtype, world)
    assert sum(i["n_ghosts"] for i in infos) > 0
    assert np.array_equal(x1, xd), np.abs(x1 - xd).max()
    np.testing.assert_allclose(Ed, E1, rtol=1e-12, atol=0)
    np.testing.assert_allclose(Rd, R1, rtol=1e-9, atol=0)


def test_full_config5_two_rank_loopback_one_iteration():
    s = G.config5_muscle_stack()
    s.iterations = 2
    x1, E1, _ = single(s, "f32")
    xd, Ed, _, infos = decomposed(s, "f32", 2)
    assert np.array_equal(x1, xd)
    assert all(i["n_ghosts"] > 0 for i in infos)


def test_batched_sample_minor_decomposition_is_bitwise():
    """n_batch >= 32 (sample-minor position layout): halo pack/unpack address samples by group and lane."""
    s = G.config4_batched(n_samples=40, n=4, iterations=12)
    x1, E1, R1 = single(s, "f32")
    xd, Ed, Rd, infos = decomposed(s, "f32", 2)
    assert infos[0]["n_batch"] == 40 and sum(i["n_ghosts"] for i in infos) > 0
    assert np.array_equal(x1, xd), np.abs(x1 - xd).max()
    np.testing.assert_allclose(Ed, E1, rtol=1e-12, atol=0)


@pytest.mark.parametrize("cfg,world", [(5, 2), (3, 3)])
def test_decomposition_without_overlap_is_bitwise(cfg, world):
    """The serial exchange order (colour pass, then its exchange) gives the same bits as the overlapped one."""
    s = G.make_config(cfg, "small")
    x1, E1, _ = single(s, "f32")
    xd, Ed, _, _ = decomposed(s, "f32", world, overlap=False)
    assert np.array_equal(x1, xd)
