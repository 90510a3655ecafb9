"""GPU parity: the CUDA path (through the C ABI) against the serial fp64 oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star): fp64 max |x_gpu - x_orc| <= 1e-10 x bbox-diagonal and relative
energy <= 1e-10; fp32 <= 1e-4 x bbox-diagonal and relative energy <= 1e-5, after the same iteration
count from the same x^0 with the same colouring.
"""
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


def run_gpu(scene, dtype, iterations=None, accel=None, split=None):
    from paper_2306_09021_b200 import context_from_scene
    ctx = context_from_scene(scene, device=0, dtype=dtype)
    n = scene.iterations if iterations is None else iterations
    acc = scene.accel if accel is None else accel
    parts = [n] if split is None else split
    for k in parts:
        ctx.iterate(k, acc, scene.omega, scene.rho, scene.gamma)
    E, r = ctx.energy_residual()
    x = ctx.get_positions().cpu().numpy().astype(np.float64)
    q = ctx.query()
    ctx.close()
    return x, E, r, q


def run_oracle(scene, sample=0, iterations=None, accel=None):
    from oracle import Oracle
    o = Oracle(scene, sample)
    n = scene.iterations if iterations is None else iterations
    acc = scene.accel if accel is None else accel
    x0 = scene.x0[sample]
    x, _ = o.iterate(x0, x0, 0, n, acc, scene.omega, scene.rho, scene.gamma)
    return x, o.energy(x), o.residual(x), o


def assert_parity(scene, dtype, xg, Eg, xo, Eo, extra=""):
    tx, te = TOL[dtype]
    diag = scene.bbox_diag()
    err = np.abs(xg - xo).max() / diag
    erel = abs(Eg - Eo) / max(abs(Eo), 1e-300)
    assert err <= tx, f"{scene.name} {dtype} {extra}: position error {err:.3e} > {tx}"
    assert erel <= te, f"{scene.name} {dtype} {extra}: energy error {erel:.3e} > {te}"
    return err, erel


CASES = [
    (1, "full", "f64", None), (1, "full", "f32", None), (1, "full", "f64", "sor"), (1, "full", "f64", "chebyshev"),
    (2, "small", "f64", None), (2, "small", "f32", None), (3, "small", "f64", None), (3, "small", "f32", None),
    (5, "small", "f64", None), (5, "small", "f32", None),
]


@pytest.mark.parametrize("cfg,scale,dtype,accel", CASES)
def test_parity_iterations(cfg, scale, dtype, accel):
    s = G.make_config(cfg, scale)
    if accel == "sor":
        s.accel, s.omega = "sor", 1.5
    elif accel == "chebyshev":
        s.accel, s.rho, s.gamma = "chebyshev", 0.95, 1.7
    xg, Eg, rg, _ = run_gpu(s, dtype)
    xo, Eo, ro, _ = run_oracle(s)
    assert_parity(s, dtype, xg[0], Eg[0], xo, Eo)
    # the residual is evaluated by the GPU at its own iterate; compare against the oracle at that iterate
    from oracle import Oracle
    o = Oracle(s)
    r_at = o.residual(xg[0])
    assert abs(rg[0] - r_at) <= (1e-9 if dtype == "f64" else 2e-3) * max(r_at, o.residual(s.x0[0]) * 1e-3)


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_fcr_and_nh_tiny_cube_fp64(model):
    s = G.config1_tiny_cube()
    s.model = model
    s.iterations = 60
    xg, Eg, _, _ = run_gpu(s, "f64")
    xo, Eo, _, _ = run_oracle(s)
    assert_parity(s, "f64", xg[0], Eg[0], xo, Eo)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_batched_parity_and_independence(dtype):
    s = G.make_config(4, "small")
    xg, Eg, rg, q = run_gpu(s, dtype)
    assert q["n_batch"] == s.n_batch
    for b in range(s.n_batch):
        xo, Eo, _, _ = run_oracle(s, sample=b)
        assert_parity(s, dtype, xg[b], Eg[b], xo, Eo, extra=f"sample {b}")
    # P14: a sample run alone equals the same sample inside the batch, bitwise
    alone, Ea, _, _ = run_gpu(s.sample(3), dtype)
    assert np.array_equal(alone[0], xg[3]) and Ea[0] == Eg[3]


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_batched_sample_minor_layout_ragged(dtype):
    # n_batch >= 32 switches to the sample-minor layout and the warp-per-vertex batched kernel; 40 samples
    # = one full group of 32 lanes + a ragged group of 8
    s = G.config4_batched(n_samples=40, n=5, iterations=30)
    xg, Eg, rg, q = run_gpu(s, dtype)
    for b in (0, 31, 32, 39):
        xo, Eo, _, _ = run_oracle(s, sample=b)
        assert_parity(s, dtype, xg[b], Eg[b], xo, Eo, extra=f"sample {b}")
    # the same sample alone (thread-per-vertex kernel, sample-major layout) gives the same iterate up to
    # the rounding of a different kernel instantiation
    alone, Ea, ra, _ = run_gpu(s.sample(33), dtype)
    tol = 1e-14 if dtype == "f64" else 1e-6
    assert np.abs(alone[0] - xg[33]).max() <= tol * s.bbox_diag()
    assert abs(Ea[0] - Eg[33]) <= max(tol, 1e-12) * abs(Eg[33])


@pytest.mark.parametrize("cfg,dtype", [(3, "f32"), (2, "f32"), (3, "f64")])
def test_stable_neohookean_parity(cfg, dtype):
    # eq:snh (reading Z18) on the NH and FCR scenes
    s = G.make_config(cfg, "small")
    s.model = "snh"
    xg, Eg, _, _ = run_gpu(s, dtype)
    xo, Eo, _, _ = run_oracle(s)
    assert_parity(s, dtype, xg[0], Eg[0], xo, Eo)


def test_energy_residual_at_x0_fp64():
    from oracle import Oracle
    for cfg in (1, 2, 3, 5):
        s = G.make_config(cfg, "small")
        xg, Eg, rg, _ = run_gpu(s, "f64", iterations=0)
        o = Oracle(s)
        assert np.abs(xg[0] - s.x0[0]).max() == 0.0
        Eo, ro = o.energy(s.x0[0]), o.residual(s.x0[0])
        assert abs(Eg[0] - Eo) <= 1e-11 * abs(Eo), cfg
        assert abs(rg[0] - ro) <= 1e-10 * ro, cfg


def test_split_calls_continue_acceleration_state():
    s = G.config1_tiny_cube()
    s.accel, s.rho, s.gamma, s.iterations = "chebyshev", 0.95, 1.7, 23
    a, Ea, _, _ = run_gpu(s, "f64")
    b, Eb, _, _ = run_gpu(s, "f64", split=[5, 0, 11, 7])
    assert np.array_equal(a, b) and Ea[0] == Eb[0]


def test_spring_network_without_tets():
    s = G.spring_network()
    s.iterations = 40
    xg, Eg, _, _ = run_gpu(s, "f64")
    xo, Eo, _, _ = run_oracle(s)
    assert_parity(s, "f64", xg[0], Eg[0], xo, Eo)


def test_edge_meshes():
    # single tet with one free vertex; two disconnected tets with ragged chunks; everything pinned
    X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], float)
    from test_oracle_mesh import make_scene
    s = make_scene(X, [[0, 1, 2, 3]], pinned=[0, 1, 2], x0=X + np.array([[0, 0, 0], [0, 0, 0], [0, 0, 0], [0.2, 0.1, -0.3]]))
    s.iterations = 7
    xg, Eg, _, _ = run_gpu(s, "f64")
    xo, Eo, _, _ = run_oracle(s)
    assert_parity(s, "f64", xg[0], Eg[0], xo, Eo)
    s2 = make_scene(X, [[0, 1, 2, 3]], pinned=[0, 1, 2, 3])
    xg, Eg, rg, q = run_gpu(s2, "f64", iterations=3)
    assert q["n_free"] == 0 and np.array_equal(xg[0], X) and rg[0] == 0.0


def test_nonfinite_is_reported():
    from paper_2306_09021_b200 import PBNGError, context_from_scene
    s = G.config1_tiny_cube()
    x0 = s.x0.copy()
    free = np.setdiff1d(np.arange(s.n_vertices), s.pinned)
    x0[0, free[7]] = np.nan
    ctx = context_from_scene(s, device=0, dtype="f64", set_positions=False)
    ctx.set_positions(x0)
    ctx.iterate(2)
    with pytest.raises(PBNGError) as ei:
        ctx.energy_residual()
    assert ei.value.status == 7


def test_host_buffers_roundtrip():
    import torch
    from paper_2306_09021_b200 import context_from_scene
    s = G.make_config(3, "small")
    ctx = context_from_scene(s, device=0, dtype="f32", set_positions=False)
    xh = torch.from_numpy(s.x0.astype(np.float32)).pin_memory()
    ctx.set_positions(xh)
    out = torch.empty_like(xh).pin_memory()
    ctx.get_positions(out)
    assert torch.equal(out, xh)


# ------------------------------------------------------------------------------------------------
# BASELINE.json full sizes (bench.py's launch configuration), on outputs the oracle can afford
# ------------------------------------------------------------------------------------------------

def test_full_config4_sampled_samples_all_iterations():
    s = G.config4_batched()  # 4096 x 16^3, fp32, 100 Chebyshev iterations
    xg, Eg, _, q = run_gpu(s, "f32")
    assert q["n_batch"] == 4096 and q["n_colours"] == 8
    for b in (0, 1777, 4095):
        xo, Eo, _, _ = run_oracle(s, sample=b)
        assert_parity(s, "f32", xg[b], Eg[b], xo, Eo, extra=f"sample {b}")


@pytest.mark.parametrize("n_samples", [72, 97])
def test_batched_odd_group_count(n_samples):
    # 3 / 4 sample groups of 32 (the last ragged): the packed two-group fp32 kernel pairs groups (0, 1),
    # (2, 3) -- with 3 groups the last pair is padded by a zeroed group that is never stored
    s = G.config4_batched(n_samples=n_samples, n=4, iterations=20)
    xg, Eg, rg, q = run_gpu(s, "f32")
    assert q["n_batch"] == n_samples
    for b in (0, 63, 64, n_samples - 1):
        xo, Eo, _, _ = run_oracle(s, sample=b)
        assert_parity(s, "f32", xg[b], Eg[b], xo, Eo, extra=f"sample {b}")


@pytest.mark.parametrize("dtype", ["f64", "f32"])
@pytest.mark.parametrize("gamma,rho", [(0.5, 0.5), (1.7, 0.95), (0.5, 0.95), (1.7, 0.5)])
def test_chebyshev_gamma_closed_form_gpu(gamma, rho, dtype):
    # the oracle's closed-form pin (test_oracle_solver.py) run through the C ABI: one node tied to an
    # anchor, so the PBNG step is exact and e_{l+1} = omega_{l+1}(1-gamma) e_l + (1-omega_{l+1}) e_{l-1}
    # (PAPER.md:603-612); one iterate call per iteration continues the acceleration state
    from paper_2306_09021_b200 import context_from_scene
    from test_oracle_solver import _one_node_problem, chebyshev_error_recurrence
    s = _one_node_problem()
    t = s.wc["anchor"][0]
    n = 13
    ref = chebyshev_error_recurrence(s.x0[0][0] - t, n, rho, gamma)
    ctx = context_from_scene(s, device=0, dtype=dtype)
    tol = (1e-13 if dtype == "f64" else 2e-6) * np.abs(t).max()
    for l in range(n):
        ctx.iterate(1, "chebyshev", 1.0, rho, gamma)
        x = ctx.get_positions().cpu().numpy().astype(np.float64)[0, 0]
        assert np.abs((x - t) - ref[l + 1]).max() <= tol, (l, x - t, ref[l + 1])
    ctx.close()
