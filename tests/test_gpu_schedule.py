"""The pipelined (dataflow) schedule of pbng_iterate against the per-colour-launch schedule.

Both schedules make every vertex read exactly the same neighbour values (include/pbng.h pbng_schedule;
PAPER.md:693-705 fixes only the colour order), so the iterates, energies and residuals must be BITWISE
equal -- not merely within tolerance.  Iteration counts above 64 span several persistent launches.
"""
import numpy as np
import pytest

from scenes import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def run(scene, dtype, schedule, parts, accel=None):
    from paper_2306_09021_b200 import context_from_scene
    ctx = context_from_scene(scene, device=0, dtype=dtype)
    ctx.set_schedule(schedule)
    acc = scene.accel if accel is None else accel
    for k in parts:
        ctx.iterate(k, acc, scene.omega, scene.rho, scene.gamma)
    E, r = ctx.energy_residual()
    x = ctx.get_positions().cpu().numpy()
    q = ctx.query()
    ctx.close()
    return x, E, r, q


CASES = [
    (1, "full", "f64", None, [70]), (1, "full", "f64", "sor", [3, 66]), (1, "full", "f64", "chebyshev", [65, 2]),
    (2, "small", "f32", None, [20]), (3, "small", "f32", None, [30]), (3, "small", "f64", "sor", [7]),
    (5, "small", "f32", None, [12]), (5, "small", "f64", None, [5]), (4, "small", "f32", None, [9]),
]


@pytest.mark.parametrize("cfg,scale,dtype,accel,parts", CASES)
def test_pipelined_equals_colour_launches_bitwise(cfg, scale, dtype, accel, parts):
    s = G.make_config(cfg, scale)
    if accel == "sor":
        s.accel, s.omega = "sor", 1.5
    elif accel == "chebyshev":
        s.accel, s.rho, s.gamma = "chebyshev", 0.95, 1.7
    xa, Ea, ra, qa = run(s, dtype, "colour_launches", parts)
    xb, Eb, rb, qb = run(s, dtype, "pipelined", parts)
    assert qa["schedule"] == 1 and qb["schedule"] == 2
    assert np.array_equal(xa, xb), f"max diff {np.abs(xa - xb).max()}"
    assert np.array_equal(Ea, Eb) and np.array_equal(ra, rb)
    assert qb["iteration"] == qa["iteration"] == sum(parts)


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_pipelined_models_and_backward_euler(model):
    s = G.make_config(5, "small")
    s.model = model
    from paper_2306_09021_b200 import context_from_scene
    out = []
    for sched in ("colour_launches", "pipelined"):
        ctx = context_from_scene(s, device=0, dtype="f32")
        ctx.set_schedule(sched)
        ctx.set_inertia(1e-2, np.asarray(s.x0))
        ctx.iterate(10, "chebyshev", 1.0, 0.9, 1.0)
        out.append((ctx.get_positions().cpu().numpy(), ctx.energy_residual()))
        ctx.close()
    assert np.array_equal(out[0][0], out[1][0])
    assert np.array_equal(out[0][1][0], out[1][1][0])


_FULL_C3 = """
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from scenes import generators as G
from test_gpu_schedule import run
s = G.make_config(3, "full")
xa, Ea, _, qa = run(s, "f32", "colour_launches", [3])
xb, Eb, _, qb = run(s, "f32", "pipelined", [3])
assert qa["schedule"] == 1 and qb["schedule"] == 2
assert np.array_equal(xa, xb) and np.array_equal(Ea, Eb)
print("bitwise")
"""


def test_full_config3_pipelined_bitwise():
    # the pipelined schedule reads the plain three-id records; full-size config 3 uses path-ordered records
    # by default (colour launches only), so this comparison runs with PBNG_PATH=0 in a child process
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    code = _FULL_C3.format(root=os.path.dirname(here), tests=here)
    p = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, PBNG_PATH="0"), capture_output=True,
                       text=True, timeout=900)
    assert p.returncode == 0 and "bitwise" in p.stdout, p.stderr[-2000:]


def _batched_c5(n_samples):
    # config 5 (small) as a batch of NH problems: gravity (f^ext), springs + plane contacts (weak
    # constraints); every sample with its own noise
    s = G.make_config(5, "small")
    s.model = "nh"
    rng = np.random.default_rng(5)
    x0 = np.repeat(s.x0, n_samples, axis=0)
    free = np.setdiff1d(np.arange(s.n_vertices), s.pinned)
    x0[:, free] += rng.uniform(-0.02, 0.02, (n_samples, free.size, 3)) * s.h
    s.x0 = x0
    s.targets = np.repeat(s.targets, n_samples, axis=0)
    return s


@pytest.mark.parametrize("case", ["cheb100", "sor70", "c5_gravity_constraints", "c5_backward_euler", "empty_colours"])
def test_batched_window_schedule_equals_colour_launches_bitwise(case):
    """The windowed persistent schedule of the batched fp32 NH layout (sample-group pairs advance through the
    colours independently, an item waits only for its own group pair's previous colour pass) gives exactly
    the colour launches' iterates: ragged sample counts, > 64 iterations (two launches), SOR / Chebyshev /
    none, body force, weak constraints, backward Euler."""
    from paper_2306_09021_b200 import context_from_scene
    if case == "cheb100":
        s, parts, acc = G.config4_batched(n_samples=100, n=5, iterations=70), [70, 3], None
    elif case == "sor70":
        s, parts, acc = G.config4_batched(n_samples=65, n=4, iterations=70), [66, 4], "sor"
        s.accel, s.omega = "sor", 1.5
    elif case == "empty_colours":  # colours without free vertices: the waits chain over the non-empty ones
        from test_gpu_path_records import batch_of
        X = np.array([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [-1, 0, 0], [0, -1, 0], [0, 0, -1],
                      [0.4, 0.4, -0.8]], float)
        T = np.array([[0, 1, 2, 3], [0, 1, 2, 7], [0, 4, 5, 6]], np.int32)
        load = np.array([[0.1, 0, 0], [0, 0.1, 0], [-0.1, 0, 0], [0, -0.1, 0], [0, 0, -0.1]])
        s, parts, acc = batch_of(X, T, [1, 2, 4, 5, 6], 64, 0.05, 3, 25, load=load), [25], None
    else:
        s, parts, acc = _batched_c5(72), [12], None
    import os
    out = []
    for sched in ("colour_launches", "auto"):
        os.environ["PBNG_B2_WINDOW"] = "8" if sched == "auto" else "0"  # read by every pbng_iterate call
        ctx = context_from_scene(s, device=0, dtype="f32")
        assert ctx.query()["n_batch"] == s.n_batch
        ctx.set_schedule(sched)
        if case == "c5_backward_euler":
            ctx.set_inertia(1e-2, np.asarray(s.x0))
        for k in parts:
            ctx.iterate(k, s.accel, s.omega, s.rho, s.gamma)
        E, r = ctx.energy_residual()
        out.append((ctx.get_positions().cpu().numpy(), E, r, ctx.query()["kernel_launches"]))
        ctx.close()
    del os.environ["PBNG_B2_WINDOW"]
    assert np.array_equal(out[0][0], out[1][0]), np.abs(out[0][0] - out[1][0]).max()
    assert np.array_equal(out[0][1], out[1][1]) and np.array_equal(out[0][2], out[1][2])
    assert out[1][3] < out[0][3]  # the windowed schedule: one launch per <= 64 iterations


def test_full_config3_pipelined_path_records_bitwise():
    """Path-ordered records under the pipelined schedule (one-warp items walking the same records) give the
    colour launches' bits (measured slower on config 3, so auto keeps the colour launches)."""
    s = G.make_config(3, "full")
    xa, Ea, _, qa = run(s, "f32", "colour_launches", [2])
    xb, Eb, _, qb = run(s, "f32", "pipelined", [2])
    assert qa["schedule"] == 1 and qb["schedule"] == 2
    assert np.array_equal(xa, xb) and np.array_equal(Ea, Eb)
