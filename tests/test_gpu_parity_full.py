"""Full-size, all-iteration GPU parity (BASELINE.json configs 2, 3 and 5 at their full sizes and iteration
counts, in bench.py's launch configuration) against the OpenMP build of the oracle.

The OpenMP oracle is the serial oracle's source compiled with -fopenmp; it is bitwise identical to the
serial build (tests/test_oracle_openmp.py) and mirrors the paper's OpenMP loop over a colour
(PAPER.md:710).  north_star tolerances after the same iteration count: fp64 1e-10 x bbox diagonal /
1e-10 relative energy; fp32 1e-4 x bbox diagonal / 1e-5 relative energy.  For fp32 each case also
reports the oracle's energy at the GPU iterate, E_orc(x_gpu), next to E_orc(x_orc): the first separates
iteration drift from the fp32 evaluation of the energy (SURVEY.md §8(c) "GPU vs oracle tolerances").
Set PBNG_PARITY_LOG=<path> to append one JSON line per case.
"""
import json
import os
import time

import numpy as np
import pytest

from scenes import generators as G

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

TOL = {"f64": (1e-10, 1e-10), "f32": (1e-4, 1e-5)}


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _host_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


_ORACLE_CACHE = {}


def oracle_run(key, scene):
    """x^L and E(x^L) of the OpenMP oracle (cached per module run: fp32 and fp64 share a config's run)."""
    if key not in _ORACLE_CACHE:
        from oracle import Oracle, threads
        threads(_host_threads())
        o = Oracle(scene, omp=True)
        if getattr(scene, "given_colours", None) is not None:
            o.set_colours(scene.given_colours)  # both sides visit the caller's colouring (pbng_color_given)
        x0 = scene.x0[0]
        t = time.perf_counter()
        x, _ = o.iterate(x0, x0, 0, scene.iterations, scene.accel, scene.omega, scene.rho, scene.gamma)
        _ORACLE_CACHE[key] = (o, x, o.energy(x), time.perf_counter() - t)
    return _ORACLE_CACHE[key]


def gpu_run(scene, dtype):
    from paper_2306_09021_b200 import context_from_scene
    ctx = context_from_scene(scene, device=0, dtype=dtype, colours=getattr(scene, "given_colours", None))
    ctx.iterate(scene.iterations, scene.accel, scene.omega, scene.rho, scene.gamma)
    E, r = ctx.energy_residual()
    x = ctx.get_positions().cpu().numpy().astype(np.float64)[0]
    ctx.close()
    return x, float(E[0])


def check(name, scene, dtype, key):
    o, xo, Eo, t_orc = oracle_run(key, scene)
    xg, Eg = gpu_run(scene, dtype)
    tx, te = TOL[dtype]
    err = float(np.abs(xg - xo).max() / scene.bbox_diag())
    erel = abs(Eg - Eo) / abs(Eo)
    E_at_gpu = o.energy(xg)
    line = {"case": name, "dtype": dtype, "iterations": scene.iterations,
            "max_pos_err_over_bbox_diag": err, "rel_energy_err": erel, "energy_gpu": Eg,
            "energy_oracle": Eo, "oracle_energy_at_gpu_iterate": E_at_gpu,
            "rel_iteration_drift": abs(E_at_gpu - Eo) / abs(Eo),
            "rel_fp_evaluation_err": abs(Eg - E_at_gpu) / abs(Eo),
            "oracle_threads": _host_threads(), "oracle_s": t_orc}
    print(json.dumps(line))
    log = os.environ.get("PBNG_PARITY_LOG")
    if log:
        with open(log, "a") as f:
            f.write(json.dumps(line) + "\n")
    assert err <= tx, f"{name} {dtype}: position error {err:.3e} > {tx}"
    assert erel <= te, f"{name} {dtype}: energy error {erel:.3e} > {te}"
    # the oracle's own energy at the GPU iterate is within the same bound (iteration drift alone)
    assert line["rel_iteration_drift"] <= te


@pytest.mark.parametrize("dtype", ["f32", "f64"])
def test_full_config3_all_iterations(dtype):
    s = G.config3_hetero_cube()  # 128^3, 12.6M tets, NH, per-tet lognormal E, SOR 1.5, 50 iterations
    check("config3_all_iterations", s, dtype, "c3")


def test_full_config3_given_4_colouring_all_iterations():
    """Config 3 at full size on the caller-supplied 4-colouring of the Kuhn grid (pbng_color_given): the
    CUDA path against the oracle visiting the same colouring, all 50 iterations."""
    s = G.config3_hetero_cube()
    s.given_colours = G.kuhn_grid_colouring(128, 128, 128)
    check("config3_kuhn4_all_iterations", s, "f32", "c3k4")


@pytest.mark.parametrize("noise_seed", [0, 1, 2, 3])
def test_full_config2_all_iterations(noise_seed):
    # fixed-corotated fp32 with Chebyshev (rho 0.95, gamma 1.7) over all 100 iterations, on four noise
    # seeds: the margin of the fp32 polar approximations against the 1e-5 energy bound
    s = G.config2_twisted_bar(noise_seed=noise_seed)
    check(f"config2_all_iterations_seed{noise_seed}", s, "f32", f"c2_{noise_seed}")


def test_full_config5_all_iterations():
    s = G.config5_muscle_stack()  # 8 x 48^3, springs + plane contacts + gravity, FCR fp32, 130 iterations
    check("config5_all_iterations", s, "f32", "c5")
