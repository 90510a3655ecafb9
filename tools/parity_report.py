"""Print the GPU-vs-oracle parity errors of the BASELINE configs (the cases of tests/test_gpu_parity.py at
full size) as one JSON line per case, for BASELINE.md's results table.  Test infrastructure: imports the
oracle.  Run on a GPU box:  python tools/parity_report.py > gpurun_out/parity.jsonl"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    full = "--full-fcr" in sys.argv  # configs 2 and 5 over all their iterations (oracle: ~3 and ~30 min)
    from oracle import Oracle
    from paper_2306_09021_b200 import context_from_scene
    from scenes import generators as G
    cases = [("config1", G.config1_tiny_cube(), "f64", None, [0]),
             ("config2", G.config2_twisted_bar(), "f32", 4, [0]),
             ("config3", G.config3_hetero_cube(), "f32", 1, [0]),
             ("config3_f64", G.config3_hetero_cube(), "f64", 1, [0]),
             ("config4", G.config4_batched(), "f32", None, [0, 1777, 4095]),
             ("config5", G.config5_muscle_stack(), "f32", 1, [0])]
    if full:
        cases = [("config2_all_iterations", G.config2_twisted_bar(), "f32", None, [0]),
                 ("config5_all_iterations", G.config5_muscle_stack(), "f32", None, [0])]
    if "--full-nh" in sys.argv:  # config 3 over its 50 iterations (oracle ~9 min)
        cases = [("config3_all_iterations", G.config3_hetero_cube(), "f32", None, [0])]
    if "--full-nh-f64" in sys.argv:  # the fp64 measurement variant of config 3 over its 50 iterations
        cases = [("config3_f64_all_iterations", G.config3_hetero_cube(), "f64", None, [0])]
    if "--many-c4" in sys.argv:  # config 4: 64 seeded random samples over all 100 iterations (~2 s each)
        picks = sorted(np.random.default_rng(2306).choice(4096, size=64, replace=False).tolist())
        cases = [("config4_64_samples", G.config4_batched(), "f32", None, picks)]
    for name, s, dtype, iters, samples in cases:
        n = s.iterations if iters is None else iters
        ctx = context_from_scene(s, device=0, dtype=dtype)
        ctx.iterate(n, s.accel, s.omega, s.rho, s.gamma)
        E, _ = ctx.energy_residual()
        x = ctx.get_positions().cpu().numpy().astype(np.float64)
        ctx.close()
        for b in samples:
            o = Oracle(s, b)
            x0 = s.x0[b]
            xo, _ = o.iterate(x0, x0, 0, n, s.accel, s.omega, s.rho, s.gamma)
            Eo = o.energy(xo)
            print(json.dumps({"case": name, "dtype": dtype, "iterations": n, "sample": b,
                              "max_pos_err_over_bbox_diag": float(np.abs(x[b] - xo).max() / s.bbox_diag()),
                              "rel_energy_err": float(abs(E[b] - Eo) / abs(Eo)),
                              "energy_gpu": float(E[b]), "energy_oracle": float(Eo)}), flush=True)


if __name__ == "__main__":
    main()
