"""Config-2 fp32 parity over all 100 iterations on several noise seeds for the library named by PBNG_LIB
(test infrastructure: runs the OpenMP oracle; oracle results are cached in the given directory so that
several library variants can be compared in one job).

    python tools/parity_variants.py <cache_dir> [seeds...]
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    from oracle import Oracle, threads
    from paper_2306_09021_b200 import context_from_scene
    from scenes import generators as G
    cache = sys.argv[1]
    seeds = [int(a) for a in sys.argv[2:]] or [0, 1, 2, 3]
    os.makedirs(cache, exist_ok=True)
    threads(len(os.sched_getaffinity(0)))
    for sd in seeds:
        s = G.config2_twisted_bar(noise_seed=sd)
        f = os.path.join(cache, f"c2_seed{sd}.npz")
        if os.path.exists(f):
            z = np.load(f)
            xo, Eo = z["x"], float(z["E"])
        else:
            o = Oracle(s, omp=True)
            xo, _ = o.iterate(s.x0[0], s.x0[0], 0, s.iterations, s.accel, s.omega, s.rho, s.gamma)
            Eo = o.energy(xo)
            np.savez(f, x=xo, E=Eo)
        ctx = context_from_scene(s, device=0, dtype="f32")
        ctx.iterate(s.iterations, s.accel, s.omega, s.rho, s.gamma)
        E, _ = ctx.energy_residual()
        x = ctx.get_positions().cpu().numpy().astype(np.float64)[0]
        ctx.close()
        print(json.dumps({"lib": os.environ.get("PBNG_LIB", "default"), "seed": sd,
                          "pos": float(np.abs(x - xo).max() / s.bbox_diag()), "energy": abs(float(E[0]) - Eo) / abs(Eo)}),
              flush=True)


if __name__ == "__main__":
    main()
