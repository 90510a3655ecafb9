"""Config 3 (full size) with the greedy colouring (8 colours) against a caller-supplied 4-colouring of the Kuhn
grid (pbng_color_given, scenes.kuhn_grid_colouring): ms per iteration of the colour sweeps, vertex-updates/s,
and energy / Newton residual after the config's 50 iterations (both orders are valid PBNG).

    python tools/colouring_timing.py [--dtype f32] [--n 128] [--reps 5]
One JSON line per colouring."""
import argparse
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch
    from paper_2306_09021_b200 import context_from_scene
    from scenes import generators as G

    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="f32")
    ap.add_argument("--n", type=int, default=128)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--config", type=int, default=3, choices=[2, 3, 4, 5],
                    help="2: twisted bar; 3: one n^3 cube; 4: 4096 samples of a 16^3 cube; 5: 8 stacked blocks")
    args = ap.parse_args()
    if args.config == 4:
        args.n = 16
        s = G.config4_batched()
        k4 = G.kuhn_grid_colouring(16, 16, 16)
    elif args.config == 2:
        s = G.config2_twisted_bar()
        k4 = G.kuhn_grid_colouring(32, 32, 128)
    elif args.config == 5:
        # block b is coloured (i + j + k + b) mod 4: the binding springs join the top face of block b to the
        # bottom face of block b + 1 at the same (i, j), colours (i + j + 48 + b) and (i + j + b + 1) mod 4
        s = G.config5_muscle_stack()
        one = G.kuhn_grid_colouring(48, 48, 48)
        k4 = np.concatenate([(one + b) % 4 for b in range(8)]).astype(np.int32)
    else:
        s = G.config3_hetero_cube(n=args.n)
        k4 = G.kuhn_grid_colouring(args.n, args.n, args.n)
    acc = (s.accel, s.omega, s.rho, s.gamma)
    for name, col in (("greedy", None), ("kuhn4", k4)):
        ctx = context_from_scene(s, device=0, dtype=args.dtype, colours=col)
        q = ctx.query()
        ctx.iterate(3, *acc)
        torch.cuda.synchronize()
        times = []
        for _ in range(args.reps):
            ctx.set_positions(np.asarray(s.x0))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.iterate(args.iters, *acc)
            e1.record()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) / args.iters)
        ctx.set_positions(np.asarray(s.x0))
        E0, R0 = ctx.energy_residual()
        ctx.iterate(s.iterations, *acc)
        E, R = ctx.energy_residual()
        ms = float(np.median(times))
        print(json.dumps({"colouring": name, "n_colours": int(ctx.n_colours), "dtype": ctx.dtype, "records": q["records"],
                          "ms_per_iter": ms, "min_ms": float(min(times)),
                          "config": args.config, "vupd_per_s": q["n_free"] * q["n_batch"] / (ms / 1e3), "iterations": s.iterations,
                          "energy_x0": float(E0[0]), "residual_x0": float(R0[0]),
                          "energy": float(E[0]), "residual": float(R[0]),
                          "residual_mean_over_samples": float(np.mean(R))}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
