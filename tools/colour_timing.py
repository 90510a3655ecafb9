"""Warm per-colour-pass times of a config's sweep (public per-colour calls, CUDA events around each pass on
the context stream): how the iteration time splits over the colours, and the fixed cost per launch
(intercept of time vs vertices).  python tools/colour_timing.py [--config 3] [--reps 20]"""
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
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--dtype", default=None)
    a = ap.parse_args()
    s = G.make_config(a.config, "full")
    ctx = context_from_scene(s, device=0, dtype=a.dtype)
    ctx.set_schedule("colour_launches")
    nc = ctx.n_colours
    col = np.asarray(ctx.colours)
    free = np.ones(s.n_vertices, bool)
    free[s.pinned] = False
    nv = [int(((col == c) & free).sum()) for c in range(nc)]
    acc = (s.accel, s.omega, s.rho, s.gamma)
    ctx.iterate(3, *acc)
    st = torch.cuda.current_stream()
    t = np.zeros((a.reps, nc))
    for r in range(a.reps):
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(nc + 1)]
        ev[0].record(st)
        for c in range(nc):
            ctx.sweep_colour(c, *acc)
            ev[c + 1].record(st)
        ctx.end_iteration(s.accel)
        torch.cuda.synchronize()
        t[r] = [ev[c].elapsed_time(ev[c + 1]) * 1e3 for c in range(nc)]
    us = np.median(t, axis=0)
    b, a0 = np.polyfit(nv, us, 1)
    print(json.dumps({"config": a.config, "dtype": ctx.dtype, "vertices": nv, "us": us.round(2).tolist(),
                      "sum_us": float(us.sum()), "fit_us_per_1k_vertices": float(b * 1e3),
                      "fit_fixed_us_per_launch": float(a0)}))


if __name__ == "__main__":
    main()
