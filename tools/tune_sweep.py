"""Time the colour sweep on a BASELINE config for the sweep variant selected by PBNG_SWEEP_PIPE.

    PBNG_SWEEP_PIPE=1 python tools/tune_sweep.py [--config 3] [--iters 10] [--reps 5]
Prints one JSON line: ms per iteration, vertex-updates/s, algorithmic GB/s of the sweep and the energy
after the timed iterations (all variants do the same arithmetic in the same order).
"""
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
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--dtype", default=None)
    ap.add_argument("--records", default="auto", help="pair-record layout: auto | stored | rest")
    args = ap.parse_args()
    s = G.make_config(args.config, "full")
    ctx = context_from_scene(s, device=0, dtype=args.dtype, records=args.records)
    if os.environ.get("PBNG_L2PERSIST", "1") == "0":
        ctx.set_l2_persistence(False)
    q = ctx.query()
    acc = (s.accel, s.omega, s.rho, s.gamma)
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
    E, R = ctx.energy_residual()
    ms = float(np.median(times))
    byts = q["sweep_bytes"] + (q["accel_bytes"] if s.accel != "none" else 0)
    print(json.dumps({"pipe": os.environ.get("PBNG_SWEEP_PIPE", "default"), "config": args.config,
                      "records": q["records"],
                      "dtype": ctx.dtype, "ms_per_iter": ms, "min_ms": float(min(times)),
                      "vupd_per_s": q["n_free"] * q["n_batch"] / (ms / 1e3),
                      "GBps": byts / (ms / 1e3) / 1e9, "energy": float(E[0]), "residual": float(R[0])}))


if __name__ == "__main__":
    main()
