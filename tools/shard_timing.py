"""Per-GPU shard of config 4 at N GPUs (4096 / N samples): ms per iteration of the batched sweep under the
colour launches and the windowed persistent schedule (PBNG_B2_WINDOW), on one GPU.  Strong-scaling
evidence for the multi-GPU default (bench.py --gpus N shards config 4).

    python tools/shard_timing.py [--n 1 2 4 8] [--windows 0 2 4 8]
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
    ap.add_argument("--n", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--windows", type=int, nargs="+", default=[0, 2, 4, 8])
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args()
    full = G.config4_batched()
    for n in a.n:
        s = full.samples(0, 4096 // n)
        ctx = context_from_scene(s, device=0)
        q = ctx.query()
        for w in a.windows:
            os.environ["PBNG_B2_WINDOW"] = str(w)
            ctx.set_positions(np.asarray(s.x0))
            ctx.iterate(4, s.accel, s.omega, s.rho, s.gamma)
            times = []
            for _ in range(3):
                ctx.set_positions(np.asarray(s.x0))
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ctx.iterate(a.iters, s.accel, s.omega, s.rho, s.gamma)
                e1.record()
                torch.cuda.synchronize()
                times.append(e0.elapsed_time(e1) / a.iters)
            ms = float(np.median(times))
            print(json.dumps({"gpus": n, "samples": s.n_batch, "window": w, "ms_per_iter": ms,
                              "vupd_per_s": q["n_free"] * q["n_batch"] / (ms / 1e3)}), flush=True)
        ctx.close()


if __name__ == "__main__":
    main()
