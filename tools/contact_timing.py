"""Cost of dynamic weak constraints at scale (the paper reports recolouring at < 680 ms
against 67 s of simulation per frame).

Two blocks colliding with n^3 Kuhn cells per block, backward Euler; every step:
detect contacts (pbng_detect_contacts), replace the constraints with incremental recolouring
(pbng_update_constraints: in place when no colour changes, re-layout otherwise), set the inertial target,
iterate K times.  Prints one JSON line per step and a summary with the update's share of the step.

    python tools/contact_timing.py [--n 32 48] [--steps 12] [--iters 40] [--dtype f32]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import numpy as np
    import torch
    from paper_2306_09021_b200 import context_from_scene
    from scenes import generators as G

    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, nargs="+", default=[32, 48])
    ap.add_argument("--steps", type=int, default=12)
    ap.add_argument("--iters", type=int, default=40)
    ap.add_argument("--dtype", default="f32")
    a = ap.parse_args()
    for n in a.n:
        s = G.two_blocks_colliding(n=n, dtype=a.dtype)
        dt, th, kn = s.meta["dt"], s.meta["thickness"], s.meta["k_n"]
        ctx = context_from_scene(s, device=0, dtype=a.dtype)
        td = torch.float32 if a.dtype == "f32" else torch.float64
        xg_prev = torch.tensor(s.meta["x_prev"][None], dtype=td, device="cuda:0")
        xg = torch.tensor(s.x0, dtype=td, device="cuda:0")
        rows = []
        for step in range(1, a.steps + 1):
            tgt = G.targets_at(s, step)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            wc = ctx.detect_contacts(th, kn)  # synchronises (returns host records)
            t1 = time.perf_counter()
            nrec = ctx.update_constraints(wc, targets=tgt)  # synchronises
            t2 = time.perf_counter()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.set_inertia(dt, 2 * xg - xg_prev)
            ctx.iterate(a.iters)
            x_new = ctx.get_positions()
            e1.record()
            torch.cuda.synchronize()
            xg_prev, xg = xg, x_new
            r = {"n": n, "step": step, "contacts": int(len(wc)), "recoloured": int(nrec),
                 "detect_ms": 1e3 * (t1 - t0), "update_ms": 1e3 * (t2 - t1), "iterate_ms": e0.elapsed_time(e1)}
            rows.append(r)
            print(json.dumps(r), flush=True)
        q = ctx.query()
        ctx.close()
        tot = sum(r["detect_ms"] + r["update_ms"] + r["iterate_ms"] for r in rows[1:])
        upd = sum(r["update_ms"] for r in rows[1:])
        det = sum(r["detect_ms"] for r in rows[1:])
        print(json.dumps({"summary": True, "n": n, "vertices": q["n_vertices"], "tets": q["n_tets"],
                          "iterations_per_step": a.iters, "steps_timed": len(rows) - 1,
                          "update_share": upd / tot, "detect_share": det / tot,
                          "relayout_steps": sum(1 for r in rows[1:] if r["recoloured"] > 0),
                          "mean_update_ms": upd / (len(rows) - 1), "mean_step_ms": tot / (len(rows) - 1),
                          "paper": "recolouring < 680 ms of 67 s per frame (< 1%), PAPER.md:756"}), flush=True)


if __name__ == "__main__":
    main()
