import sys, os, numpy as np, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch
from scenes import generators as G
from paper_2306_09021_b200 import context_from_scene
s = G.two_blocks_colliding(n=4)
dt, th, kn = s.meta["dt"], s.meta["thickness"], s.meta["k_n"]
ctx = context_from_scene(s, device=0, dtype="f64")
xp = torch.tensor(s.meta["x_prev"][None], dtype=torch.float64, device="cuda:0")
xc = torch.tensor(s.x0, dtype=torch.float64, device="cuda:0")
out = {}
for step in range(1, 5):
    tgt = G.targets_at(s, step)
    wc = ctx.detect_contacts(th, kn)
    n = ctx.update_constraints(wc, targets=tgt)
    q = ctx.query()
    x_after = ctx.get_positions().cpu().numpy()
    ctx.set_inertia(dt, 2 * xc - xp)
    E1 = ctx.energy_residual()
    ctx.iterate(1)
    x1 = ctx.get_positions().cpu().numpy()
    ctx.iterate(19)
    xp, xc = xc, ctx.get_positions()
    out[step] = {"n": n, "q": {k: q[k] for k in ("n_pairs", "n_pair_slots", "n_colours", "schedule", "n_weak_constraints")},
                 "E": [float(E1[0][0]), float(E1[1][0])], "x_after": x_after.tolist(), "x1": x1.tolist(), "x20": xc.cpu().numpy().tolist(),
                 "colours": ctx.get_colours()[0].tolist()}
json.dump(out, open(sys.argv[1], "w"))
