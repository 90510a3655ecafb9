"""Debug: two blocks colliding, stored path records (PBNG_SPLIT=1) vs rest-recompute records, step by step."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np
import torch
from scenes import generators as G
from paper_2306_09021_b200 import context_from_scene

s = G.two_blocks_colliding(n=4)
dt, th, kn = s.meta["dt"], s.meta["thickness"], s.meta["k_n"]
ctxs = {r: context_from_scene(s, device=0, dtype="f64", records=r) for r in ("stored", "rest")}
for r, c in ctxs.items():
    print(r, c.query()["records"], c.query()["n_pair_slots"])
xp = {r: torch.tensor(s.meta["x_prev"][None], dtype=torch.float64, device="cuda:0") for r in ctxs}
xg = {r: torch.tensor(s.x0, dtype=torch.float64, device="cuda:0") for r in ctxs}
for step in range(1, 6):
    tgt = G.targets_at(s, step)
    wcs = {}
    for r, c in ctxs.items():
        wc = c.detect_contacts(th, kn)
        wcs[r] = wc
        c.set_inertia(dt, 2 * xg[r] - xp[r])
        n = c.update_constraints(wc, targets=tgt)
        c.iterate(int(sys.argv[1]) if len(sys.argv) > 1 else 20)
        xp[r], xg[r] = xg[r], c.get_positions()
        print(step, r, "contacts", len(wc), "recoloured", n, "records", c.query()["records"])
    d = (xg["stored"] - xg["rest"]).abs().cpu().numpy()[0].max(axis=1)
    bad = np.nonzero(d > 1e-12)[0]
    print("step", step, "maxdiff", d.max(), "n_bad", bad.size, "bad", bad[:20])
    if bad.size:
        cn = set()
        for w in wcs["rest"]:
            cn.update(w["idx0"][: w["n0"]].tolist()); cn.update(w["idx1"][: w["n1"]].tolist())
        print("bad with constraints", [int(b) for b in bad[:20] if b in cn])
