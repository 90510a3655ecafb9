"""Probe: two independent half-size config-3 problems on two streams concurrently vs one after the other
(upper bound of what overlapping colour-pass tails across two halves could save)."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np, torch
from scenes import generators as G
from paper_2306_09021_b200 import context_from_scene
full = G.config3_hetero_cube()
half = G.config3_hetero_cube(n=128)
# half-height slab: 128 x 128 x 64 cells via the generator's grid with nz = 64 is not exposed; use n=101 (~half the vertices)
half = G.config3_hetero_cube(n=101)
acc = (full.accel, full.omega, full.rho, full.gamma)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
c1 = context_from_scene(half, device=0, stream=s1); c2 = context_from_scene(half, device=0, stream=s2)
cf = context_from_scene(full, device=0)
for c in (c1, c2, cf): c.iterate(3, *acc)
torch.cuda.synchronize()
def t(fn, reps=5):
    ts = []
    for _ in range(reps):
        torch.cuda.synchronize(); e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))
def conc():
    ev = torch.cuda.Event(); ev.record(); s1.wait_event(ev); s2.wait_event(ev)
    c1.iterate(10, *acc); c2.iterate(10, *acc)
    e1 = torch.cuda.Event(); e2 = torch.cuda.Event(); e1.record(s1); e2.record(s2)
    torch.cuda.current_stream().wait_event(e1); torch.cuda.current_stream().wait_event(e2)
def seq():
    ev = torch.cuda.Event(); ev.record(); s1.wait_event(ev)
    c1.iterate(10, *acc); e1 = torch.cuda.Event(); e1.record(s1); s2.wait_event(e1)
    c2.iterate(10, *acc); e2 = torch.cuda.Event(); e2.record(s2); torch.cuda.current_stream().wait_event(e2)
def one():
    cf.iterate(10, *acc)
nf = cf.query()["n_free"]; nh = c1.query()["n_free"]
r = {"full_ms_per_iter": t(one) / 10, "full_free": nf, "half_free_each": nh,
     "two_halves_concurrent_ms_per_iter": t(conc) / 10, "two_halves_sequential_ms_per_iter": t(seq) / 10}
r["concurrent_vupd_per_s"] = 2 * nh / (r["two_halves_concurrent_ms_per_iter"] / 1e3)
r["full_vupd_per_s"] = nf / (r["full_ms_per_iter"] / 1e3)
print(json.dumps(r))
