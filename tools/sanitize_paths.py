"""Drive every kernel path of libpbng once on small scenes and check that each returns finite energies /
residuals (the non-finite flag is also checked by the library), e.g. under compute-sanitizer where a pool
allows it (`compute-sanitizer --tool memcheck python tools/sanitize_paths.py`; this pool refuses it):

Paths: colour launches (thread-per-vertex, split 2/4/8) and the pipelined schedule for Neo-Hookean,
fixed-corotated and stable Neo-Hookean in fp32 and fp64 with no / SOR / Chebyshev acceleration; the
sample-minor batched kernels (scalar and packed two-group); backward Euler; weak constraints; the
domain-decomposition halo pack / unpack and peer-store push (loopback, overlapped); contact detection + incremental
recolouring; energy / residual; positions in / out."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    import torch

    from paper_2306_09021_b200 import context_from_scene, dd
    from scenes import generators as G

    def run(s, dtype, schedule=None, iters=3):
        ctx = context_from_scene(s, device=0, dtype=dtype)
        if schedule:
            ctx.set_schedule(schedule)
        ctx.iterate(iters, s.accel, s.omega, s.rho, s.gamma)
        E, R = ctx.energy_residual()
        x = ctx.get_positions()
        assert np.all(np.isfinite(E)) and np.all(np.isfinite(R)) and bool(torch.isfinite(x).all())
        ctx.close()

    for cfg in (1, 5):
        s = G.make_config(cfg, "small")
        for dtype in ("f32", "f64"):
            for model in ("nh", "fcr", "snh"):
                s.model = model
                for accel in ("none", "sor", "chebyshev"):
                    s.accel, s.omega, s.rho, s.gamma = accel, 1.5, 0.9, 1.0
                    for sched in ("colour_launches", "pipelined"):
                        run(s, dtype, sched)
                print(f"config {cfg} {dtype} {model}", flush=True)
    for cfg in (2, 3):  # their own models / accelerations, both schedules
        s = G.make_config(cfg, "small")
        for dtype in ("f32", "f64"):
            for sched in ("colour_launches", "pipelined"):
                run(s, dtype, sched)
        print(f"config {cfg}", flush=True)
    # batched layouts (n_batch >= 32): scalar kernel (fp64, FCR) and the packed two-group kernel (fp32 NH)
    for n_samples, dtype, model in ((40, "f32", "nh"), (72, "f32", "nh"), (40, "f64", "nh"), (40, "f32", "fcr")):
        s = G.config4_batched(n_samples=n_samples, n=3, iterations=3)
        s.model = model
        run(s, dtype)
        print(f"batched {n_samples} {dtype} {model}", flush=True)
    # backward Euler
    s = G.make_config(5, "small")
    ctx = context_from_scene(s, device=0, dtype="f32")
    ctx.set_inertia(1e-2, np.asarray(s.x0))
    ctx.iterate(3, "none")
    ctx.energy_residual()
    ctx.close()
    # domain decomposition (loopback, overlapped exchange)
    for cfg in (3, 5):
        s = G.make_config(cfg, "small")
        ctxs, _ = dd.loopback_contexts(s, 2, dtype="f32")
        grp = dd.Group(ctxs)
        grp.iterate(2, s.accel, s.omega, s.rho, s.gamma)
        # the peer-store transport: rows stored straight into the other rank's ghost rows (bounds asserted)
        grp.set_transport("peer")
        grp.iterate(2, s.accel, s.omega, s.rho, s.gamma)
        for c in ctxs:
            E, R = c.energy_residual()
            assert np.all(np.isfinite(E)) and np.all(np.isfinite(R))
        grp.close()
        torch.cuda.synchronize()
        for c in ctxs:
            c.close()
        print(f"dd config {cfg} (copies + peer stores)", flush=True)
    s = G.config4_batched(n_samples=40, n=4, iterations=4)
    ctxs, _ = dd.loopback_contexts(s, 3, dtype="f32")
    grp = dd.Group(ctxs)
    grp.set_transport("peer")
    grp.iterate(3, s.accel, s.omega, s.rho, s.gamma)
    for c in ctxs:
        c.energy_residual()
    grp.close()
    for c in ctxs:
        c.close()
    print("dd batched sample-minor layout, 3 ranks, peer stores", flush=True)
    # path-ordered NH records: config 3 at a size where one warp per chunk is chosen (sweep_kernel path
    # mode), the batched sh-6 layout (path records), its windowed persistent schedule, a disconnected link
    s = G.config3_hetero_cube(n=80)
    run(s, "f32", iters=2)
    run(s, "f64", iters=1)
    s = G.config4_batched(n_samples=70, n=4, iterations=5)
    run(s, "f32")
    os.environ["PBNG_B2_WINDOW"] = "2"
    run(s, "f32", iters=66)
    del os.environ["PBNG_B2_WINDOW"]
    print("path records + window", flush=True)
    # contact detection + incremental recolouring
    s = G.two_blocks_colliding(n=3, gap=0.01)
    ctx = context_from_scene(s, device=0, dtype="f64")
    wc = ctx.detect_contacts(0.02, 1e8)
    ctx.update_constraints(wc)
    ctx.iterate(2, "none")
    ctx.close()
    print("contacts", len(wc), flush=True)
    torch.cuda.synchronize()
    print("sanitize paths done", flush=True)


if __name__ == "__main__":
    main()
