"""Dynamic weak constraints on the GPU: the library's device proximity detection
against the oracle's brute force at the same positions, and the paper's 'two blocks colliding' backward-
Euler example stepped with per-step detection + incremental recolouring
 against the oracle doing the same with its own detection and recolouring."""
import numpy as np
import pytest

from scenes import generators as G

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_cuda():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _free(s):
    f = np.ones(s.n_vertices, bool)
    f[s.pinned] = False
    return f


def _as_sets(vs, tris, w1):
    return {(int(v), tuple(int(t) for t in tri)): tuple(w) for v, tri, w in zip(vs, tris, w1)}


def compare(gpu_wc, orc_wc, tol=1e-9, k_atol=1e-6):
    g = _as_sets(gpu_wc["idx0"][:, 0], gpu_wc["idx1"][:, :3], gpu_wc["w1"][:, :3])
    o = _as_sets(orc_wc["idx0"][:, 0], orc_wc["idx1"][:, :3], orc_wc["w1"][:, :3])
    assert set(g) == set(o)
    for k in g:
        np.testing.assert_allclose(g[k], o[k], atol=tol)
    np.testing.assert_allclose(gpu_wc["K"], orc_wc["K"], rtol=1e-9, atol=k_atol)
    assert np.all(gpu_wc["n0"] == 1) and np.all(gpu_wc["n1"] == 3)


@pytest.mark.parametrize("dtype", ["f64", "f32"])
def test_device_detection_equals_oracle(dtype):
    import oracle.oracle as O
    from paper_2306_09021_b200 import context_from_scene
    s = G.two_blocks_colliding(n=4, gap=0.01)
    rng = np.random.default_rng(5)
    x = s.X + rng.uniform(-0.004, 0.004, s.X.shape)
    x[s.pinned] = s.X[s.pinned]
    ctx = context_from_scene(s, device=0, dtype=dtype)
    ctx.set_positions(x[None])
    xg = ctx.get_positions().cpu().numpy()[0].astype(np.float64)  # the device's copy (f32-rounded)
    wc = ctx.detect_contacts(0.02, 1e8)
    c = O.detect_contacts(s.X, xg, s.tets, _free(s), 0.02)
    assert c["count"] > 20 and len(wc) == c["count"]
    compare(wc, O.contact_constraints(c, 1e8))
    # separated: nothing
    ctx.set_positions(s.X[None] - np.where(np.arange(s.n_vertices) < 125, 0.05, -0.05)[None, :, None] * [1, 0, 0])
    assert len(ctx.detect_contacts(0.02, 1e8)) == 0
    ctx.close()


@pytest.mark.parametrize("inertia_first,records", [(False, "stored"), (True, "stored"), (True, "rest"),
                                                   (False, "table")])
def test_two_blocks_colliding_backward_euler_matches_oracle(inertia_first, records):
    """inertia_first: the backward-Euler target is set BEFORE pbng_update_constraints, which must carry it
    (and the iterate) over -- in place when the incremental recolouring changes no colour, across the
    re-layout otherwise; both paths occur in this run.  records = "rest" / "table": the lower-byte record
    layouts (pbng_set_records), which every re-layout must rebuild."""
    import torch

    import oracle.oracle as O
    from paper_2306_09021_b200 import context_from_scene
    s = G.two_blocks_colliding(n=4)
    dt, th, kn, K = s.meta["dt"], s.meta["thickness"], s.meta["k_n"], 20
    free = _free(s)
    # --- GPU: detect -> update (incremental recolour) -> inertia -> iterate, every step
    ctx = context_from_scene(s, device=0, dtype="f64", records=records)
    assert ctx.query()["records"] == {"stored": 1, "rest": 2, "table": 3}[records]
    xg_prev = torch.tensor(s.meta["x_prev"][None], dtype=torch.float64, device="cuda:0")
    xg = torch.tensor(s.x0, dtype=torch.float64, device="cuda:0")
    gpu_hist, gpu_wcs = [], []
    # --- oracle: the same with its own detection and recolouring
    col = O.Oracle(s).colours()
    nodes_prev = []
    xo_prev = s.meta["x_prev"].copy()
    xo = s.x0[0].copy()
    n_contact_steps = 0
    recoloured = []
    for step in range(1, 9):
        tgt = G.targets_at(s, step)
        wc = ctx.detect_contacts(th, kn)
        if inertia_first:
            ctx.set_inertia(dt, 2 * xg - xg_prev)
        recoloured.append(ctx.update_constraints(wc, targets=tgt))
        if not inertia_first:
            ctx.set_inertia(dt, 2 * xg - xg_prev)
        ctx.iterate(K)
        xg_prev, xg = xg, ctx.get_positions()
        gpu_hist.append(xg.cpu().numpy()[0])
        gpu_wcs.append(wc)

        c = O.detect_contacts(s.X, xo, s.tets, free, th)
        owc = O.contact_constraints(c, kn)
        # separately integrated trajectories differ by rounding (~1e-14): K = k_n n n^T then differs by
        # ~k_n 1e-14
        compare(wc, owc, tol=1e-9, k_atol=1e-12 * kn)
        n_contact_steps += c["count"] > 0
        nodes = O.constraint_nodes(owc) if c["count"] else []
        prev = {tuple(sorted(set(n))) for n in nodes_prev}
        is_new = [tuple(sorted(set(n))) not in prev for n in nodes]
        col, _ = O.recolor_incremental(s.n_vertices, s.tets, nodes, is_new, col)
        nodes_prev = nodes
        sc = G.two_blocks_colliding(n=4)
        sc.wc = owc if c["count"] else None
        sc.targets = tgt
        o = O.Oracle(sc)
        o.set_colours(col)
        o.set_inertia(dt, 2 * xo - xo_prev)
        x_in = xo.copy()
        x_in[sc.pinned] = tgt[0]
        x_new, _ = o.iterate(x_in, x_in, 0, K, "none")
        xo_prev, xo = xo, x_new
        gcol, _ = ctx.get_colours()
        assert np.array_equal(gcol, col), f"step {step}: colourings differ"
        err = np.abs(gpu_hist[-1] - xo).max() / s.bbox_diag()
        assert err <= 1e-10, f"step {step}: position error {err:.3e}"
    assert n_contact_steps >= 4  # the blocks met (step 3) and stayed in contact
    assert any(r == 0 for r in recoloured) and any(r > 0 for r in recoloured), recoloured
    ctx.close()


def test_detection_on_a_batched_context_uses_the_requested_sample():
    import oracle.oracle as O
    from paper_2306_09021_b200 import context_from_scene
    base = G.two_blocks_colliding(n=3, gap=0.01)
    nb = 40  # sample-minor layout (n_batch >= 32)
    rng = np.random.default_rng(9)
    xs = base.X[None] + rng.uniform(-0.004, 0.004, (nb,) + base.X.shape)
    xs[:, base.pinned] = base.X[base.pinned]
    s = G.two_blocks_colliding(n=3, gap=0.01)
    s.x0 = xs
    s.targets = np.repeat(base.targets, nb, axis=0)
    ctx = context_from_scene(s, device=0, dtype="f64")
    assert ctx.n_batch == nb
    for b in (0, 33, 39):
        wc = ctx.detect_contacts(0.02, 1e8, sample=b)
        c = O.detect_contacts(s.X, xs[b], s.tets, _free(s), 0.02)
        assert len(wc) == c["count"] > 0
        compare(wc, O.contact_constraints(c, 1e8))
    ctx.close()
