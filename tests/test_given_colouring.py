"""pbng_color_given (include/pbng.h): a caller-supplied node colouring instead of the greedy one.
defines a node colouring (nodes of one colour share no element and no weak constraint); any such colouring is a
valid colour-parallel Gauss-Seidel order and fewer colours mean fewer, larger passes
(PAPER.md:707-709).  On a Kuhn grid (i + j + k) mod 4 is one (scenes.kuhn_grid_colouring), where the greedy
colouring in index order takes 8 colours.

CPU: the oracle with the given colouring is pinned by what does not depend on the colouring -- the PBNG fixed
point (the energy minimiser; north_star: residual 1e-8 against brute force) -- and the library's host logic
accepts exactly the valid colourings.  GPU: the CUDA path equals the oracle visiting the same colouring."""
import numpy as np
import pytest

from scenes import generators as G

TOL = {"f64": (1e-10, 1e-10), "f32": (1e-4, 1e-5)}


def cube(n, iterations):
    s = G.config3_hetero_cube(n=n, iterations=iterations)
    return s, G.kuhn_grid_colouring(n, n, n)


def test_kuhn_colouring_is_a_node_colouring_with_4_colours():
    X, tets = G.kuhn_grid(3, 4, 5, 0.5)
    col = G.kuhn_grid_colouring(3, 4, 5)
    assert col.shape == (X.shape[0],) and set(col.tolist()) == {0, 1, 2, 3}
    assert all(len(set(r)) == 4 for r in col[tets].tolist())


def test_oracle_fixed_point_does_not_depend_on_the_colouring():
    """Gauss-Seidel orders differ per iteration but share the fixed point: after enough iterations the greedy
    (8 colours) and the given (4 colours) oracles agree and both have a vanishing Newton residual."""
    from oracle import Oracle
    s, col = cube(4, 400)
    x0 = s.x0[0]
    a = Oracle(s)
    b = Oracle(s)
    b.set_colours(col)
    assert a.n_colours == 8 and b.n_colours == 4
    xa, _ = a.iterate(x0, x0, 0, s.iterations, "none", 1.0, 0.0, 1.0)
    xb, _ = b.iterate(x0, x0, 0, s.iterations, "none", 1.0, 0.0, 1.0)
    r0 = a.residual(x0)
    assert a.residual(xa) <= 1e-8 * r0 and a.residual(xb) <= 1e-8 * r0
    assert np.abs(xa - xb).max() <= 1e-9 * s.bbox_diag()
    # one iteration differs: the orders really are different
    ya, _ = a.iterate(x0, x0, 0, 1, "none", 1.0, 0.0, 1.0)
    yb, _ = b.iterate(x0, x0, 0, 1, "none", 1.0, 0.0, 1.0)
    assert np.abs(ya - yb).max() > 1e-6 * s.bbox_diag()


def test_host_logic_accepts_valid_and_rejects_invalid_colourings():
    from paper_2306_09021_b200 import context_from_scene
    from paper_2306_09021_b200.pbng import PBNGError
    s, col = cube(5, 3)
    ctx = context_from_scene(s, device=-1, dtype="f64", colours=col)
    q = ctx.query()
    assert ctx.n_colours == 4 and q["n_colours"] == 4
    greedy = context_from_scene(s, device=-1, dtype="f64")
    assert greedy.n_colours == 8 and greedy.query()["n_pairs"] == q["n_pairs"]
    bad = col.copy()
    v = int(s.tets[7][1])
    bad[v] = col[int(s.tets[7][2])]  # two vertices of tet 7 now share a colour
    with pytest.raises(PBNGError):
        ctx.color(bad)
    neg = col.copy()
    neg[3] = -1
    with pytest.raises(PBNGError):
        ctx.color(neg)
    ctx.close()
    greedy.close()


def test_constraint_nodes_must_differ_in_colour():
    from paper_2306_09021_b200 import context_from_scene
    from paper_2306_09021_b200.pbng import PBNGError
    s = G.make_config(5, "small")  # blocks bound by springs: a spring's two end nodes share no tet
    ctx = context_from_scene(s, device=-1, dtype="f64")
    col = ctx.colours.copy()
    assert ctx.color(col)[1] == ctx.n_colours  # the greedy colouring is itself accepted
    springs = [q for q in range(s.n_wc) if int(s.wc["n0"][q]) > 0 and int(s.wc["n1"][q]) > 0]
    assert springs
    q = springs[0]
    a, b = int(s.wc["idx0"][q][0]), int(s.wc["idx1"][q][0])
    assert a != b
    col2 = col.copy()
    col2[a] = col2[b]
    with pytest.raises(PBNGError):
        ctx.color(col2)
    ctx.close()


@pytest.mark.gpu
@pytest.mark.parametrize("n,dtype,accel", [(14, "f64", "sor"), (14, "f32", "sor"), (9, "f64", "chebyshev"),
                                           (9, "f32", "none")])
def test_gpu_equals_oracle_on_the_given_colouring(n, dtype, accel):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import Oracle
    from paper_2306_09021_b200 import context_from_scene
    s, col = cube(n, 30)
    s.accel = accel
    if accel == "chebyshev":
        s.rho, s.gamma = 0.95, 1.7
    o = Oracle(s)
    o.set_colours(col)
    x0 = s.x0[0]
    xo, _ = o.iterate(x0, x0, 0, s.iterations, s.accel, s.omega, s.rho, s.gamma)
    ctx = context_from_scene(s, device=0, dtype=dtype, colours=col)
    assert ctx.n_colours == 4
    ctx.iterate(s.iterations, s.accel, s.omega, s.rho, s.gamma)
    E, _ = ctx.energy_residual()
    xg = ctx.get_positions().cpu().numpy().astype(np.float64)[0]
    ctx.close()
    tx, te = TOL[dtype]
    assert np.abs(xg - xo).max() / s.bbox_diag() <= tx
    assert abs(float(E[0]) - o.energy(xo)) / abs(o.energy(xo)) <= te


@pytest.mark.gpu
def test_gpu_given_colouring_schedules_agree_bitwise_and_record_layouts_agree():
    """On the 4-colouring the pipelined schedule gives the bits of the colour launches (same per-vertex
    arithmetic, tests/test_gpu_schedule.py), and table and stored records agree to fp32 rounding."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2306_09021_b200 import context_from_scene
    s, col = cube(16, 12)  # h = 1/16: rest tuples exact in binary, so the table layout applies
    xs = {}
    for records, schedule in (("table", "colour_launches"), ("table", "pipelined"), ("stored", "colour_launches")):
        ctx = context_from_scene(s, device=0, dtype="f32", colours=col, records=records)
        ctx.set_schedule(schedule)
        assert ctx.n_colours == 4
        ctx.iterate(s.iterations, s.accel, s.omega, s.rho, s.gamma)
        xs[(records, schedule)] = ctx.get_positions().cpu().numpy()
        ctx.close()
    assert np.array_equal(xs[("table", "colour_launches")], xs[("table", "pipelined")])
    d = np.abs(xs[("table", "colour_launches")].astype(np.float64) - xs[("stored", "colour_launches")])
    assert d.max() <= 1e-5 * s.bbox_diag()


def _stack_colouring(n_blocks, n):
    # block b coloured (i + j + k + b) mod 4: a binding spring joins (i, j, n) of block b to (i, j, 0) of block
    # b + 1, colours (i + j + n + b) and (i + j + b + 1) mod 4, distinct while (n - 1) mod 4 != 0
    one = G.kuhn_grid_colouring(n, n, n)
    return np.concatenate([(one + b) % 4 for b in range(n_blocks)]).astype(np.int32)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,dtype", [(2, "f64"), (2, "f32"), (5, "f64"), (5, "f32")])
def test_gpu_equals_oracle_on_given_colourings_fixed_corotated(cfg, dtype):
    """Fixed-corotated configs (twisted bar with Chebyshev; stacked blocks with springs and contacts) on
    4-colourings: the split / pipelined kernels against the oracle visiting the same colouring."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from oracle import Oracle
    from paper_2306_09021_b200 import context_from_scene
    s = G.make_config(cfg, "small")
    col = G.kuhn_grid_colouring(6, 6, 24) if cfg == 2 else _stack_colouring(3, 7)
    s.iterations = 12
    o = Oracle(s)
    o.set_colours(col)
    x0 = s.x0[0]
    xo, _ = o.iterate(x0, x0, 0, s.iterations, s.accel, s.omega, s.rho, s.gamma)
    ctx = context_from_scene(s, device=0, dtype=dtype, colours=col)
    assert ctx.n_colours == 4
    ctx.iterate(s.iterations, s.accel, s.omega, s.rho, s.gamma)
    E, _ = ctx.energy_residual()
    xg = ctx.get_positions().cpu().numpy().astype(np.float64)[0]
    ctx.close()
    tx, te = TOL[dtype]
    assert np.abs(xg - xo).max() / s.bbox_diag() <= tx
    assert abs(float(E[0]) - o.energy(xo)) / abs(o.energy(xo)) <= te
