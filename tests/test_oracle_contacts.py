"""Dynamic weak constraints: the oracle's closest point, boundary extraction, bodies,
contact detection and incremental recolouring pinned against closed forms, brute force
and an independent validity checker; and the library's host-side incremental recolouring (host-only
context, no GPU) against the oracle's, bit for bit."""
import numpy as np
import pytest

import oracle.oracle as O
from scenes import generators as G

pytestmark = pytest.mark.filterwarnings("ignore")


# ---- closest point on a triangle ------------------------------------------------------------------------
TRI = (np.array([0.0, 0.0, 0.0]), np.array([1.0, 0.0, 0.0]), np.array([0.0, 1.0, 0.0]))


@pytest.mark.parametrize("p,expect", [
    ((0.2, 0.2, 1.0), (0.6, 0.2, 0.2)),        # interior: the plane projection
    ((0.25, 0.5, -3.0), (0.25, 0.25, 0.5)),
    ((-1.0, -1.0, 0.5), (1.0, 0.0, 0.0)),      # vertex regions
    ((2.0, -0.5, 0.0), (0.0, 1.0, 0.0)),
    ((-0.5, 3.0, 0.2), (0.0, 0.0, 1.0)),
    ((0.5, -1.0, 0.0), (0.5, 0.5, 0.0)),       # edge regions
    ((-2.0, 0.25, 1.0), (0.75, 0.0, 0.25)),
    ((1.0, 1.0, 0.0), (0.0, 0.5, 0.5)),
])
def test_closest_point_closed_forms(p, expect):
    np.testing.assert_allclose(O.closest_point_triangle(p, *TRI), expect, atol=1e-15)


def test_closest_point_beats_dense_sampling():
    rng = np.random.default_rng(11)
    g = np.linspace(0.0, 1.0, 81)
    U, V = np.meshgrid(g, g)
    m = U + V <= 1.0
    bary = np.stack([1 - U[m] - V[m], U[m], V[m]], 1)
    for _ in range(40):
        a, b, c, p = rng.normal(size=(4, 3))
        w = O.closest_point_triangle(p, a, b, c)
        assert np.all(w >= -1e-14) and abs(w.sum() - 1.0) < 1e-14
        q = w[0] * a + w[1] * b + w[2] * c
        samples = bary @ np.stack([a, b, c])
        d_best = np.min(np.linalg.norm(samples - p, axis=1))
        assert np.linalg.norm(p - q) <= d_best + 1e-12
        assert np.linalg.norm(p - q) >= d_best - 0.05 * np.linalg.norm(b - a + c - a)  # sampling resolution


# ---- boundary and bodies --------------------------------------------------------------------------------
@pytest.mark.parametrize("n", [1, 2, 4])
def test_surface_of_kuhn_cube_is_closed_and_outward(n):
    X, T = G.kuhn_grid(n, n, n, 1.0 / n)
    tri, tt = O.surface(T, X)
    assert len(tri) == 12 * n * n  # 2 triangles per boundary cell face
    centre = X.mean(0)
    area = np.zeros(3)
    for t in tri:
        a, b, c = X[t]
        nrm = np.cross(b - a, c - a)
        assert np.dot(nrm, (a + b + c) / 3 - centre) > 0  # outward (convex body)
        area += nrm / 2
    np.testing.assert_allclose(area, 0.0, atol=1e-12)  # closed surface: vector area sums to zero
    edges = {}
    for t in tri:  # every edge is shared by exactly two triangles with opposite orientation
        for k in range(3):
            e = (t[k], t[(k + 1) % 3])
            edges[e] = edges.get(e, 0) + 1
    assert all(edges.get((j, i), 0) == 1 for (i, j) in edges)


def test_bodies_are_connected_components():
    s = G.config5_muscle_stack(n_blocks=3, n=2)
    b = O.bodies(s.n_vertices, s.tets)
    assert len(np.unique(b)) == 3
    nvb = 27
    for k in range(3):
        assert np.all(b[k * nvb:(k + 1) * nvb] == k * nvb)


# ---- contact detection ----------------------------------------------------------------------------------
def _free(s):
    f = np.ones(s.n_vertices, bool)
    f[s.pinned] = False
    return f


def test_separated_blocks_have_no_contacts():
    s = G.two_blocks_colliding(gap=0.1)
    c = O.detect_contacts(s.X, s.X, s.tets, _free(s), 0.02)
    assert c["count"] == 0 and np.all(c["tri"] == -1)


def test_single_vertex_over_triangle_interior():
    s = G.two_blocks_colliding(n=2, gap=0.5)
    y = s.X.copy()
    nvb = 27
    # a left-block vertex on its x = 1 face, moved to 0.01 in front of the right block's x = 1.5 face
    v = np.nonzero(np.isclose(s.X[:nvb, 0], 1.0) & np.isclose(s.X[:nvb, 1], 0.5) & np.isclose(s.X[:nvb, 2], 0.5))[0][0]
    y[v] = [1.49, 0.4, 0.55]
    c = O.detect_contacts(s.X, y, s.tets, _free(s), 0.02)
    assert c["count"] == 1 and c["tri"][v, 0] >= 0
    tri = c["tri"][v]
    q = c["bary"][v] @ y[tri]
    np.testing.assert_allclose(q, [1.5, 0.4, 0.55], atol=1e-14)  # the projection onto the face
    np.testing.assert_allclose(np.abs(c["normal"][v]), [1.0, 0.0, 0.0], atol=1e-14)
    assert c["normal"][v][0] < 0  # the right block's left face points to -x (outward)
    wc = O.contact_constraints(c, 1e8)
    assert wc["idx0"][0, 0] == v and np.isclose(wc["K"][0], [1e8, 0, 0, 0, 0, 0]).all()


def test_detection_equals_brute_force_rule():
    s = G.two_blocks_colliding(n=3, gap=0.01)
    rng = np.random.default_rng(3)
    y = s.X + rng.uniform(-0.003, 0.003, s.X.shape)
    free = _free(s)
    th = 0.02
    c = O.detect_contacts(s.X, y, s.tets, free, th)
    tri, _ = O.surface(s.tets, s.X)
    body = O.bodies(s.n_vertices, s.tets)
    on = np.zeros(s.n_vertices, bool)
    on[tri.reshape(-1)] = True
    ties = 0
    for v in range(s.n_vertices):
        cand = []
        if on[v] and free[v]:
            for k, t in enumerate(tri):
                if body[t[0]] == body[v]:
                    continue
                w = O.closest_point_triangle(y[v], *y[t])
                d2 = np.sum((y[v] - w @ y[t]) ** 2)
                if d2 <= th * th:
                    cand.append((d2, k))
        if not cand:
            assert c["tri"][v, 0] == -1
        else:  # the lowest index among the (near-)least distances (shared edges / vertices tie)
            dmin = min(d for d, _ in cand)
            k = min(k for d, k in cand if d <= dmin + 1e-10 * th * th)
            ties += sum(1 for d, _ in cand if d <= dmin + 1e-10 * th * th) > 1
            assert list(c["tri"][v]) == list(tri[k])
    assert c["count"] > 0 and ties > 0


# ---- incremental recolouring ----------------------------------------------------------------------------
def valid(colours, tets, nodes):
    for t in tets:
        if len(set(colours[t])) != 4:
            return False
    for n in nodes:
        u = sorted(set(n))
        if len(set(colours[u])) != len(u):
            return False
    return True


def test_recolour_without_new_constraints_is_identity():
    s = G.make_config(5, "small")
    o = O.Oracle(s)
    col = o.colours()
    nodes = O.constraint_nodes(s.wc)
    out, ch = O.recolor_incremental(s.n_vertices, s.tets, nodes, np.zeros(len(nodes), bool), col)
    assert ch == 0 and np.array_equal(out, col)


@pytest.mark.parametrize("seed", [0, 1, 2, 3])
def test_recolour_random_insertions_valid_and_local(seed):
    s = G.two_blocks_colliding(n=3, gap=0.0)
    o = O.Oracle(s)
    col = o.colours()
    rng = np.random.default_rng(seed)
    nodes = []
    for step in range(4):
        new = [list(rng.choice(s.n_vertices, size=rng.integers(2, 5), replace=False)) for _ in range(6)]
        allnodes = nodes + new
        is_new = np.array([False] * len(nodes) + [True] * len(new))
        out, ch = O.recolor_incremental(s.n_vertices, s.tets, allnodes, is_new, col)
        assert valid(out, s.tets, allnodes)
        extra = np.zeros(s.n_vertices, bool)
        for n in new:
            extra[n] = True
        assert np.all(out[~extra] == col[~extra])  # only incident nodes change
        assert ch == int(np.sum(out != col))
        col, nodes = out, allnodes


def test_recolour_keeps_previous_colour_when_free():
    # a constraint between two nodes of different colours that share no stencil: nobody changes
    s = G.two_blocks_colliding(n=2, gap=0.5)
    o = O.Oracle(s)
    col = o.colours()
    a = 0
    b = next(v for v in range(27, 54) if col[v] != col[a])
    out, ch = O.recolor_incremental(s.n_vertices, s.tets, [[a, b]], [True], col)
    assert ch == 0 and np.array_equal(out, col)
    # two same-coloured nodes of different blocks: visited in ascending order, the first one sees its
    # colour held by the second and moves; the second then keeps its colour (reading Z20)
    b = next(v for v in range(27, 54) if col[v] == col[a])
    out, ch = O.recolor_incremental(s.n_vertices, s.tets, [[a, b]], [True], col)
    assert ch == 1 and out[a] != col[a] and out[b] == col[b] and valid(out, s.tets, [[a, b]])


def _wc_from_nodes(nodes):
    n = len(nodes)
    wc = {"n0": np.ones(n, np.int32), "n1": np.zeros(n, np.int32), "idx0": np.zeros((n, 4), np.int32),
          "idx1": np.zeros((n, 4), np.int32), "w0": np.zeros((n, 4)), "w1": np.zeros((n, 4)),
          "anchor": np.zeros((n, 3)), "K": np.zeros((n, 6))}
    for k, nd in enumerate(nodes):
        wc["n0"][k] = 1
        wc["idx0"][k, 0] = nd[0]
        wc["w0"][k, 0] = 1.0
        wc["n1"][k] = len(nd) - 1
        wc["idx1"][k, :len(nd) - 1] = nd[1:]
        wc["w1"][k, :len(nd) - 1] = 1.0 / (len(nd) - 1)
        wc["K"][k, :3] = 1e3
    return wc


@pytest.mark.parametrize("seed", [0, 5])
def test_library_incremental_recolour_equals_oracle(seed):
    """Host-only library context: pbng_update_constraints recolours exactly as the oracle."""
    from paper_2306_09021_b200 import context_from_scene
    s = G.two_blocks_colliding(n=3, gap=0.0)
    ctx = context_from_scene(s, device=-1, dtype="f64")
    col, _ = ctx.get_colours()
    o = O.Oracle(s)
    assert np.array_equal(col, o.colours())
    rng = np.random.default_rng(seed)
    nodes = []
    for step in range(3):
        new = [[int(v) for v in rng.choice(s.n_vertices, size=rng.integers(2, 5), replace=False)] for _ in range(5)]
        keep = nodes[1:]  # one constraint removed, the others kept
        allnodes = keep + new
        is_new = [False] * len(keep) + [True] * len(new)
        expect, ch = O.recolor_incremental(s.n_vertices, s.tets, allnodes, is_new, col)
        n_re = ctx.update_constraints(_wc_from_nodes(allnodes))
        got, ncol = ctx.get_colours()
        assert np.array_equal(got, expect) and n_re == ch
        assert ncol == expect.max() + 1
        col, nodes = got, allnodes
    q = ctx.query()
    assert q["n_weak_constraints"] == len(nodes)
    ctx.close()
