"""Pins for the oracle's rest-state precompute, body force, error
handling and the greedy node colouring (Table 1)."""
import json
import os

import numpy as np
import pytest

from oracle import Oracle
from oracle.oracle import OracleError
from scenes import generators as G

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def make_scene(X, tets, pinned=(), model="nh", E=1e5, nu=0.3, density=0.0, gravity=(0, 0, 0), wc=None, x0=None):
    X = np.asarray(X, float)
    tets = np.asarray(tets, np.int32).reshape(-1, 4)
    pinned = np.asarray(pinned, np.int32)
    x0 = (X if x0 is None else np.asarray(x0, float))[None].copy()
    return G.Scene("t", X, tets, model, np.atleast_1d(np.asarray(E, float)), nu, density,
                   np.asarray(gravity, float), pinned, x0[:, pinned].copy(), x0, wc=wc)


UNIT_TET = ([[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1]], [[0, 1, 2, 3]])


def test_unit_tet_volume_mass_and_gradients():
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))["unit_tet"]
    s = make_scene(*UNIT_TET, density=1.0, gravity=(0, 0, -1.0))
    o = Oracle(s)
    B, V = o.rest()
    assert abs(V[0] - g["volume"]) < 1e-16
    X = np.asarray(UNIT_TET[0], float)
    Dm = (X[1:] - X[0]).T
    assert np.allclose(B[0], np.linalg.inv(Dm), atol=1e-15)
    assert np.allclose(o.fext()[:, 2], -g["nodal_mass_per_density"], atol=1e-16)


@pytest.mark.parametrize("cfg", [1, 3, 5])
def test_volume_body_force_and_rest_gradient(cfg):
    s = G.make_config(cfg, "small")
    o = Oracle(s)
    B, V = o.rest()
    ext = s.X.max(0) - s.X.min(0)
    blocks = s.meta.get("blocks", 1)
    vol = ext[0] * ext[1] * ext[2] if cfg != 5 else ext[0] * ext[1] * ext[2]
    assert abs(V.sum() - vol) <= 1e-12 * vol * max(1, blocks)
    # V matches numpy's determinant of the rest edge matrix
    Xt = s.X[s.tets]
    Dm = np.transpose(Xt[:, 1:] - Xt[:, :1], (0, 2, 1))
    assert np.allclose(V, np.abs(np.linalg.det(Dm)) / 6, rtol=1e-13, atol=0)
    # sum of the consistent body force = rho g |Omega|
    f = o.fext().sum(0)
    assert np.allclose(f, s.density * s.gravity * vol, rtol=1e-12, atol=1e-12)
    # F = I at rest and F = A for an affine map y = A X + b
    rng = np.random.Generator(np.random.PCG64(3))
    A = np.eye(3) + 0.2 * rng.standard_normal((3, 3))
    y = s.X @ A.T + np.array([0.3, -1.0, 2.0])
    for e in rng.choice(s.n_tets, size=20, replace=False):
        assert np.allclose(o.deformation_gradient(s.X, e), np.eye(3), atol=1e-12)
        assert np.allclose(o.deformation_gradient(y, e), A, atol=1e-11)


def test_degenerate_element_is_rejected_with_index():
    X = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [1, 1, 0]]
    tets = [[0, 1, 2, 3], [0, 1, 4, 2]]  # second tet is flat (all z = 0)
    with pytest.raises(OracleError) as ei:
        Oracle(make_scene(X, tets))
    assert ei.value.code == 2 and ei.value.bad == 1


def test_isolated_free_vertex_is_rejected():
    X = [[0, 0, 0], [1, 0, 0], [0, 1, 0], [0, 0, 1], [5, 5, 5]]
    with pytest.raises(OracleError) as ei:
        Oracle(make_scene(X, [[0, 1, 2, 3]]))
    assert ei.value.code == 3 and ei.value.bad == 4
    Oracle(make_scene(X, [[0, 1, 2, 3]], pinned=[4]))  # pinned isolated vertex is fine


def test_bad_poisson_ratio_rejected():
    with pytest.raises(OracleError):
        Oracle(make_scene(*UNIT_TET, nu=0.5))


# ------------------------------------------------------------------------------------------------
# colouring
# ------------------------------------------------------------------------------------------------

def check_colouring(scene, colour):
    """Independent validity checker: no element or weak constraint has two nodes of one colour."""
    t = colour[scene.tets]
    for a in range(4):
        for b in range(a + 1, 4):
            assert not np.any(t[:, a] == t[:, b])
    if scene.wc is not None:
        wc = scene.wc
        for c in range(wc["n0"].shape[0]):
            nodes = list(wc["idx0"][c, :wc["n0"][c]]) + list(wc["idx1"][c, :wc["n1"][c]])
            nodes = list(dict.fromkeys(int(v) for v in nodes))
            cs = [int(colour[v]) for v in nodes]
            assert len(set(cs)) == len(cs)


def greedy_reference(scene):
    """Brute-force restatement of PAPER.md:702-705 over python sets (tiny inputs only)."""
    nv = scene.n_vertices
    stencils = [list(map(int, t)) for t in scene.tets]
    if scene.wc is not None:
        wc = scene.wc
        for c in range(wc["n0"].shape[0]):
            stencils.append(list(wc["idx0"][c, :wc["n0"][c]]) + list(wc["idx1"][c, :wc["n1"][c]]))
    S = [set() for _ in stencils]
    inc = [[] for _ in range(nv)]
    for k, st in enumerate(stencils):
        for v in set(int(u) for u in st):
            inc[v].append(k)
    out = np.zeros(nv, np.int32)
    for v in range(nv):
        used = set().union(*[S[k] for k in inc[v]]) if inc[v] else set()
        c = 0
        while c in used:
            c += 1
        out[v] = c
        for k in inc[v]:
            S[k].add(c)
    return out


def test_table1_particle_colour_counts():
    g = json.load(open(os.path.join(GOLD, "table1_colours.json")))
    for row in g["rows"]:
        X, T = G.five_tet_grid(row["n"])
        assert T.shape[0] == (row["n"] - 1) ** 3 * 5
        s = make_scene(X, T)
        o = Oracle(s)
        assert o.n_colours == row["particle_colors"], row
        check_colouring(s, o.colours())


def test_single_and_disjoint_tets():
    s = make_scene(*UNIT_TET)
    assert Oracle(s).n_colours == 4
    X = np.concatenate([np.asarray(UNIT_TET[0], float), np.asarray(UNIT_TET[0], float) + 3])
    s2 = make_scene(X, [[0, 1, 2, 3], [4, 5, 6, 7]])
    o2 = Oracle(s2)
    assert o2.n_colours == 4 and np.array_equal(o2.colours(), [0, 1, 2, 3, 0, 1, 2, 3])


@pytest.mark.parametrize("cfg", [1, 2, 3, 4, 5])
def test_colouring_valid_and_matches_bruteforce(cfg):
    s = G.make_config(cfg, "small")
    o = Oracle(s)
    c = o.colours()
    check_colouring(s, c)
    assert np.array_equal(c, Oracle(s).colours())  # deterministic
    if s.n_vertices < 3000:
        assert np.array_equal(c, greedy_reference(s))


def test_spring_network_colouring():
    s = G.spring_network()
    o = Oracle(s)
    check_colouring(s, o.colours())
    assert np.array_equal(o.colours(), greedy_reference(s))


def test_config1_class_sizes_survey_regression():
    # regression against the survey's own computation (not a paper value)
    o = Oracle(G.config1_tiny_cube())
    assert np.array_equal(np.bincount(o.colours()), [27, 25, 18, 25, 15, 3, 6, 6])
