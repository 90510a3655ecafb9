"""Pins for the oracle's PBNG iteration (§7 eq:pbgn_dx / eq:mod_hess, §7.2 acceleration, §8
colour sweep): finite differences of the energy, dense assembly of eq:mod_hess, textbook block
Gauss-Seidel on a quadratic spring network, closed-form sub-iterates, acceleration closed forms, and the
fixed point against a brute-force global Newton solve (north_star item 4)."""
import numpy as np
import pytest

from oracle import Oracle, chebyshev_omega, mod_hess_density
from scenes import generators as G

from test_oracle_mesh import make_scene


def scene_with_model(model):
    s = G.config1_tiny_cube()
    s.model = model
    return s


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_nodal_force_is_minus_energy_gradient(model):
    # P4: f_i + f^ext_i = -dE/dx_i by central differences of the total energy
    s = scene_with_model(model)
    o = Oracle(s)
    x = s.x0[0].copy()
    rng = np.random.Generator(np.random.PCG64(11))
    r = o.forces(x)
    for i in rng.choice(s.n_vertices, size=12, replace=False):
        for a in range(3):
            h = 1e-6
            xp, xm = x.copy(), x.copy()
            xp[i, a] += h
            xm[i, a] -= h
            g = (o.energy(xp) - o.energy(xm)) / (2 * h)
            assert abs(-g - r[i, a]) <= 1e-6 * (1 + np.abs(r).max()), (i, a, -g, r[i, a])


def test_nodal_force_with_weak_constraints_fd():
    s = G.make_config(5, "small", dtype="f64")
    o = Oracle(s)
    x = s.x0[0].copy()
    wc = s.wc
    touched = np.unique(np.concatenate([wc["idx0"][:, 0], wc["idx1"][wc["n1"] > 0, 0]]))
    r = o.forces(x)
    for i in touched[:10]:
        for a in range(3):
            h = 1e-7
            xp, xm = x.copy(), x.copy()
            xp[i, a] += h
            xm[i, a] -= h
            g = (o.energy(xp) - o.energy(xm)) / (2 * h)
            assert abs(-g - r[i, a]) <= 1e-6 * (1 + np.abs(r).max())


@pytest.mark.parametrize("model", ["nh", "fcr"])
def test_nodal_hessian_dense_assembly_and_closed_form(model):
    # A_i = sum_e V_e G_e^T Ctilde_e G_e with G_e = d vec(F_e)/d x_i = I (x) g  (eq:mod_hess),
    # and equivalently 2 mu |g|^2 I + lambda (cof F g)(cof F g)^T per element.
    s = scene_with_model(model)
    o = Oracle(s)
    x = s.x0[0]
    B, V = o.rest()
    mu = s.E[0] / (2 * (1 + s.nu))
    lam = s.E[0] * s.nu / ((1 + s.nu) * (1 - 2 * s.nu))
    free = np.setdiff1d(np.arange(s.n_vertices), s.pinned)
    for i in free[:15]:
        f, A = o.nodal(x, i)
        Ad = np.zeros((3, 3))
        Ac = np.zeros((3, 3))
        for e in np.nonzero((s.tets == i).any(1))[0]:
            slot = int(np.nonzero(s.tets[e] == i)[0][0])
            Xt = s.X[s.tets[e]]
            Dinv = np.linalg.inv((Xt[1:] - Xt[0]).T)
            g = Dinv[slot - 1] if slot > 0 else -Dinv.sum(0)
            xt = x[s.tets[e]]
            F = (xt[1:] - xt[0]).T @ Dinv
            Gm = np.zeros((9, 3))
            for a in range(3):
                for b in range(3):
                    Gm[3 * a + b, a] = g[b]
            Ad += V[e] * Gm.T @ mod_hess_density(mu, lam, F) @ Gm
            w = (np.linalg.det(F) * np.linalg.inv(F).T) @ g
            Ac += V[e] * (2 * mu * (g @ g) * np.eye(3) + lam * np.outer(w, w))
        assert np.allclose(A, Ad, rtol=1e-12, atol=0)
        assert np.allclose(A, Ac, rtol=1e-10, atol=0)
        assert np.all(np.linalg.eigvalsh(A) > 0)


def test_rest_state_is_fixed():
    # P12: no loads, pins at rest, x = X -> one sweep returns X
    s = G.config1_tiny_cube()
    s.gravity = np.zeros(3)
    s.targets = s.X[s.pinned][None].copy()
    for model in ("nh", "fcr"):
        s.model = model
        o = Oracle(s)
        y = o.sweep(s.X)
        assert np.abs(y - s.X).max() <= 1e-14 * s.h


def test_translation_equivariance():
    s = G.config1_tiny_cube()
    s.gravity = np.zeros(3)
    s.pinned = np.zeros(0, np.int32)
    s.targets = np.zeros((1, 0, 3))
    o = Oracle(s)
    x = s.x0[0]
    t = np.array([0.37, -1.25, 2.5])
    a = o.sweep(x) + t
    b = o.sweep(x + t)
    assert np.abs(a - b).max() <= 1e-12


def test_residual_at_rest_under_gravity_closed_form():
    # at rest, r_i = f^ext_i = m_i g with lumped m_i = sum_e rho V_e / 4 (numpy volumes)
    s = G.config1_tiny_cube()
    s.targets = s.X[s.pinned][None].copy()
    o = Oracle(s)
    Xt = s.X[s.tets]
    V = np.abs(np.linalg.det(np.transpose(Xt[:, 1:] - Xt[:, :1], (0, 2, 1)))) / 6
    m = np.zeros(s.n_vertices)
    np.add.at(m, s.tets.reshape(-1), np.repeat(V * s.density / 4, 4))
    free = np.setdiff1d(np.arange(s.n_vertices), s.pinned)
    expect = np.sqrt(np.sum((m[free, None] * s.gravity[None]) ** 2))
    assert abs(o.residual(s.X) - expect) <= 1e-12 * expect


def _assemble_quadratic(scene):
    """Global K, b of the weak-constraint energy 1/2 sum_c C_c^T K_c C_c, C_c = S_c y - a_c."""
    n = scene.n_vertices
    wc = scene.wc
    K = np.zeros((3 * n, 3 * n))
    b = np.zeros(3 * n)
    for c in range(wc["n0"].shape[0]):
        s = np.zeros(n)
        for q in range(wc["n0"][c]):
            s[wc["idx0"][c, q]] += wc["w0"][c, q]
        for q in range(wc["n1"][c]):
            s[wc["idx1"][c, q]] -= wc["w1"][c, q]
        a = wc["anchor"][c] if wc["n1"][c] == 0 else np.zeros(3)
        k = wc["K"][c]
        Kc = np.array([[k[0], k[3], k[5]], [k[3], k[1], k[4]], [k[5], k[4], k[2]]])
        K += np.kron(np.outer(s, s), Kc)
        b += np.kron(s, Kc @ a)
    return K, b


def test_spring_network_sweep_is_block_gauss_seidel():
    # P10: quadratic energy -> A_i is the exact diagonal block, one PBNG sweep == one block Gauss-Seidel
    # sweep on K y = b in the same (colour, index) order
    s = G.spring_network()
    o = Oracle(s)
    K, b = _assemble_quadratic(s)
    col = o.colours()
    y = s.x0[0].reshape(-1).copy()
    for c in range(o.n_colours):
        for i in np.nonzero(col == c)[0]:
            I = slice(3 * i, 3 * i + 3)
            rhs = b[I] - K[I] @ y + K[I, I] @ y[I]
            y[I] = np.linalg.solve(K[I, I], rhs)
    z = o.sweep(s.x0[0]).reshape(-1)
    assert np.abs(y - z).max() <= 1e-12 * (1 + np.abs(y).max())
    # and repeated sweeps converge to the global minimiser K^{-1} b
    x = s.x0[0]
    for _ in range(3000):
        x = o.sweep(x)
    assert np.abs(x.reshape(-1) - np.linalg.solve(K, b)).max() < 1e-8


def test_single_spring_to_anchor_is_exact_in_one_subiterate():
    # a lone node tied to an anchor lands exactly on it (no elements)
    X = np.array([[0.0, 0.0, 0.0]])
    wc = G._empty_wc(1)
    wc["n0"][0] = 1
    wc["w0"][0, 0] = 1.0
    wc["anchor"][0] = (0.3, -0.2, 0.9)
    wc["K"][0] = (5.0, 7.0, 9.0, 1.0, 0.5, -0.3)
    s = make_scene(X, np.zeros((0, 4)), wc=wc, x0=np.array([[2.0, 1.0, -1.0]]))
    y = Oracle(s).sweep(s.x0[0])
    assert np.allclose(y[0], wc["anchor"][0], atol=1e-14)


def _one_node_problem():
    X = np.array([[0.0, 0.0, 0.0]])
    wc = G._empty_wc(1)
    wc["n0"][0] = 1
    wc["w0"][0, 0] = 1.0
    wc["anchor"][0] = (1.0, 2.0, 3.0)
    wc["K"][0, :3] = 4.0
    return make_scene(X, np.zeros((0, 4)), wc=wc, x0=np.array([[0.0, 0.0, 0.0]]))


def test_sor_closed_form_on_exactly_solvable_problem():
    # With x_PBNG = t every iteration, x^{l+1} = w t + (1 - w) x^{l-1} (reading Z7):
    # e_{l+1} = (1 - w) e_{l-1} with x^{-1} = x^0 (Z8).
    s = _one_node_problem()
    o = Oracle(s)
    t = s.wc["anchor"][0]
    w = 1.5
    x, xm1 = s.x0[0], s.x0[0]
    e = [x[0] - t, x[0] - t]  # e_{-1}, e_0
    for _ in range(8):
        x, xm1 = o.iterate(x, xm1, 0 if len(e) == 2 else len(e) - 2, 1, "sor", omega=w)
        e.append((1 - w) * e[-2])
        assert np.allclose(x[0] - t, e[-1], atol=1e-13)


def test_chebyshev_index_convention_and_limit():
    # omega_1 = omega_2 = 1 ("1 for l < 2"): with gamma = 1 an exact PBNG step stays exact.
    s = _one_node_problem()
    o = Oracle(s)
    t = s.wc["anchor"][0]
    x, xm1 = s.x0[0], s.x0[0]
    for l in range(6):
        x, xm1 = o.iterate(x, xm1, l, 1, "chebyshev", rho=0.95, gamma=1.0)
        assert np.allclose(x[0], t, atol=1e-12)
    # the recurrence's fixed point is the optimal Chebyshev weight 2 / (1 + sqrt(1 - rho^2))
    for rho in (0.5, 0.9, 0.95):
        assert abs(chebyshev_omega(2000, rho) - 2 / (1 + np.sqrt(1 - rho ** 2))) < 1e-12
        seq = [chebyshev_omega(m, rho) for m in range(1, 40)]
        assert seq[0] == 1.0 and seq[1] == 1.0
        # from omega_3 = 2 / (2 - rho^2) the weights decrease monotonically towards the limit
        assert all(b <= a for a, b in zip(seq[2:], seq[3:]))


def chebyshev_weights_from_paper(m_max, rho):
    """omega_1..omega_{m_max} written out from PAPER.md:603-608 (reading Z5): 1 for the first two
    iterates, 2/(2 - rho^2) for the third, then 4/(4 - rho^2 omega_prev).  Independent of the oracle."""
    w = [None, 1.0, 1.0]
    while len(w) <= m_max:
        w.append(2.0 / (2.0 - rho * rho) if len(w) == 3 else 4.0 / (4.0 - rho * rho * w[-1]))
    return w


def chebyshev_error_recurrence(e0, n, rho, gamma, variant="paper"):
    """Error e_l = x^l - t on a problem whose PBNG step is exact (p = t every iteration).  From
    x^{l+1} = omega_{l+1}(gamma (p - x^l) + x^l - x^{l-1}) + x^{l-1}:
        e_{l+1} = omega_{l+1} (1 - gamma) e_l + (1 - omega_{l+1}) e_{l-1},   e_{-1} = e_0 (Z8).
    The two misreadings this pin must reject:
      'gamma_on_prev' : gamma multiplies (p - x^{l-1}) instead of (p - x^l)
      'omega_l'       : omega_l used in place of omega_{l+1}"""
    w = chebyshev_weights_from_paper(n + 2, rho)
    em1, e = e0.copy(), e0.copy()
    out = [e.copy()]
    for l in range(n):
        om = w[l] if (variant == "omega_l" and l >= 1) else w[l + 1]
        if variant == "gamma_on_prev":
            en = om * (-gamma * em1 + e - em1) + em1
        else:
            en = om * (1.0 - gamma) * e + (1.0 - om) * em1
        em1, e = e, en
        out.append(e.copy())
    return out


@pytest.mark.parametrize("gamma", [0.5, 1.7])
@pytest.mark.parametrize("rho", [0.5, 0.95])
def test_chebyshev_gamma_closed_form_on_exactly_solvable_problem(gamma, rho):
    # VERDICT r1 "What's weak" 1: pins gamma's placement and the omega_{l+1} index for gamma != 1.
    s = _one_node_problem()
    o = Oracle(s)
    t = s.wc["anchor"][0]
    n = 13
    ref = chebyshev_error_recurrence(s.x0[0][0] - t, n, rho, gamma)
    x, xm1 = s.x0[0], s.x0[0]
    for l in range(n):
        x, xm1 = o.iterate(x, xm1, l, 1, "chebyshev", rho=rho, gamma=gamma)
        assert np.abs((x[0] - t) - ref[l + 1]).max() <= 1e-13 * np.abs(t).max(), l
    # the pin discriminates: both misreadings leave the paper's trajectory by far more than the tolerance
    for bad in ("gamma_on_prev", "omega_l"):
        alt = chebyshev_error_recurrence(s.x0[0][0] - t, n, rho, gamma, bad)
        assert max(np.abs(a - b).max() for a, b in zip(alt, ref)) > 1e-3 * np.abs(t).max(), bad


@pytest.mark.parametrize("accel", ["sor", "chebyshev"])
def test_acceleration_degenerate_cases(accel):
    # P13: SOR omega = 1 == plain; Chebyshev gamma = 1, rho = 0 == plain
    s = G.config1_tiny_cube()
    o = Oracle(s)
    x0 = s.x0[0]
    plain, _ = o.iterate(x0, x0, 0, 7, "none")
    acc, _ = o.iterate(x0, x0, 0, 7, accel, omega=1.0, rho=0.0, gamma=1.0)
    # equal up to the rounding of (p - x) + x
    assert np.abs(plain - acc).max() <= 1e-13 * s.h


def test_split_iteration_equals_single_call():
    # the acceleration state (l, x^{l-1}) continues across calls
    s = G.config1_tiny_cube()
    o = Oracle(s)
    x0 = s.x0[0]
    a, am = o.iterate(x0, x0, 0, 9, "chebyshev", rho=0.95, gamma=1.7)
    b, bm = o.iterate(x0, x0, 0, 4, "chebyshev", rho=0.95, gamma=1.7)
    b, bm = o.iterate(b, bm, 4, 5, "chebyshev", rho=0.95, gamma=1.7)
    assert np.array_equal(a, b) and np.array_equal(am, bm)


def _newton(o, s, x0, tol=1e-12, max_it=60):
    """Brute-force global Newton on E(x) over the free DOFs: FD Hessian of the oracle's forces,
    backtracking line search on the energy."""
    free = np.setdiff1d(np.arange(s.n_vertices), s.pinned)
    dof = (free[:, None] * 3 + np.arange(3)[None]).reshape(-1)
    x = x0.copy().reshape(-1)
    r0 = np.linalg.norm(o.forces(x).reshape(-1)[dof])
    for _ in range(max_it):
        r = o.forces(x).reshape(-1)[dof]
        if np.linalg.norm(r) <= tol * r0:
            break
        H = np.zeros((dof.size, dof.size))
        h = 1e-7 * s.h
        for j, d in enumerate(dof):
            xp, xm = x.copy(), x.copy()
            xp[d] += h
            xm[d] -= h
            H[:, j] = -(o.forces(xp).reshape(-1)[dof] - o.forces(xm).reshape(-1)[dof]) / (2 * h)
        H = 0.5 * (H + H.T)
        step = np.linalg.solve(H, r)
        E0 = o.energy(x)
        a = 1.0
        while a > 1e-8:
            xt = x.copy()
            xt[dof] += a * step
            if o.energy(xt) <= E0 + 1e-4 * a * (-(r @ step)):
                break
            a *= 0.5
        x = xt
    return x.reshape(-1, 3), r0


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_pbng_fixed_point_equals_global_newton(model):
    # P11 / north_star item 4: every stationary point of the sweep has f_i + f^ext_i = 0
    s = scene_with_model(model)
    o = Oracle(s)
    x0 = s.x0[0]
    xn, r0 = _newton(o, s, x0)
    x = x0
    for it in range(400):
        x_new, _ = o.iterate(x, x, 0, 50, "none")
        change = np.abs(x_new - x).max()
        x = x_new
        if change < 1e-14 * s.h:
            break
    assert o.residual(x) <= 1e-8 * r0
    assert o.residual(xn) <= 1e-10 * r0
    assert np.abs(x - xn).max() <= 1e-6 * s.bbox_diag()
