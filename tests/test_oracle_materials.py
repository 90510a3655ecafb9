"""Pins for the oracle's constitutive layer (§3.1 eq:cor/eq:nh/eq:lame, §7.1 eq:mod_hess_dens,
§"Lamé Coefficients").  Every check compares the oracle against something other than itself: printed
worked examples, closed forms, finite differences, invariances, or numpy's SVD."""
import json
import os

import numpy as np
import pytest

from oracle import cofactor, lame, mod_hess_density, piola, polar, psi

GOLD = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.Generator(np.random.PCG64(20240601))


def rand_rot(rng):
    q, r = np.linalg.qr(rng.standard_normal((3, 3)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] = -q[:, 0]
    return q


def rand_F(rng, inverted=False):
    U, V = rand_rot(rng), rand_rot(rng)
    s = rng.uniform(0.3, 1.8, size=3)
    if inverted:
        s[2] = -s[2]
    return U @ np.diag(s) @ V.T


def test_lame_golden():
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    for row in g["lame"]:
        mu, lam = lame(row["E"], row["nu"])
        assert abs(mu - row["mu"]) <= row["tol"]
        assert abs(lam - row["lambda"]) <= row["tol"]


@pytest.mark.parametrize("E,nu", [(1e5, 0.5), (1e5, 0.7), (-1.0, 0.3), (1e5, -0.1)])
def test_lame_rejects(E, nu):
    with pytest.raises(Exception):
        lame(E, nu)


def test_snh_printed_form_with_reparameterised_lame():
    # eq:snh evaluated literally with mu_s = 4 mu/3, lambda_s = lambda + 5 mu/6 and the
    # volume coefficient lambda_s / 2 (reading Z18), raw (unshifted) at a generic F
    mu, lam = 1.3, 2.2
    ms, ls = 4 * mu / 3, lam + 5 * mu / 6
    F = np.array([[1.1, 0.2, -0.1], [0.05, 0.9, 0.3], [0.0, -0.2, 1.2]])
    ic, J = np.sum(F * F), np.linalg.det(F)
    printed = 0.5 * ms * (ic - 3) + 0.5 * ls * (J - 1 - 3 * ms / (4 * ls)) ** 2 - 0.5 * ms * np.log(1 + ic)
    assert abs(psi("snh", mu, lam, F, raw=True) - printed) < 1e-13


def test_psi_golden():
    g = json.load(open(os.path.join(GOLD, "closed_forms.json")))
    for row in g["psi"]:
        v = psi(row["model"], row["mu"], row["lambda"], np.array(row["F"], float), raw=row["raw"])
        assert abs(v - row["value"]) < 1e-12


def test_cofactor_identities():
    # cof(diag(a,b,c)) = diag(bc, ac, ab); cof(F) F^T = det(F) I; cof = det F^{-T}
    assert np.allclose(cofactor(np.diag([2.0, 3.0, 5.0])), np.diag([15.0, 10.0, 6.0]), rtol=0, atol=0)
    for _ in range(200):
        F = RNG.standard_normal((3, 3))
        Cf = cofactor(F)
        d = np.linalg.det(F)
        assert np.allclose(Cf @ F.T, d * np.eye(3), atol=1e-12 * max(1, abs(d)))
        assert np.allclose(Cf, d * np.linalg.inv(F).T, rtol=1e-9, atol=1e-12)
    # singular F: still defined, rank-one identity holds
    F = np.array([[1.0, 2, 3], [2, 4, 6], [0, 1, 1]])
    assert np.allclose(cofactor(F) @ F.T, 0.0, atol=1e-12)


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_zero_energy_and_stress_at_rest(model):
    mu, lam = lame(1e5, 0.3)
    assert abs(psi(model, mu, lam, np.eye(3))) < 1e-9
    assert np.abs(piola(model, mu, lam, np.eye(3))).max() < 1e-9
    if model == "fcr":  # corotated: every rotation is a global minimiser
        for _ in range(50):
            Q = rand_rot(RNG)
            assert abs(psi(model, mu, lam, Q)) < 1e-6
            assert np.abs(piola(model, mu, lam, Q)).max() < 1e-6


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_piola_matches_finite_differences(model):
    mu, lam = 1.3, 2.1
    for t in range(60):
        F = rand_F(RNG, inverted=(t % 3 == 0))
        P = piola(model, mu, lam, F)
        h = 1e-6 * (1 + np.linalg.norm(F))
        Pfd = np.zeros((3, 3))
        for a in range(3):
            for b in range(3):
                E = np.zeros((3, 3))
                E[a, b] = h
                Pfd[a, b] = (psi(model, mu, lam, F + E) - psi(model, mu, lam, F - E)) / (2 * h)
        assert np.abs(P - Pfd).max() <= 1e-6 * (1 + np.abs(P).max())


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_rotation_invariance(model):
    mu, lam = 1.7, 0.9
    for t in range(60):
        F = rand_F(RNG, inverted=(t % 4 == 0))
        Q = rand_rot(RNG)
        a, b = psi(model, mu, lam, F), psi(model, mu, lam, Q @ F)
        assert abs(a - b) <= 1e-12 * max(1.0, abs(a))
        assert np.allclose(piola(model, mu, lam, Q @ F), Q @ piola(model, mu, lam, F), atol=1e-12, rtol=0)


def _np_cofactor(F):
    # signed 2x2 minors via numpy determinants (independent of the oracle's closed form)
    out = np.empty((3, 3))
    for a in range(3):
        for b in range(3):
            m = np.delete(np.delete(F, a, axis=0), b, axis=1)
            out[a, b] = (-1) ** (a + b) * np.linalg.det(m)
    return out


def test_modified_hessian_is_spd_with_closed_form_spectrum():
    # Ctilde = 2 mu I_9 + lambda vec(cof F) vec(cof F)^T: eigenvalues 2mu (x8) and 2mu + lambda |cof F|^2
    # ("a scaled version of the identity with a rank-one update"), for any F incl. det <= 0.
    mu, lam = 0.8, 3.0
    Fs = [rand_F(RNG, inverted=(t % 2 == 0)) for t in range(40)]
    Fs += [np.array([[1.0, 2, 3], [2, 4, 6], [0, 1, 1]]), np.zeros((3, 3)), np.diag([1.0, 1, -1])]
    for F in Fs:
        T = mod_hess_density(mu, lam, F)
        assert np.allclose(T, T.T, atol=0)
        w = np.sort(np.linalg.eigvalsh(T))
        cn = _np_cofactor(F)
        top = 2 * mu + lam * np.sum(cn * cn)
        assert np.allclose(w[:8], 2 * mu, rtol=1e-12, atol=1e-12)
        assert abs(w[8] - top) <= 1e-12 * top
        assert w[0] >= 2 * mu * (1 - 1e-12)


def _fd_density_hessian(model, mu, lam, F, h=1e-5):
    H = np.zeros((9, 9))
    for j in range(9):
        E = np.zeros(9)
        E[j] = h
        Pp = piola(model, mu, lam, F + E.reshape(3, 3)).reshape(9)
        Pm = piola(model, mu, lam, F - E.reshape(3, 3)).reshape(9)
        H[:, j] = (Pp - Pm) / (2 * h)
    return 0.5 * (H + H.T)


@pytest.mark.parametrize("model", ["nh", "fcr", "snh"])
def test_lame_consistency_at_identity(model):
    # the Hessian at F = I must equal linear elasticity's 2 mu P_sym + lambda I(x)I, which is
    # why eq:nh uses lambdahat = mu + lambda (and why eq:snh is read with the cited model's re-parameterised
    # Lame pair, reading Z18).  Also Ctilde(I) - C(I) = 2 mu P_skew (PSD).
    mu, lam = lame(1e5, 0.3)
    H = _fd_density_hessian(model, mu, lam, np.eye(3), h=1e-4)
    I9 = np.eye(9)
    K = np.zeros((9, 9))  # commutation (transpose) operator
    for a in range(3):
        for b in range(3):
            K[3 * a + b, 3 * b + a] = 1
    Psym, Pskew = 0.5 * (I9 + K), 0.5 * (I9 - K)
    vI = np.eye(3).reshape(9)
    Hle = 2 * mu * Psym + lam * np.outer(vI, vI)
    assert np.abs(H - Hle).max() <= 1e-5 * np.abs(Hle).max()
    Ct = mod_hess_density(mu, lam, np.eye(3))
    assert np.abs((Ct - Hle) - 2 * mu * Pskew).max() <= 1e-5 * np.abs(Hle).max()


def _numpy_closest_rotation(F):
    U, s, Vt = np.linalg.svd(F)
    if np.linalg.det(U) * np.linalg.det(Vt) < 0:
        U[:, 2] = -U[:, 2]
        s[2] = -s[2]
    return U @ Vt, s


def test_polar_rotation_matches_numpy_svd():
    # P8: R(F) vs numpy.linalg.svd with the sign correction of reading Z4, incl. inverted / near-singular F.
    n_checked = 0
    for t in range(20000):
        kind = t % 4
        if kind == 0:
            F = RNG.standard_normal((3, 3))
        elif kind == 1:
            F = rand_F(RNG, inverted=True)
        elif kind == 2:
            U, V = rand_rot(RNG), rand_rot(RNG)
            F = U @ np.diag([RNG.uniform(0.5, 2), RNG.uniform(0.5, 2), RNG.uniform(-1e-7, 1e-7)]) @ V.T
        else:
            F = np.eye(3) + 0.3 * RNG.standard_normal((3, 3))
        Rn, s = _numpy_closest_rotation(F)
        # R is unique only when the two smallest signed singular values do not cancel
        if abs(s[1] + s[2]) < 1e-6 * max(1.0, abs(s[0])):
            continue
        R = polar(F)
        assert abs(np.linalg.det(R) - 1) < 1e-12
        assert np.abs(R.T @ R - np.eye(3)).max() < 1e-12
        gap = abs(s[1] + s[2])
        assert np.abs(R - Rn).max() <= 1e-12 + 1e-13 / gap, (F, R, Rn)
        n_checked += 1
    assert n_checked > 19000


def test_polar_special_cases():
    assert np.allclose(polar(np.eye(3)), np.eye(3), atol=1e-15)
    Q = rand_rot(RNG)
    assert np.allclose(polar(Q), Q, atol=1e-13)
    # diag(3, 2, -1): the reflection is removed on the smallest singular direction -> R = I
    assert np.allclose(polar(np.diag([3.0, 2.0, -1.0])), np.eye(3), atol=1e-15)
    # rank-one F: still a rotation
    R = polar(np.outer([1.0, 2, 3], [0.5, -1, 2]))
    assert abs(np.linalg.det(R) - 1) < 1e-12
