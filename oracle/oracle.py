"""TEST INFRASTRUCTURE ONLY: ctypes wrapper around oracle/pbng_oracle.c (plain serial fp64 C).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may import
this module.  It performs argument marshalling only; all arithmetic is in pbng_oracle.c.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "pbng_oracle.c")
_SO = os.path.join(_HERE, "liborc.so")
_SO_OMP = os.path.join(_HERE, "liborc_omp.so")
_lock = threading.Lock()
_lib = None
_lib_omp = None

ACCEL = {"none": 0, "sor": 1, "chebyshev": 2}
MODEL = {"nh": 0, "fcr": 1, "snh": 2}
ERR = {0: "ok", 1: "invalid argument", 2: "degenerate element", 3: "isolated vertex", 4: "out of memory"}


class OracleError(RuntimeError):
    def __init__(self, code, bad=-1):
        super().__init__(f"oracle error {code} ({ERR.get(code, '?')}), index {bad}")
        self.code = code
        self.bad = bad


def build_oracle(force: bool = False, omp: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no FP contraction so the arithmetic is as written).  omp=True
    builds the same source with -fopenmp (liborc_omp.so): the colour pass runs its nodes on all host
    threads, as the paper's implementation does; results are bitwise those of the serial
    build (each node reads only other colours; sums are taken in a fixed order)."""
    so = _SO_OMP if omp else _SO
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(_SRC):
        tmp = so + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-std=c99", "-fPIC", "-shared"]
                              + (["-fopenmp"] if omp else []) + ["-o", tmp, _SRC, "-lm"])
        os.replace(tmp, so)
    return so


class _Scene(C.Structure):
    _fields_ = [
        ("nv", C.c_int64), ("X", C.c_void_p), ("nt", C.c_int64), ("tets", C.c_void_p),
        ("model", C.c_int32), ("E", C.c_void_p), ("nE", C.c_int64), ("nu", C.c_double),
        ("density", C.c_double), ("gravity", C.c_double * 3), ("npin", C.c_int64), ("pinned", C.c_void_p),
        ("nwc", C.c_int64), ("wc_n0", C.c_void_p), ("wc_n1", C.c_void_p), ("wc_idx0", C.c_void_p),
        ("wc_idx1", C.c_void_p), ("wc_w0", C.c_void_p), ("wc_w1", C.c_void_p), ("wc_anchor", C.c_void_p),
        ("wc_K", C.c_void_p),
    ]


def lib(omp: bool = False):
    """The serial oracle library, or (omp=True) the OpenMP build of the same source."""
    global _lib, _lib_omp
    with _lock:
        if (_lib_omp if omp else _lib) is None:
            L = C.CDLL(build_oracle(omp=omp))
            vp, d, i64, i32 = C.c_void_p, C.c_double, C.c_int64, C.c_int32
            L.orc_cofactor.argtypes = [vp, vp]
            L.orc_det.argtypes = [vp]
            L.orc_det.restype = d
            L.orc_lame.argtypes = [d, d, vp, vp]
            L.orc_lame.restype = C.c_int
            L.orc_polar.argtypes = [vp, vp]
            L.orc_psi.argtypes = [C.c_int, d, d, vp, C.c_int]
            L.orc_psi.restype = d
            L.orc_piola.argtypes = [C.c_int, d, d, vp, vp]
            L.orc_mod_hess_density.argtypes = [d, d, vp, vp]
            L.orc_prepare.argtypes = [C.POINTER(_Scene), C.POINTER(vp), C.POINTER(i64)]
            L.orc_prepare.restype = C.c_int
            L.orc_free.argtypes = [vp]
            L.orc_num_colours.argtypes = [vp]
            L.orc_num_colours.restype = i32
            L.orc_get_colour.argtypes = [vp, vp]
            L.orc_get_rest.argtypes = [vp, vp, vp]
            L.orc_get_fext.argtypes = [vp, vp]
            L.orc_deformation_gradient.argtypes = [vp, vp, i64, vp]
            L.orc_nodal.argtypes = [vp, vp, i64, vp, vp]
            L.orc_sweep_colour.argtypes = [vp, vp, i32]
            L.orc_sweep_colour.restype = i64
            L.orc_sweep.argtypes = [vp, vp]
            L.orc_sweep.restype = i64
            L.orc_chebyshev_omega.argtypes = [i64, d]
            L.orc_chebyshev_omega.restype = d
            L.orc_iterate.argtypes = [vp, vp, vp, i64, i32, i32, d, d, d]
            L.orc_iterate.restype = i64
            L.orc_forces.argtypes = [vp, vp, vp]
            L.orc_residual.argtypes = [vp, vp]
            L.orc_residual.restype = d
            L.orc_energy.argtypes = [vp, vp, vp]
            L.orc_energy.restype = d
            L.orc_set_inertia.argtypes = [vp, d, vp]
            L.orc_set_inertia.restype = C.c_int
            L.orc_get_mass.argtypes = [vp, vp]
            L.orc_recolor_incremental.argtypes = [i64, i64, vp, i64, vp, vp, vp, vp, vp, C.POINTER(i64)]
            L.orc_recolor_incremental.restype = C.c_int
            L.orc_closest_point_triangle.argtypes = [vp, vp, vp, vp, vp]
            L.orc_surface.argtypes = [i64, vp, vp, vp, vp]
            L.orc_surface.restype = i64
            L.orc_bodies.argtypes = [i64, i64, vp, vp]
            L.orc_detect_contacts.argtypes = [i64, vp, vp, i64, vp, vp, d, vp, vp, vp]
            L.orc_detect_contacts.restype = i64
            L.orc_contact_stiffness.argtypes = [vp, d, d, vp]
            L.orc_set_colours.argtypes = [vp, vp]
            L.orc_set_colours.restype = C.c_int
            L.orc_threads.argtypes = [C.c_int]
            L.orc_threads.restype = C.c_int
            if omp:
                _lib_omp = L
            else:
                _lib = L
    return _lib_omp if omp else _lib


def threads(n: int = 0) -> int:
    """Set (n > 0) and return the OpenMP oracle's thread count."""
    return int(lib(omp=True).orc_threads(int(n)))


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _mat(F):
    return np.ascontiguousarray(np.asarray(F, dtype=np.float64).reshape(3, 3))


def lame(E: float, nu: float):
    mu, lam = C.c_double(), C.c_double()
    st = lib().orc_lame(E, nu, C.byref(mu), C.byref(lam))
    if st:
        raise OracleError(st)
    return mu.value, lam.value


def cofactor(F):
    F = _mat(F)
    out = np.empty((3, 3))
    lib().orc_cofactor(_p(F), _p(out))
    return out


def polar(F):
    F = _mat(F)
    out = np.empty((3, 3))
    lib().orc_polar(_p(F), _p(out))
    return out


def psi(model: str, mu: float, lam: float, F, raw: bool = False) -> float:
    F = _mat(F)
    return lib().orc_psi(MODEL[model], mu, lam, _p(F), int(raw))


def piola(model: str, mu: float, lam: float, F):
    F = _mat(F)
    out = np.empty((3, 3))
    lib().orc_piola(MODEL[model], mu, lam, _p(F), _p(out))
    return out


def mod_hess_density(mu: float, lam: float, F):
    """Ctilde as a 9x9 matrix, row (alpha,gamma) = 3*alpha+gamma, column (beta,delta) = 3*beta+delta."""
    F = _mat(F)
    out = np.empty((9, 9))
    lib().orc_mod_hess_density(mu, lam, _p(F), _p(out))
    return out


def chebyshev_omega(m: int, rho: float) -> float:
    return lib().orc_chebyshev_omega(m, rho)


# ---- dynamic weak constraints ----------------------------------------------------
def _i32(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.int32))


def _f64(a):
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def constraint_nodes(wc) -> list:
    """Node list of every weak constraint of a scenes-style dict (side 0 then side 1, as given)."""
    if wc is None:
        return []
    out = []
    for c in range(len(wc["n0"])):
        out.append([int(v) for v in wc["idx0"][c][:wc["n0"][c]]] + [int(v) for v in wc["idx1"][c][:wc["n1"][c]]])
    return out


def recolor_incremental(nv: int, tets, nodes: list, is_new, colour_prev):
    """PAPER.md:748-754 incremental recolouring (pbng_oracle.c orc_recolor_incremental): returns
    (colours, number of nodes whose colour changed)."""
    tets = _i32(tets).reshape(-1, 4)
    off = np.zeros(len(nodes) + 1, np.int64)
    for c, n in enumerate(nodes):
        off[c + 1] = off[c] + len(n)
    flat = _i32(np.concatenate([np.asarray(n, np.int32) for n in nodes]) if nodes else np.zeros(1, np.int32))
    new = np.ascontiguousarray(np.asarray(is_new, dtype=np.uint8).reshape(-1)) if nodes else np.zeros(1, np.uint8)
    prev = _i32(colour_prev)
    out = np.empty(nv, np.int32)
    ch = C.c_int64()
    st = lib().orc_recolor_incremental(nv, tets.shape[0], _p(tets), len(nodes), _p(off), _p(flat), _p(new), _p(prev),
                                       _p(out), C.byref(ch))
    if st:
        raise OracleError(st)
    return out, ch.value


def closest_point_triangle(p, a, b, c):
    args = [_f64(v).reshape(3) for v in (p, a, b, c)]
    out = np.empty(3)
    lib().orc_closest_point_triangle(*[_p(v) for v in args], _p(out))
    return out


def surface(tets, X):
    tets = _i32(tets).reshape(-1, 4)
    X = _f64(X).reshape(-1, 3)
    tri = np.empty((4 * tets.shape[0] + 1, 3), np.int32)
    tt = np.empty(4 * tets.shape[0] + 1, np.int32)
    n = lib().orc_surface(tets.shape[0], _p(tets), _p(X), _p(tri), _p(tt))
    if n < 0:
        raise OracleError(4)
    return tri[:n].copy(), tt[:n].copy()


def bodies(nv: int, tets):
    tets = _i32(tets).reshape(-1, 4)
    out = np.empty(nv, np.int32)
    lib().orc_bodies(nv, tets.shape[0], _p(tets), _p(out))
    return out


def detect_contacts(X, y, tets, free_mask, thickness: float):
    """Per-vertex closest other-body boundary triangle within `thickness` (pbng_oracle.c
    orc_detect_contacts): dict of tri (nv, 3; -1 = none), bary (nv, 3), normal (nv, 3), count."""
    X = _f64(X).reshape(-1, 3)
    y = _f64(y).reshape(-1, 3)
    tets = _i32(tets).reshape(-1, 4)
    fm = np.ascontiguousarray(np.asarray(free_mask, dtype=np.uint8))
    nv = X.shape[0]
    tri = np.empty((nv, 3), np.int32)
    bary = np.empty((nv, 3))
    nrm = np.empty((nv, 3))
    n = lib().orc_detect_contacts(nv, _p(X), _p(y), tets.shape[0], _p(tets), _p(fm), float(thickness), _p(tri),
                                  _p(bary), _p(nrm))
    if n < 0:
        raise OracleError(4)
    return {"tri": tri, "bary": bary, "normal": nrm, "count": int(n)}


def contact_constraints(contacts, kn: float, kt: float = 0.0) -> dict:
    """The weak constraints of detected contacts, in ascending vertex order (scenes-style dict): side 0 =
    the vertex, side 1 = the triangle with barycentric weights, K = k_n n n^T + k_t (I - n n^T)."""
    vs = np.nonzero(contacts["tri"][:, 0] >= 0)[0]
    n = len(vs)
    wc = {"n0": np.ones(n, np.int32), "n1": np.full(n, 3, np.int32), "idx0": np.zeros((n, 4), np.int32),
          "idx1": np.zeros((n, 4), np.int32), "w0": np.zeros((n, 4)), "w1": np.zeros((n, 4)),
          "anchor": np.zeros((n, 3)), "K": np.zeros((n, 6))}
    for k, v in enumerate(vs):
        wc["idx0"][k, 0] = v
        wc["w0"][k, 0] = 1.0
        wc["idx1"][k, :3] = contacts["tri"][v]
        wc["w1"][k, :3] = contacts["bary"][v]
        nv_ = _f64(contacts["normal"][v])
        K6 = np.empty(6)
        lib().orc_contact_stiffness(_p(nv_), float(kn), float(kt), _p(K6))
        wc["K"][k] = K6
    return wc


class Oracle:
    """Prepared oracle for one sample of a scene (scenes.Scene)."""

    def __init__(self, scene, sample: int = 0, omp: bool = False):
        """omp=True runs the same oracle source built with OpenMP (bitwise identical, all host threads)."""
        L = lib(omp)
        self._L = L
        self.scene = scene
        self.sample = sample
        self._keep = []

        def keep(a, dt):
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return _p(a)

        s = _Scene()
        s.nv = scene.n_vertices
        s.X = keep(scene.X, np.float64)
        s.nt = scene.n_tets
        s.tets = keep(scene.tets if scene.n_tets else np.zeros((1, 4), np.int32), np.int32)
        s.model = MODEL[scene.model]
        s.E = keep(scene.E, np.float64)
        s.nE = int(np.asarray(scene.E).size)
        s.nu = scene.nu
        s.density = scene.density
        for k in range(3):
            s.gravity[k] = float(scene.gravity[k])
        s.npin = int(scene.pinned.size)
        s.pinned = keep(scene.pinned if scene.pinned.size else np.zeros(1, np.int32), np.int32)
        wc = scene.wc
        if wc is None:
            s.nwc = 0
            z4 = np.zeros((1, 4), np.int32)
            s.wc_n0 = keep(np.zeros(1, np.int32), np.int32)
            s.wc_n1 = keep(np.zeros(1, np.int32), np.int32)
            s.wc_idx0 = keep(z4, np.int32)
            s.wc_idx1 = keep(z4, np.int32)
            s.wc_w0 = keep(np.zeros((1, 4)), np.float64)
            s.wc_w1 = keep(np.zeros((1, 4)), np.float64)
            s.wc_anchor = keep(np.zeros((1, 3)), np.float64)
            s.wc_K = keep(np.zeros((1, 6)), np.float64)
        else:
            s.nwc = int(wc["n0"].shape[0])
            s.wc_n0 = keep(wc["n0"], np.int32)
            s.wc_n1 = keep(wc["n1"], np.int32)
            s.wc_idx0 = keep(wc["idx0"], np.int32)
            s.wc_idx1 = keep(wc["idx1"], np.int32)
            s.wc_w0 = keep(wc["w0"], np.float64)
            s.wc_w1 = keep(wc["w1"], np.float64)
            s.wc_anchor = keep(wc["anchor"], np.float64)
            s.wc_K = keep(wc["K"], np.float64)
        handle = C.c_void_p()
        bad = C.c_int64(-1)
        st = L.orc_prepare(C.byref(s), C.byref(handle), C.byref(bad))
        self._keep = []
        if st:
            raise OracleError(st, bad.value)
        self._h = handle
        self.nv = scene.n_vertices
        self.nt = scene.n_tets

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and getattr(self, "_L", None) is not None:
            self._L.orc_free(h)
            self._h = None

    # ---- precompute getters ------------------------------------------------------------------------
    def set_colours(self, colours) -> None:
        """Use a given colouring (e.g. recolor_incremental's) for the sweeps."""
        c = np.ascontiguousarray(np.asarray(colours, dtype=np.int32))
        st = self._L.orc_set_colours(self._h, _p(c))
        if st:
            raise OracleError(st)

    @property
    def n_colours(self) -> int:
        return int(self._L.orc_num_colours(self._h))

    def colours(self) -> np.ndarray:
        out = np.empty(self.nv, np.int32)
        self._L.orc_get_colour(self._h, _p(out))
        return out

    def rest(self):
        B = np.empty((max(self.nt, 1), 3, 3))
        V = np.empty(max(self.nt, 1))
        self._L.orc_get_rest(self._h, _p(B), _p(V))
        return B[:self.nt], V[:self.nt]

    def mass(self) -> np.ndarray:
        out = np.empty(self.nv)
        self._L.orc_get_mass(self._h, _p(out))
        return out

    def set_inertia(self, dt: float, xtilde=None):
        """Backward Euler (eq:fem_be): dt > 0 with xtilde = 2 x^n - x^{n-1}; dt = 0 -> quasistatic."""
        xt = None if xtilde is None else self._x(xtilde)
        st = self._L.orc_set_inertia(self._h, float(dt), _p(xt) if xt is not None else None)
        if st:
            raise OracleError(st)

    def fext(self) -> np.ndarray:
        out = np.empty((self.nv, 3))
        self._L.orc_get_fext(self._h, _p(out))
        return out

    # ---- evaluation --------------------------------------------------------------------------------
    def _x(self, x):
        x = np.ascontiguousarray(np.asarray(x, dtype=np.float64).reshape(self.nv, 3))
        return x

    def deformation_gradient(self, x, e: int):
        x = self._x(x)
        F = np.empty((3, 3))
        self._L.orc_deformation_gradient(self._h, _p(x), e, _p(F))
        return F

    def nodal(self, x, i: int):
        x = self._x(x)
        f = np.empty(3)
        A = np.empty((3, 3))
        self._L.orc_nodal(self._h, _p(x), int(i), _p(f), _p(A))
        return f, A

    def forces(self, x) -> np.ndarray:
        x = self._x(x)
        out = np.empty((self.nv, 3))
        self._L.orc_forces(self._h, _p(x), _p(out))
        return out

    def residual(self, x) -> float:
        x = self._x(x)
        return float(self._L.orc_residual(self._h, _p(x)))

    def energy(self, x, parts: bool = False):
        x = self._x(x)
        pr = np.empty(3)
        e = float(self._L.orc_energy(self._h, _p(x), _p(pr)))
        return (e, pr) if parts else e

    # ---- iteration ---------------------------------------------------------------------------------
    def sweep(self, x) -> np.ndarray:
        w = self._x(x).copy()
        fails = self._L.orc_sweep(self._h, _p(w))
        if fails:
            raise RuntimeError(f"{fails} nodal solves failed")
        return w

    def sweep_colour_inplace(self, w: np.ndarray, c: int) -> None:
        """One colour pass of a PBNG iteration, in place on a float64 C-contiguous (nv, 3) array."""
        assert w.dtype == np.float64 and w.flags.c_contiguous and w.shape == (self.nv, 3)
        fails = self._L.orc_sweep_colour(self._h, _p(w), int(c))
        if fails:
            raise RuntimeError(f"{fails} nodal solves failed")

    def iterate(self, x, xm1, l0: int, n: int, accel: str = "none", omega: float = 1.0, rho: float = 0.0,
                gamma: float = 1.0):
        """n accelerated PBNG iterations from iteration index l0; returns (x^{l0+n}, x^{l0+n-1})."""
        x = self._x(x).copy()
        xm1 = self._x(xm1).copy()
        fails = self._L.orc_iterate(self._h, _p(x), _p(xm1), int(l0), int(n), ACCEL[accel], float(omega),
                                  float(rho), float(gamma))
        if fails:
            raise RuntimeError(f"{fails} nodal solves failed")
        return x, xm1

    def run(self, iterations=None, x0=None):
        """The scene's full run from x^0 (x^{-1} = x^0): returns x^L."""
        sc = self.scene
        L = sc.iterations if iterations is None else iterations
        x = sc.x0[self.sample] if x0 is None else x0
        xL, _ = self.iterate(x, x, 0, L, sc.accel, sc.omega, sc.rho, sc.gamma)
        return xL
