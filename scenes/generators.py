"""Seeded synthetic scenes shaped like the paper's workloads (BASELINE.json `configs`).

Holds no PBNG arithmetic: vertex lattices, tet connectivity, Dirichlet sets/targets, initial states,
material draws and weak-constraint records only.  Readings of the configs follow SURVEY.md §8(c)
"Config readings" and are listed in DESIGN.md "Input recipe".

Numbering conventions (they are part of the parity contract because the greedy colouring of
PAPER.md:702-705 visits vertices in ascending index):
  * grid vertex (i, j, k) of an (nx, ny, nz)-cell grid has index i + (nx+1)*(j + (ny+1)*k)  (x fastest);
  * cells are emitted in the same x-fastest order;
  * Kuhn split: per cell, one tet per axis permutation (a, b, c) in lexicographic order
    (0,1,2),(0,2,1),(1,0,2),(1,2,0),(2,0,1),(2,1,0): vertices v0, v0+e_a, v0+e_a+e_b, v0+e_a+e_b+e_c,
    with the last two swapped for odd permutations so that every rest tet is positively oriented
    (det[e_a, e_a+e_b, e_a+e_b+e_c] = sign of the permutation);
  * multi-block meshes are block-major.
Random draws use numpy Generator(PCG64(SEED_BASE + config_index)).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Optional

import numpy as np

SEED_BASE = 230609021

# weak-constraint record (SURVEY.md §8(b) pbng_weak_constraint): side 0 = up to 4 weighted nodes,
# side 1 = up to 4 weighted nodes, or (n1 == 0) a fixed anchor point.  K symmetric: xx,yy,zz,xy,yz,xz.
WC_FIELDS = ("n0", "n1", "idx0", "idx1", "w0", "w1", "anchor", "K")


@dataclass
class Scene:
    name: str
    X: np.ndarray                 # (nv, 3) float64 rest positions
    tets: np.ndarray              # (nt, 4) int32
    model: str                    # "nh" (PAPER.md:291 eq:nh) | "fcr" (PAPER.md:285 eq:cor)
    E: np.ndarray                 # (nt,) float64 Young's modulus per tet (or shape (1,) for uniform)
    nu: float
    density: float
    gravity: np.ndarray           # (3,)
    pinned: np.ndarray            # (npin,) int32, ascending
    targets: np.ndarray           # (n_batch, npin, 3) float64
    x0: np.ndarray                # (n_batch, nv, 3) float64 initial positions (pinned rows == targets)
    wc: Optional[dict] = None     # weak constraints, fields WC_FIELDS
    iterations: int = 1
    accel: str = "none"           # "none" | "sor" | "chebyshev"
    omega: float = 1.0
    rho: float = 0.0
    gamma: float = 1.0
    dtype: str = "f64"
    h: float = 1.0
    meta: dict = field(default_factory=dict)

    @property
    def n_vertices(self) -> int:
        return int(self.X.shape[0])

    @property
    def n_tets(self) -> int:
        return int(self.tets.shape[0])

    @property
    def n_batch(self) -> int:
        return int(self.x0.shape[0])

    @property
    def n_wc(self) -> int:
        return 0 if self.wc is None else int(self.wc["n0"].shape[0])

    @property
    def n_free(self) -> int:
        return self.n_vertices - int(self.pinned.shape[0])

    def bbox_diag(self) -> float:
        ext = self.X.max(axis=0) - self.X.min(axis=0)
        return float(np.sqrt((ext * ext).sum()))

    def sample(self, s: int) -> "Scene":
        """Sample s of a batched scene as a stand-alone scene (P14 batch independence)."""
        out = Scene(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        out.targets = self.targets[s:s + 1].copy()
        out.x0 = self.x0[s:s + 1].copy()
        out.name = f"{self.name}[{s}]"
        return out

    def samples(self, lo: int, hi: int) -> "Scene":
        out = Scene(**{k: getattr(self, k) for k in self.__dataclass_fields__})
        out.targets = self.targets[lo:hi].copy()
        out.x0 = self.x0[lo:hi].copy()
        out.name = f"{self.name}[{lo}:{hi}]"
        return out


def _rng(config_index: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(SEED_BASE + config_index))


def grid_vertices(nx: int, ny: int, nz: int, h: float, origin=(0.0, 0.0, 0.0)) -> np.ndarray:
    nv = (nx + 1) * (ny + 1) * (nz + 1)
    idx = np.arange(nv, dtype=np.int64)
    i = idx % (nx + 1)
    j = (idx // (nx + 1)) % (ny + 1)
    k = idx // ((nx + 1) * (ny + 1))
    X = np.stack([i, j, k], axis=1).astype(np.float64) * h
    return X + np.asarray(origin, dtype=np.float64)


_PERMS = ((0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0))
_PERM_ODD = (False, True, True, False, False, True)


def kuhn_grid(nx: int, ny: int, nz: int, h: float, origin=(0.0, 0.0, 0.0), vertex_offset: int = 0):
    """6-tet (Kuhn/Freudenthal) split of an nx*ny*nz-cell grid. Returns (X, tets)."""
    X = grid_vertices(nx, ny, nz, h, origin)
    nc = nx * ny * nz
    c = np.arange(nc, dtype=np.int64)
    ci = c % nx
    cj = (c // nx) % ny
    ck = c // (nx * ny)
    v0 = ci + (nx + 1) * (cj + (ny + 1) * ck)
    step = (1, nx + 1, (nx + 1) * (ny + 1))
    tets = np.empty((nc, 6, 4), dtype=np.int64)
    for p, (a, b, cc) in enumerate(_PERMS):
        t1 = v0 + step[a]
        t2 = t1 + step[b]
        t3 = t2 + step[cc]
        if _PERM_ODD[p]:
            t2, t3 = t3, t2
        tets[:, p, 0] = v0
        tets[:, p, 1] = t1
        tets[:, p, 2] = t2
        tets[:, p, 3] = t3
    tets = (tets.reshape(-1, 4) + vertex_offset).astype(np.int32)
    return X, tets


def kuhn_grid_colouring(nx: int, ny: int, nz: int) -> np.ndarray:
    """An input for pbng_color_given / the oracle's set_colours: colour (i + j + k) mod 4 of grid vertex
    (i, j, k) of kuhn_grid(nx, ny, nz).  Two vertices of one Kuhn tet differ by a non-zero offset in {0,1}^3,
    so their index sums differ by 1, 2 or 3: no two vertices of a tet share a colour."""
    i, j, k = np.meshgrid(np.arange(nx + 1), np.arange(ny + 1), np.arange(nz + 1), indexing="ij")
    col = (i + j + k) % 4
    return np.ascontiguousarray(col.transpose(2, 1, 0).reshape(-1).astype(np.int32))  # v = i + (nx+1)(j + (ny+1) k)


def five_tet_grid(n: int, h: float = 1.0):
    """Alternating 5-tet split of an n^3-VERTEX grid ((n-1)^3 cells); the mesh family whose sizes match
    PAPER.md Table 1 (32K vertices / 150K elements = 32^3 / 31^3*5).  Cells with even
    (ci+cj+ck) use the central tet {000,110,101,011}; odd cells the complementary one, so faces conform."""
    nx = n - 1
    X = grid_vertices(nx, nx, nx, h)
    nc = nx ** 3
    c = np.arange(nc, dtype=np.int64)
    ci = c % nx
    cj = (c // nx) % nx
    ck = c // (nx * nx)
    v0 = ci + (nx + 1) * (cj + (nx + 1) * ck)
    s = (1, nx + 1, (nx + 1) ** 2)

    def corner(a, b, cc):
        return v0 + a * s[0] + b * s[1] + cc * s[2]

    even = ((ci + cj + ck) % 2) == 0
    # even cells: central {000,110,101,011}, corner tets at 100, 010, 001, 111
    even_tets = [
        (corner(0, 0, 0), corner(1, 1, 0), corner(1, 0, 1), corner(0, 1, 1)),
        (corner(1, 0, 0), corner(0, 0, 0), corner(1, 1, 0), corner(1, 0, 1)),
        (corner(0, 1, 0), corner(0, 0, 0), corner(1, 1, 0), corner(0, 1, 1)),
        (corner(0, 0, 1), corner(0, 0, 0), corner(1, 0, 1), corner(0, 1, 1)),
        (corner(1, 1, 1), corner(1, 1, 0), corner(1, 0, 1), corner(0, 1, 1)),
    ]
    # odd cells: central {100,010,001,111}, corner tets at 000, 110, 101, 011
    odd_tets = [
        (corner(1, 0, 0), corner(0, 1, 0), corner(0, 0, 1), corner(1, 1, 1)),
        (corner(0, 0, 0), corner(1, 0, 0), corner(0, 1, 0), corner(0, 0, 1)),
        (corner(1, 1, 0), corner(1, 0, 0), corner(0, 1, 0), corner(1, 1, 1)),
        (corner(1, 0, 1), corner(1, 0, 0), corner(0, 0, 1), corner(1, 1, 1)),
        (corner(0, 1, 1), corner(0, 1, 0), corner(0, 0, 1), corner(1, 1, 1)),
    ]
    tets = np.empty((nc, 5, 4), dtype=np.int64)
    for t in range(5):
        for q in range(4):
            tets[:, t, q] = np.where(even, even_tets[t][q], odd_tets[t][q])
    return X, tets.reshape(-1, 4).astype(np.int32)


def _layer(X: np.ndarray, axis: int, value: float) -> np.ndarray:
    return np.nonzero(np.isclose(X[:, axis], value, rtol=0.0, atol=1e-9))[0].astype(np.int32)


def _finish(name, X, tets, model, E, nu, density, gravity, pinned, targets, x0, **kw) -> Scene:
    pinned = np.asarray(pinned, dtype=np.int32)
    order = np.argsort(pinned, kind="stable")
    pinned = pinned[order]
    targets = np.asarray(targets, dtype=np.float64)[:, order, :]
    x0 = np.asarray(x0, dtype=np.float64)
    x0[:, pinned, :] = targets
    E = np.atleast_1d(np.asarray(E, dtype=np.float64))
    return Scene(name=name, X=X, tets=tets, model=model, E=E, nu=float(nu), density=float(density),
                 gravity=np.asarray(gravity, dtype=np.float64), pinned=pinned, targets=targets,
                 x0=x0, **kw)


def config1_tiny_cube(n: int = 4, dtype: str = "f64", iterations: int = 200) -> Scene:
    """Config 1: 4^3-cell unit cube (h = 0.25), NH, E=1e5, nu=0.3, rho=1000, g=-9.8 z.  Bottom layer
    pinned at rest, top layer at rest + (0,0,0.25); free vertices start at X + U(-0.1h, 0.1h)^3."""
    h = 1.0 / n
    X, tets = kuhn_grid(n, n, n, h)
    rng = _rng(1)
    noise = rng.uniform(-0.1 * h, 0.1 * h, size=X.shape)
    bottom = _layer(X, 2, 0.0)
    top = _layer(X, 2, 1.0)
    pinned = np.concatenate([bottom, top])
    targets = np.concatenate([X[bottom], X[top] + np.array([0.0, 0.0, 0.25])])[None]
    x0 = (X + noise)[None].copy()
    return _finish("config1_tiny_cube", X, tets, "nh", 1e5, 0.3, 1000.0, (0.0, 0.0, -9.8), pinned,
                   targets, x0, iterations=iterations, accel="none", omega=1.0, dtype=dtype, h=h)


def config2_twisted_bar(nx: int = 32, nz: int = 128, dtype: str = "f32", iterations: int = 100,
                        gamma: float = 1.7, noise_seed: int = 0) -> Scene:
    """Config 2: 32x32x128-cell bar 0.25 x 0.25 x 1 (h = 1/128), FCR, E=1e6, nu=0.45.  z=0 pinned at
    rest, z=1 layer rotated +90 deg about the bar axis through (0.125, 0.125).  Free vertices start at
    rest + U(+-0.05h).  Chebyshev rho=0.95, gamma = 1.7."""
    h = 1.0 / nz
    X, tets = kuhn_grid(nx, nx, nz, h)
    length = nz * h
    # noise_seed > 0 draws the noise from another stream, PCG64(SEED_BASE + 2 + 1000 noise_seed) (margin checks)
    rng = _rng(2 + 1000 * noise_seed)
    noise = rng.uniform(-0.05 * h, 0.05 * h, size=X.shape)
    bottom = _layer(X, 2, 0.0)
    top = _layer(X, 2, length)
    cx = cy = 0.5 * nx * h
    Xt = X[top]
    # +90 deg about +z: (dx, dy) -> (-dy, dx)  (exact rotation matrix [[0,-1],[1,0]])
    rot = np.stack([cx - (Xt[:, 1] - cy), cy + (Xt[:, 0] - cx), Xt[:, 2]], axis=1)
    pinned = np.concatenate([bottom, top])
    targets = np.concatenate([X[bottom], rot])[None]
    x0 = (X + noise)[None].copy()
    return _finish("config2_twisted_bar", X, tets, "fcr", 1e6, 0.45, 1000.0, (0.0, 0.0, 0.0), pinned,
                   targets, x0, iterations=iterations, accel="chebyshev", rho=0.95, gamma=gamma,
                   dtype=dtype, h=h)


def config3_hetero_cube(n: int = 128, dtype: str = "f32", iterations: int = 50) -> Scene:
    """Config 3: n^3-cell unit cube (h = 1/n), NH, per-tet E ~ lognormal(ln 1e5, 0.5) drawn in tet order,
    nu=0.4.  Bottom pinned at rest, top pinned at z = 0.7; initial state = affine compression z -> 0.7 z.
    SOR omega=1.5."""
    h = 1.0 / n
    X, tets = kuhn_grid(n, n, n, h)
    rng = _rng(3)
    E = rng.lognormal(mean=np.log(1e5), sigma=0.5, size=tets.shape[0])
    bottom = _layer(X, 2, 0.0)
    top = _layer(X, 2, 1.0)
    pinned = np.concatenate([bottom, top])
    tt = X[top].copy()
    tt[:, 2] = 0.7
    targets = np.concatenate([X[bottom], tt])[None]
    x0 = X.copy()
    x0[:, 2] *= 0.7
    return _finish("config3_hetero_cube", X, tets, "nh", E, 0.4, 1000.0, (0.0, 0.0, 0.0), pinned,
                   targets, x0[None], iterations=iterations, accel="sor", omega=1.5, dtype=dtype, h=h)


def config4_batched(n_samples: int = 4096, n: int = 16, dtype: str = "f32", iterations: int = 100,
                    gamma: float = 1.7) -> Scene:
    """Config 4: n_samples independent copies of an n^3-cell unit cube (h = 1/n), NH, E=1e5, nu=0.3.
    Per sample s (drawn in sample order): u_s ~ U[0,1), n_s ~ N(0, I_3) normalised; top-layer
    displacement d_s = 0.3 u_s^(1/3) n_s (uniform in the ball of radius 0.3 x side).  Bottom pinned at
    rest, top at rest + d_s, initial state X + z d_s.  Chebyshev rho=0.95.  The draws always cover 4096
    samples so that any prefix equals the same samples of the full batch."""
    h = 1.0 / n
    X, tets = kuhn_grid(n, n, n, h)
    rng = _rng(4)
    total = max(4096, n_samples)
    u = rng.random(total)
    g = rng.standard_normal((total, 3))
    nhat = g / np.linalg.norm(g, axis=1, keepdims=True)
    d = (0.3 * np.cbrt(u))[:, None] * nhat
    d = d[:n_samples]
    bottom = _layer(X, 2, 0.0)
    top = _layer(X, 2, 1.0)
    pinned = np.concatenate([bottom, top])
    targets = np.empty((n_samples, pinned.shape[0], 3))
    targets[:, :bottom.shape[0]] = X[bottom][None]
    targets[:, bottom.shape[0]:] = X[top][None] + d[:, None, :]
    x0 = X[None] + X[None, :, 2:3] * d[:, None, :]
    return _finish("config4_batched", X, tets, "nh", 1e5, 0.3, 1000.0, (0.0, 0.0, 0.0), pinned, targets,
                   x0, iterations=iterations, accel="chebyshev", rho=0.95, gamma=gamma, dtype=dtype,
                   h=h, meta={"displacement": d})


def _empty_wc(n: int) -> dict:
    return {
        "n0": np.zeros(n, np.int32), "n1": np.zeros(n, np.int32),
        "idx0": np.zeros((n, 4), np.int32), "idx1": np.zeros((n, 4), np.int32),
        "w0": np.zeros((n, 4)), "w1": np.zeros((n, 4)),
        "anchor": np.zeros((n, 3)), "K": np.zeros((n, 6)),
    }


def concat_wc(parts) -> Optional[dict]:
    parts = [p for p in parts if p is not None and p["n0"].shape[0] > 0]
    if not parts:
        return None
    return {k: np.concatenate([p[k] for p in parts]) for k in WC_FIELDS}


def config5_muscle_stack(n_blocks: int = 8, n: int = 48, dtype: str = "f32", iterations: int = 130) -> Scene:
    """Config 5: n_blocks stacked n^3-cell blocks of side 0.1 m (h = 0.1/n), block-major numbering, faces
    coincident.  FCR, E=5e4, nu=0.45, rho=1000, g=-9.8 z.  Top face of the top block pinned at rest.
    Springs (K = 1e4 I, zero rest length): for each interface, each lower-block top-face vertex is bound
    with probability 0.5 (one U[0,1) draw per vertex, interfaces ascending, vertices ascending) to the
    coincident upper-block vertex.  Contacts: one per bottom-face vertex of block 0, anchor on the rigid
    plane z = 0.01, K = 1e5 z z^T.  Free vertices start at rest + U(+-0.05h).  No acceleration."""
    side = 0.1
    h = side / n
    Xs, Ts = [], []
    nvb = (n + 1) ** 3
    for b in range(n_blocks):
        Xb, Tb = kuhn_grid(n, n, n, h, origin=(0.0, 0.0, b * side), vertex_offset=b * nvb)
        Xs.append(Xb)
        Ts.append(Tb)
    X = np.concatenate(Xs)
    tets = np.concatenate(Ts)
    rng = _rng(5)
    face = np.arange((n + 1) ** 2, dtype=np.int64)  # (i, j) in x-fastest order
    top_face_local = face + n * (n + 1) ** 2
    bot_face_local = face
    springs = []
    for b in range(n_blocks - 1):
        draw = rng.random(face.shape[0])
        sel = draw < 0.5
        lo = b * nvb + top_face_local[sel]
        hi = (b + 1) * nvb + bot_face_local[sel]
        wc = _empty_wc(lo.shape[0])
        wc["n0"][:] = 1
        wc["n1"][:] = 1
        wc["idx0"][:, 0] = lo
        wc["idx1"][:, 0] = hi
        wc["w0"][:, 0] = 1.0
        wc["w1"][:, 0] = 1.0
        wc["K"][:, 0:3] = 1e4
        springs.append(wc)
    contact = _empty_wc(face.shape[0])
    contact["n0"][:] = 1
    contact["n1"][:] = 0
    contact["idx0"][:, 0] = bot_face_local
    contact["w0"][:, 0] = 1.0
    contact["anchor"][:, 0:2] = X[bot_face_local, 0:2]
    contact["anchor"][:, 2] = 0.01
    contact["K"][:, 2] = 1e5
    wc = concat_wc(springs + [contact])
    noise = rng.uniform(-0.05 * h, 0.05 * h, size=X.shape)
    top_block = (n_blocks - 1) * nvb
    pinned = top_block + top_face_local
    targets = X[pinned][None]
    x0 = (X + noise)[None].copy()
    return _finish("config5_muscle_stack", X, tets, "fcr", 5e4, 0.45, 1000.0, (0.0, 0.0, -9.8), pinned,
                   targets, x0, wc=wc, iterations=iterations, accel="none", omega=1.0, dtype=dtype, h=h,
                   meta={"n_springs": int(sum(s["n0"].shape[0] for s in springs)),
                         "n_contacts": int(face.shape[0]), "blocks": n_blocks})


def two_blocks_colliding(n: int = 4, gap: float = 0.05, speed: float = 5.0, dt: float = 0.002,
                         dtype: str = "f64") -> Scene:
    """The paper's dynamic-constraint example ('Two Blocks Colliding'): two unit blocks
    of n^3 Kuhn cells along x with a gap, block-major numbering; the outer x faces are pinned and driven
    toward each other at `speed` (targets_at(step)), and the blocks start moving at that speed
    (meta["x_prev"] = x^{-1}).  Backward Euler with dt = 0.002, R0 = 10, E = 1000, contact
    stiffness k_n = 1e8, k_t = 0.  Not stated by the paper and read here: Neo-Hookean,
    nu = 0.3, contact thickness 0.02, the initial velocity (reading Z21)."""
    h = 1.0 / n
    XA, TA = kuhn_grid(n, n, n, h)
    nvb = XA.shape[0]
    XB, TB = kuhn_grid(n, n, n, h, origin=(1.0 + gap, 0.0, 0.0), vertex_offset=nvb)
    X = np.concatenate([XA, XB])
    tets = np.concatenate([TA, TB])
    left = np.nonzero(np.isclose(X[:, 0], 0.0))[0]
    right = np.nonzero(np.isclose(X[:, 0], 2.0 + gap))[0]
    pinned = np.concatenate([left, right]).astype(np.int32)
    targets = X[pinned][None]
    x0 = X[None].copy()
    sc = _finish("two_blocks_colliding", X, tets, "nh", 1000.0, 0.3, 10.0, (0.0, 0.0, 0.0), pinned, targets, x0,
                 wc=None, iterations=20, accel="none", omega=1.0, dtype=dtype, h=h,
                 meta={"dt": dt, "speed": speed, "thickness": 0.02, "k_n": 1e8, "k_t": 0.0, "gap": gap})
    x_prev = X.copy()
    x_prev[:nvb, 0] -= speed * dt
    x_prev[nvb:, 0] += speed * dt
    sc.meta["x_prev"] = x_prev
    return sc


def targets_at(scene: Scene, step: int) -> np.ndarray:
    """Dirichlet targets of two_blocks_colliding after `step` time steps: the left face moves by
    +speed dt per step along x, the right face by -speed dt (prescribed motion, no method arithmetic)."""
    t = scene.targets.copy()
    left = scene.X[scene.pinned, 0] < 1.0
    d = scene.meta["speed"] * scene.meta["dt"] * step
    t[:, left, 0] += d
    t[:, ~left, 0] -= d
    return t


def make_config(index: int, scale: str = "full", dtype: Optional[str] = None) -> Scene:
    """Config by BASELINE.json index (1-based).  scale="full" is BASELINE.json's size; "small" is a
    reduced copy that still spans several colours, several 32-vertex chunks and a ragged tail."""
    small = scale == "small"
    if index == 1:
        s = config1_tiny_cube()
    elif index == 2:
        s = config2_twisted_bar(nx=6, nz=24) if small else config2_twisted_bar()
    elif index == 3:
        s = config3_hetero_cube(n=14) if small else config3_hetero_cube()
    elif index == 4:
        s = config4_batched(n_samples=6, n=7) if small else config4_batched()
    elif index == 5:
        s = config5_muscle_stack(n_blocks=3, n=7) if small else config5_muscle_stack()
    else:
        raise ValueError(f"unknown config {index}")
    if dtype is not None:
        s.dtype = dtype
    return s


def spring_network(n_nodes: int = 40, n_springs: int = 90, n_anchor: int = 8, seed: int = 7) -> Scene:
    """A tet-free network of weak constraints (quadratic energy) for the P10 block-Gauss-Seidel pin:
    random single-node springs, random 2-node-weighted vs 1-node constraints, anisotropic K_c =
    k_n n n^T + k_t (t0 t0^T + t1 t1^T), and anchor constraints that fix the nullspace."""
    rng = np.random.Generator(np.random.PCG64(SEED_BASE + 100 + seed))
    X = rng.uniform(0, 1, size=(n_nodes, 3))
    m = n_springs + n_anchor
    wc = _empty_wc(m)
    for c in range(n_springs):
        a = rng.choice(n_nodes, size=3, replace=False)
        wc["n0"][c] = 1
        wc["idx0"][c, 0] = a[0]
        wc["w0"][c, 0] = 1.0
        if rng.random() < 0.5:
            wc["n1"][c] = 1
            wc["idx1"][c, 0] = a[1]
            wc["w1"][c, 0] = 1.0
        else:
            t = rng.uniform(0.1, 0.9)
            wc["n1"][c] = 2
            wc["idx1"][c, 0:2] = a[1:3]
            wc["w1"][c, 0:2] = (t, 1.0 - t)
        nrm = rng.standard_normal(3)
        nrm /= np.linalg.norm(nrm)
        kn, kt = rng.uniform(1.0, 10.0), rng.uniform(0.1, 2.0)
        Km = kt * np.eye(3) + (kn - kt) * np.outer(nrm, nrm)  # k_n nn^T + k_t (I - nn^T)
        wc["K"][c] = (Km[0, 0], Km[1, 1], Km[2, 2], Km[0, 1], Km[1, 2], Km[0, 2])
    for q in range(n_anchor):
        c = n_springs + q
        node = rng.integers(n_nodes)
        wc["n0"][c] = 1
        wc["idx0"][c, 0] = node
        wc["w0"][c, 0] = 1.0
        wc["anchor"][c] = rng.uniform(0, 1, size=3)
        wc["K"][c, 0:3] = rng.uniform(1.0, 5.0)
    # make sure every node is touched by at least one anchor-free or anchored constraint
    touched = np.zeros(n_nodes, bool)
    for c in range(m):
        touched[wc["idx0"][c, :wc["n0"][c]]] = True
        touched[wc["idx1"][c, :wc["n1"][c]]] = True
    extra = np.nonzero(~touched)[0]
    if extra.size:
        ex = _empty_wc(extra.size)
        ex["n0"][:] = 1
        ex["idx0"][:, 0] = extra
        ex["w0"][:, 0] = 1.0
        ex["anchor"][:] = X[extra]
        ex["K"][:, 0:3] = 2.0
        wc = concat_wc([wc, ex])
    x0 = (X + rng.uniform(-0.2, 0.2, size=X.shape))[None]
    tets = np.zeros((0, 4), np.int32)
    return _finish("spring_network", X, tets, "nh", 1e5, 0.3, 0.0, (0.0, 0.0, 0.0),
                   np.zeros(0, np.int32), np.zeros((1, 0, 3)), x0, wc=wc, iterations=1, h=1.0)
