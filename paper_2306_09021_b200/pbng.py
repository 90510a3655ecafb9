"""Thin ctypes binding of libpbng (include/pbng.h) -- argument marshalling only.

Every step of the PBNG path runs in the library's CUDA kernels; PyTorch supplies device memory (the
workspace tensor), the CUDA stream and the process group.  There is no CPU fallback: if libpbng.so is
missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("PBNG_LIB", os.path.join(_HERE, "libpbng.so"))  # PBNG_LIB: tuning builds only

OK = 0
STATUS = {0: "PBNG_OK", 1: "PBNG_E_INVALID_ARGUMENT", 2: "PBNG_E_INDEX_OUT_OF_RANGE", 3: "PBNG_E_DEGENERATE_ELEMENT",
          4: "PBNG_E_ISOLATED_VERTEX", 5: "PBNG_E_BAD_ORDER", 6: "PBNG_E_NOT_COLORED", 7: "PBNG_E_NONFINITE",
          8: "PBNG_E_CUDA", 9: "PBNG_E_NCCL", 10: "PBNG_E_OUT_OF_MEMORY", 11: "PBNG_E_NO_DEVICE"}
DTYPE = {"f32": 0, "f64": 1}
MODEL = {"nh": 0, "fcr": 1, "snh": 2}
ACCEL = {"none": 0, "sor": 1, "chebyshev": 2}
SCHEDULE = {"auto": 0, "colour_launches": 1, "pipelined": 2}
RECORDS = {"auto": 0, "stored": 1, "rest": 2, "table": 3}
EXPORTS = ("pbng_create_mesh", "pbng_set_material", "pbng_set_constraints", "pbng_color", "pbng_workspace_bytes",
           "pbng_bind_workspace", "pbng_set_positions", "pbng_get_positions", "pbng_iterate", "pbng_energy_residual",
           "pbng_synchronize", "pbng_query", "pbng_profile_enable", "pbng_profile_read", "pbng_destroy",
           "pbng_last_error", "pbng_version", "pbng_sweep_colour", "pbng_end_iteration", "pbng_set_partition",
           "pbng_halo_counts", "pbng_halo_vertices", "pbng_halo_pack", "pbng_halo_unpack", "pbng_test_polar",
           "pbng_set_inertia", "pbng_set_schedule", "pbng_detect_contacts", "pbng_update_constraints",
           "pbng_get_colours", "pbng_set_l2_persistence", "pbng_sweep_colour_part", "pbng_set_stream",
           "pbng_nccl_unique_id", "pbng_partition", "pbng_group_create", "pbng_group_iterate", "pbng_group_destroy",
           "pbng_set_records", "pbng_enable_peer_halo", "pbng_group_set_transport", "pbng_color_given")

WC_DTYPE = np.dtype([("n0", "<i4"), ("n1", "<i4"), ("idx0", "<i4", 4), ("idx1", "<i4", 4), ("w0", "<f8", 4),
                     ("w1", "<f8", 4), ("anchor", "<f8", 3), ("K", "<f8", 6)])
assert WC_DTYPE.itemsize == 176


class PBNGError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Info(C.Structure):
    _fields_ = [("n_vertices", C.c_int64), ("n_tets", C.c_int64), ("n_free", C.c_int64), ("n_pinned", C.c_int64),
                ("n_weak_constraints", C.c_int64), ("n_pairs", C.c_int64), ("n_pair_slots", C.c_int64),
                ("n_batch", C.c_int32), ("n_colours", C.c_int32), ("dtype", C.c_int32), ("model", C.c_int32),
                ("iteration", C.c_int64), ("kernel_launches", C.c_int64), ("sweep_bytes", C.c_double),
                ("accel_bytes", C.c_double), ("sweep_flops", C.c_double), ("n_local_vertices", C.c_int64),
                ("n_ghosts", C.c_int64), ("rank", C.c_int32), ("n_ranks", C.c_int32), ("schedule", C.c_int32),
                ("graph_replays", C.c_int32), ("records", C.c_int32)]


_lib = None


def lib():
    """Load libpbng.so (building it in-tree first if it is missing and nvcc is available)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        from . import build as _build
        _build.build()
    L = C.CDLL(LIB_PATH)
    vp, i64, i32, d = C.c_void_p, C.c_int64, C.c_int32, C.c_double
    L.pbng_create_mesh.argtypes = [vp, i64, vp, i64, i32, C.c_int, C.c_int, C.c_size_t, C.POINTER(vp),
                                   C.POINTER(i64)]
    L.pbng_set_material.argtypes = [vp, C.c_int, vp, i64, d, d, vp]
    L.pbng_set_constraints.argtypes = [vp, vp, i64, vp, vp, i64]
    L.pbng_color.argtypes = [vp, vp, vp]
    L.pbng_workspace_bytes.argtypes = [vp, C.POINTER(C.c_uint64)]
    L.pbng_bind_workspace.argtypes = [vp, vp, C.c_uint64]
    L.pbng_set_positions.argtypes = [vp, vp]
    L.pbng_get_positions.argtypes = [vp, vp]
    L.pbng_iterate.argtypes = [vp, i32, C.c_int, d, d, d]
    L.pbng_energy_residual.argtypes = [vp, vp, vp]
    L.pbng_synchronize.argtypes = [vp]
    L.pbng_query.argtypes = [vp, C.POINTER(Info)]
    L.pbng_profile_enable.argtypes = [vp, C.c_int]
    L.pbng_profile_read.argtypes = [vp, C.POINTER(d), C.POINTER(i64)]
    L.pbng_destroy.argtypes = [vp]
    L.pbng_sweep_colour.argtypes = [vp, i32, C.c_int, d, d, d]
    L.pbng_end_iteration.argtypes = [vp, C.c_int]
    L.pbng_set_partition.argtypes = [vp, vp, i32, i32]
    L.pbng_halo_counts.argtypes = [vp, i32, i32, C.POINTER(i64), C.POINTER(i64)]
    L.pbng_halo_vertices.argtypes = [vp, i32, i32, vp, vp]
    L.pbng_halo_pack.argtypes = [vp, i32, i32, i32, vp]
    L.pbng_halo_unpack.argtypes = [vp, i32, i32, i32, vp]
    L.pbng_test_polar.argtypes = [C.c_int, vp, vp, i64, C.c_int]
    L.pbng_set_inertia.argtypes = [vp, d, vp]
    L.pbng_set_schedule.argtypes = [vp, C.c_int]
    L.pbng_set_records.argtypes = [vp, C.c_int]
    L.pbng_detect_contacts.argtypes = [vp, i32, d, d, d, vp, i64, C.POINTER(i64)]
    L.pbng_update_constraints.argtypes = [vp, vp, vp, i64, C.POINTER(i64)]
    L.pbng_get_colours.argtypes = [vp, vp, C.POINTER(i32)]
    L.pbng_set_l2_persistence.argtypes = [vp, C.c_int]
    L.pbng_sweep_colour_part.argtypes = [vp, i32, i32, C.c_int, d, d, d]
    L.pbng_set_stream.argtypes = [vp, C.c_size_t]
    L.pbng_nccl_unique_id.argtypes = [vp]
    L.pbng_partition.argtypes = [vp, vp, i32, i32, vp]
    L.pbng_group_create.argtypes = [C.POINTER(vp), i32, C.POINTER(vp)]
    L.pbng_group_iterate.argtypes = [vp, i32, C.c_int, d, d, d]
    L.pbng_group_destroy.argtypes = [vp]
    L.pbng_group_set_transport.argtypes = [vp, i32]
    L.pbng_enable_peer_halo.argtypes = [vp, i32]
    L.pbng_color_given.argtypes = [vp, vp, C.POINTER(i32), C.POINTER(i64)]
    L.pbng_last_error.restype = C.c_char_p
    L.pbng_version.restype = i32
    for name in EXPORTS:
        if name not in ("pbng_last_error", "pbng_version"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(status: int):
    if status != OK:
        raise PBNGError(status, lib().pbng_last_error().decode())


def _np(a, dt):
    return np.ascontiguousarray(np.asarray(a, dtype=dt))


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def weak_constraints_array(wc: Optional[dict]) -> np.ndarray:
    if wc is None:
        return np.zeros(0, WC_DTYPE)
    n = wc["n0"].shape[0]
    out = np.zeros(n, WC_DTYPE)
    for k in ("n0", "n1", "idx0", "idx1", "w0", "w1", "anchor", "K"):
        out[k] = wc[k]
    return out


class Context:
    """One PBNG problem (or a batch of samples sharing mesh, material and colouring) on one device.

    Mirrors the C ABI: create_mesh (constructor) -> set_material -> set_constraints -> color ->
    bind_workspace -> set_positions -> iterate / energy_residual / get_positions."""

    def __init__(self, X, tets, n_batch: int = 1, dtype: str = "f32", device=0, stream=None):
        import torch
        self._torch = torch
        L = lib()
        X = _np(X, np.float64).reshape(-1, 3)
        tets = _np(tets, np.int32).reshape(-1, 4)
        self.n_vertices = X.shape[0]
        self.n_tets = tets.shape[0]
        self.n_batch = int(n_batch)
        self.dtype = dtype
        self.np_dtype = np.float32 if dtype == "f32" else np.float64
        self.torch_dtype = torch.float32 if dtype == "f32" else torch.float64
        if isinstance(device, torch.device):
            device = device.index if device.index is not None else torch.cuda.current_device()
        self.device = int(device)
        if self.device >= 0:
            if stream is None:
                stream = torch.cuda.current_stream(self.device)
            self.stream = stream
            handle = stream.cuda_stream
        else:
            self.stream = None
            handle = 0
        h = C.c_void_p()
        bad = C.c_int64(-1)
        st = L.pbng_create_mesh(_ptr(X), X.shape[0], _ptr(tets) if tets.size else None, tets.shape[0],
                                self.n_batch, DTYPE[dtype], self.device, handle, C.byref(h), C.byref(bad))
        if st != OK:
            err = PBNGError(st, L.pbng_last_error().decode())
            err.bad_index = bad.value
            raise err
        self._h = h
        self.workspace = None

    # ---------------------------------------------------------------------------------------------
    def set_material(self, model: str, E, nu: float, density: float = 0.0, gravity=(0.0, 0.0, 0.0)):
        E = _np(np.atleast_1d(E), np.float64)
        g = _np(gravity, np.float64)
        _check(lib().pbng_set_material(self._h, MODEL[model], _ptr(E), E.size, float(nu), float(density), _ptr(g)))

    def set_constraints(self, pinned, targets, wc: Optional[dict] = None):
        pinned = _np(pinned, np.int32).reshape(-1)
        targets = _np(targets, np.float64).reshape(-1)
        w = weak_constraints_array(wc)
        _check(lib().pbng_set_constraints(self._h, _ptr(pinned) if pinned.size else None, pinned.size,
                                          _ptr(targets) if targets.size else None, _ptr(w) if w.size else None,
                                          w.size))

    def color(self, colours=None):
        """pbng_color (greedy), or pbng_color_given with the caller's node colouring."""
        n = C.c_int32()
        if colours is not None:
            out = _np(colours, np.int32).reshape(-1).copy()
            if out.shape[0] != self.n_vertices:
                raise ValueError("colours: one entry per vertex")
            bad = C.c_int64(-1)
            _check(lib().pbng_color_given(self._h, _ptr(out), C.byref(n), C.byref(bad)))
            self.colours, self.n_colours = out, n.value
            return out, n.value
        out = np.empty(self.n_vertices, np.int32)
        _check(lib().pbng_color(self._h, _ptr(out), C.byref(n)))
        self.colours, self.n_colours = out, n.value
        return out, n.value

    def workspace_bytes(self) -> int:
        b = C.c_uint64()
        _check(lib().pbng_workspace_bytes(self._h, C.byref(b)))
        return b.value

    def bind_workspace(self, tensor=None):
        torch = self._torch
        nbytes = self.workspace_bytes()
        if tensor is None:
            tensor = torch.empty(nbytes + 256, dtype=torch.uint8, device=f"cuda:{self.device}")
        ptr = tensor.data_ptr()
        pad = (-ptr) % 256
        _check(lib().pbng_bind_workspace(self._h, ptr + pad, tensor.numel() - pad))
        self.workspace = tensor
        return tensor

    # ---------------------------------------------------------------------------------------------
    def _shape(self):
        return (self.n_batch, self.n_vertices, 3)

    def set_positions(self, x):
        """x: torch tensor (device or pinned/pageable host) or numpy array, [n_batch, n_vertices, 3]."""
        torch = self._torch
        if isinstance(x, np.ndarray):
            x = torch.from_numpy(_np(x, self.np_dtype))
        if x.dtype != self.torch_dtype or not x.is_contiguous():
            x = x.to(self.torch_dtype).contiguous()
        if x.numel() != self.n_batch * self.n_vertices * 3:
            raise ValueError(f"positions must have {self._shape()} entries")
        self._x_keep = x
        _check(lib().pbng_set_positions(self._h, x.data_ptr()))

    def set_inertia(self, dt: float, xtilde=None):
        """Backward Euler: dt > 0 with xtilde = 2 x^n - x^{n-1} ([n_batch, n_vertices, 3]); dt = 0 -> quasistatic."""
        torch = self._torch
        if dt == 0 or xtilde is None:
            _check(lib().pbng_set_inertia(self._h, float(dt), None))
            self._inertia_dt = 0.0
            return
        if isinstance(xtilde, np.ndarray):
            xtilde = torch.from_numpy(_np(xtilde, self.np_dtype))
        if xtilde.dtype != self.torch_dtype or not xtilde.is_contiguous():
            xtilde = xtilde.to(self.torch_dtype).contiguous()
        self._xt_keep = xtilde
        _check(lib().pbng_set_inertia(self._h, float(dt), xtilde.data_ptr()))
        self._inertia_dt = float(dt)

    def get_positions(self, out=None):
        torch = self._torch
        if out is None:
            out = torch.empty(self._shape(), dtype=self.torch_dtype, device=f"cuda:{self.device}")
        if out.dtype != self.torch_dtype or not out.is_contiguous() or out.numel() != self.n_batch * self.n_vertices * 3:
            raise ValueError("out must be a contiguous tensor of the context dtype and shape")
        _check(lib().pbng_get_positions(self._h, out.data_ptr()))
        return out

    def iterate(self, n: int, accel: str = "none", omega: float = 1.0, rho: float = 0.0, gamma: float = 1.0):
        _check(lib().pbng_iterate(self._h, int(n), ACCEL[accel], float(omega), float(rho), float(gamma)))

    def set_l2_persistence(self, enable: bool = True):
        """Keep the gathered position buffers resident in L2 (pbng_set_l2_persistence)."""
        _check(lib().pbng_set_l2_persistence(self._h, int(bool(enable))))

    def set_schedule(self, schedule: str = "auto"):
        """'colour_launches' (one launch per colour pass), 'pipelined' (persistent dataflow launch) or 'auto'."""
        _check(lib().pbng_set_schedule(self._h, SCHEDULE[schedule]))

    def set_records(self, records: str = "auto"):
        """Pair-record layout built by color(): 'stored' rest data, 'rest' (recomputed from rest positions),
        'table' (distinct rest tuples in a table) or 'auto' (pbng_set_records; call before color())."""
        _check(lib().pbng_set_records(self._h, RECORDS[records]))

    # ---- dynamic weak constraints ----------------------------------------------------------------
    def detect_contacts(self, thickness: float, k_n: float, k_t: float = 0.0, sample: int = 0) -> np.ndarray:
        """Contact weak constraints at the current positions (pbng_detect_contacts) as a WC_DTYPE array."""
        cap = max(64, self.n_vertices)
        while True:
            out = np.zeros(cap, WC_DTYPE)
            n = C.c_int64()
            st = lib().pbng_detect_contacts(self._h, int(sample), float(thickness), float(k_n), float(k_t), _ptr(out),
                                            cap, C.byref(n))
            if st == 10 and n.value > cap:
                cap = n.value
                continue
            _check(st)
            return out[:n.value].copy()

    def update_constraints(self, wc, targets=None) -> int:
        """Replace the weak constraints (dict or WC_DTYPE array) with incremental recolouring
        (pbng_update_constraints); grows the workspace if the new layout needs it.  Returns the number of
        recoloured nodes."""
        w = wc if isinstance(wc, np.ndarray) and wc.dtype == WC_DTYPE else weak_constraints_array(wc)
        w = np.ascontiguousarray(w)
        t = None if targets is None else _np(targets, np.float64).reshape(-1)
        saved = None  # the iterate, kept for the re-bind when the new layout outgrows the workspace
        if self.device >= 0 and self.workspace is not None:
            try:
                saved = self.get_positions()
            except PBNGError:  # positions never set: nothing to keep
                saved = None
        n = C.c_int64()
        st = lib().pbng_update_constraints(self._h, _ptr(t) if t is not None else None, _ptr(w) if w.size else None,
                                           w.size, C.byref(n))
        if st == 10 and saved is not None and self.workspace_bytes() > 0:
            nbytes = self.workspace_bytes()
            self.bind_workspace(self._torch.empty(int(nbytes * 1.25) + 256, dtype=self._torch.uint8,
                                                  device=f"cuda:{self.device}"))
            self.set_positions(saved)
            # the library carries the backward-Euler target over a re-layout, but not across this re-bind:
            # set it again from the last set_inertia
            if getattr(self, "_inertia_dt", 0.0) > 0.0:
                _check(lib().pbng_set_inertia(self._h, self._inertia_dt, self._xt_keep.data_ptr()))
            self.colours, self.n_colours = self.get_colours()
            return n.value
        _check(st)
        self.colours, self.n_colours = self.get_colours()
        return n.value

    def get_colours(self):
        """The colouring in use (after incremental updates): (colour per vertex, number of colours)."""
        out = np.empty(self.n_vertices, np.int32)
        n = C.c_int32()
        _check(lib().pbng_get_colours(self._h, _ptr(out), C.byref(n)))
        return out, n.value

    def energy_residual(self):
        e = np.empty(self.n_batch)
        r = np.empty(self.n_batch)
        _check(lib().pbng_energy_residual(self._h, _ptr(e), _ptr(r)))
        return e, r

    def synchronize(self):
        _check(lib().pbng_synchronize(self._h))

    def query(self) -> dict:
        info = Info()
        _check(lib().pbng_query(self._h, C.byref(info)))
        return {k: getattr(info, k) for k, _ in Info._fields_}

    def profile_enable(self, mode: int = 2):
        """mode 1: events around every sweep launch; 2: around each iterate call's sweep launches; 0: off."""
        _check(lib().pbng_profile_enable(self._h, int(mode)))

    def profile_read(self):
        ms = C.c_double()
        n = C.c_int64()
        _check(lib().pbng_profile_read(self._h, C.byref(ms), C.byref(n)))
        return ms.value, n.value

    # ---- colour-by-colour iteration and domain decomposition -------------------------------------
    def sweep_colour(self, colour: int, accel: str = "none", omega: float = 1.0, rho: float = 0.0, gamma: float = 1.0):
        _check(lib().pbng_sweep_colour(self._h, int(colour), ACCEL[accel], float(omega), float(rho), float(gamma)))

    def sweep_colour_part(self, colour: int, part: int, accel: str = "none", omega: float = 1.0, rho: float = 0.0,
                          gamma: float = 1.0):
        """part 1: the colour's halo-send vertices; 2: the rest; 0: both (pbng_sweep_colour_part)."""
        _check(lib().pbng_sweep_colour_part(self._h, int(colour), int(part), ACCEL[accel], float(omega), float(rho),
                                            float(gamma)))

    def set_stream(self, stream):
        """Issue this context's later calls on `stream` (a torch.cuda.Stream)."""
        self.stream = stream
        _check(lib().pbng_set_stream(self._h, stream.cuda_stream))

    def end_iteration(self, accel: str = "none"):
        _check(lib().pbng_end_iteration(self._h, ACCEL[accel]))

    def set_partition(self, owner, rank: int, n_ranks: int):
        owner = _np(owner, np.int32).reshape(-1) if owner is not None else None
        self._owner = owner
        _check(lib().pbng_set_partition(self._h, _ptr(owner) if owner is not None else None, int(rank), int(n_ranks)))

    def partition(self, owner, rank: int, n_ranks: int, nccl_id: Optional[bytes] = None):
        """pbng_partition: set_partition + the library's NCCL communicator (nccl_id: the 128-byte id from
        nccl_unique_id(), identical on every rank; collective).  pbng_iterate then exchanges the halos itself
        and pbng_energy_residual returns global values."""
        owner = _np(owner, np.int32).reshape(-1) if owner is not None else None
        self._owner = owner
        idb = None if nccl_id is None else C.create_string_buffer(bytes(nccl_id), 128)
        _check(lib().pbng_partition(self._h, _ptr(owner) if owner is not None else None, int(rank), int(n_ranks), idb))

    def enable_peer_halo(self, enable: bool = True):
        """pbng_enable_peer_halo: halo rows stored straight into the neighbours' ghost rows over peer memory
        (collective over the partition's communicator; after color + bind)."""
        _check(lib().pbng_enable_peer_halo(self._h, 1 if enable else 0))

    def halo_counts(self, colour: int, peer: int):
        ns, nr = C.c_int64(), C.c_int64()
        _check(lib().pbng_halo_counts(self._h, int(colour), int(peer), C.byref(ns), C.byref(nr)))
        return ns.value, nr.value

    def halo_vertices(self, colour: int, peer: int):
        ns, nr = self.halo_counts(colour, peer)
        snd = np.empty(max(ns, 1), np.int32)
        rcv = np.empty(max(nr, 1), np.int32)
        _check(lib().pbng_halo_vertices(self._h, int(colour), int(peer), _ptr(snd), _ptr(rcv)))
        return snd[:ns], rcv[:nr]

    def halo_pack(self, colour: int, peer: int, n_fields: int, buf):
        _check(lib().pbng_halo_pack(self._h, int(colour), int(peer), int(n_fields), buf.data_ptr()))

    def halo_unpack(self, colour: int, peer: int, n_fields: int, buf):
        _check(lib().pbng_halo_unpack(self._h, int(colour), int(peer), int(n_fields), buf.data_ptr()))

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.pbng_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def nccl_unique_id() -> bytes:
    """pbng_nccl_unique_id: a fresh 128-byte NCCL unique id (call on one rank, share the bytes)."""
    buf = C.create_string_buffer(128)
    _check(lib().pbng_nccl_unique_id(buf))
    return buf.raw


class Group:
    """pbng_group_*: the in-process loopback transport over rank contexts ctxs[r] = rank r (one device)."""

    def __init__(self, ctxs):
        self.ctxs = list(ctxs)
        arr = (C.c_void_p * len(self.ctxs))(*[c._h for c in self.ctxs])
        h = C.c_void_p()
        _check(lib().pbng_group_create(arr, len(self.ctxs), C.byref(h)))
        self._h = h

    def set_transport(self, transport: str):
        """pbng_group_set_transport: "copies" (staged device-to-device copies) or "peer" (peer stores + flags)."""
        _check(lib().pbng_group_set_transport(self._h, {"copies": 0, "peer": 1}[transport]))

    def iterate(self, n: int, accel: str = "none", omega: float = 1.0, rho: float = 0.0, gamma: float = 1.0):
        _check(lib().pbng_group_iterate(self._h, int(n), ACCEL[accel], float(omega), float(rho), float(gamma)))

    def close(self):
        h = getattr(self, "_h", None)
        if h is not None and _lib is not None:
            _lib.pbng_group_destroy(h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def test_polar(F, dtype: str = "f32", device: int = 0) -> np.ndarray:
    """Test hook: the device polar rotation R(F) (fixed-corotated model) of a batch of 3x3 matrices."""
    F = _np(F, np.float64).reshape(-1, 3, 3)
    R = np.empty_like(F)
    _check(lib().pbng_test_polar(DTYPE[dtype], _ptr(F), _ptr(R), F.shape[0], int(device)))
    return R


def context_from_scene(scene, device=0, dtype: Optional[str] = None, stream=None, bind: bool = True,
                       set_positions: bool = True, partition=None, l2_persist: bool = True,
                       records: str = "auto", colours=None) -> Context:
    """Build, colour, bind and initialise a Context for a scenes.Scene (all samples of its batch).
    partition = (owner, rank, n_ranks) builds the rank-local context of a domain decomposition (driven by
    a Group or the colour-by-colour calls); (owner, rank, n_ranks, nccl_id) attaches the library's NCCL
    halo transport (pbng_partition);
    l2_persist keeps the gathered position buffers L2-resident (pbng_set_l2_persistence);
    records chooses the pair-record layout (pbng_set_records)."""
    ctx = Context(scene.X, scene.tets, n_batch=scene.n_batch, dtype=dtype or scene.dtype, device=device, stream=stream)
    ctx.set_material(scene.model, scene.E, scene.nu, scene.density, scene.gravity)
    ctx.set_constraints(scene.pinned, scene.targets, scene.wc)
    if records != "auto":
        ctx.set_records(records)
    if partition is not None:
        if len(partition) == 4:
            ctx.partition(*partition)
        else:
            ctx.set_partition(*partition)
    ctx.colours, ctx.n_colours = ctx.color(colours)
    if bind and ctx.device >= 0:
        ctx.bind_workspace()
        if l2_persist:
            ctx.set_l2_persistence(True)
        if set_positions:
            ctx.set_positions(np.asarray(scene.x0))
    return ctx
