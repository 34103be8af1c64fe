"""Thin ctypes binding of include/sldg.h (argument marshalling only).

Every step of the SLDG path runs in libsldg.so (sm_100a CUDA kernels); this module only
converts Python/numpy arguments to C and raises on non-OK status.  There is no CPU fallback:
if the shared library is missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes
import os
import weakref

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libsldg.so")

SLDG_OK, SLDG_EINVAL, SLDG_ENOMEM, SLDG_ECUDA, SLDG_ENCCL, SLDG_ENOTSUP = range(6)
SLDG_MIXED, SLDG_FP64 = 0, 1
MAX_DIM = 6
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ENOMEM", 3: "ECUDA", 4: "ENCCL", 5: "ENOTSUP"}

# every symbol include/sldg.h declares
EXPORTS = [
    "sldg_create", "sldg_create_ex", "sldg_destroy", "sldg_set_coeffs", "sldg_get_coeffs", "sldg_advect",
    "sldg_advect_device", "sldg_advect_device_bounded", "sldg_advect_pair", "sldg_advect_pair_device",
    "sldg_timeline", "sldg_mass", "sldg_shard_info", "sldg_sync", "sldg_set_stream",
    "sldg_get_stream", "sldg_memory_bytes", "sldg_last_error", "sldg_fill_random",
    "sldg_fill_separable", "sldg_profile", "sldg_kernel_time", "sldg_launch_count",
    "sldg_nccl_unique_id", "sldg_halo_widths", "sldg_halo_plan", "sldg_layer_owner",
    "sldg_sweep_kernel", "sldg_vp_create", "sldg_vp_destroy", "sldg_vp_density", "sldg_vp_field",
    "sldg_vp_step", "sldg_transpose_plan", "sldg_transpose_count", "sldg_advect_vnodes",
    "sldg_advect_vnodes_device", "sldg_vp_set_nodal", "sldg_graph_begin", "sldg_graph_end",
    "sldg_graph_launch", "sldg_graph_destroy", "sldg_peer_halo_check",
]


class SldgError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class GridDesc(ctypes.Structure):
    _fields_ = [("ndim", ctypes.c_int), ("cells", ctypes.c_int64 * MAX_DIM)]


class Domain(ctypes.Structure):
    _fields_ = [("lo", ctypes.c_double * MAX_DIM), ("hi", ctypes.c_double * MAX_DIM)]


class Dist(ctypes.Structure):
    _fields_ = [("rank", ctypes.c_int), ("world", ctypes.c_int), ("nccl_unique_id", ctypes.c_void_p),
                ("nccl_comm", ctypes.c_void_p), ("max_halo", ctypes.c_int), ("flags", ctypes.c_int)]

SLDG_DIST_FORCE_HALO = 1
SLDG_DIST_FORCE_TRANSPOSE = 2
SLDG_DIST_NCCL_SELF = 4
SLDG_DIST_PEER_HALO = 8
SLDG_DIST_PEER_VIA_FD = 16


_lib = None


def lib():
    """Load libsldg.so (raises if it has not been built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    i64, u32, dp, vp = ctypes.c_int64, ctypes.c_uint32, ctypes.POINTER(ctypes.c_double), ctypes.c_void_p
    i64p = ctypes.POINTER(ctypes.c_int64)
    sig = {
        "sldg_create": [ctypes.POINTER(GridDesc), ctypes.c_int, ctypes.POINTER(Domain), ctypes.c_int,
                        ctypes.POINTER(Dist), ctypes.POINTER(vp)],
        "sldg_create_ex": [ctypes.POINTER(GridDesc), ctypes.c_int, ctypes.POINTER(Domain), ctypes.c_int,
                           ctypes.POINTER(Dist), ctypes.POINTER(vp)],
        "sldg_destroy": [vp],
        "sldg_set_coeffs": [vp, dp, i64, i64],
        "sldg_get_coeffs": [vp, dp, i64, i64],
        "sldg_advect": [vp, ctypes.c_int, ctypes.c_double, dp, u32],
        "sldg_advect_device": [vp, ctypes.c_int, ctypes.c_double, vp, u32],
        "sldg_advect_device_bounded": [vp, ctypes.c_int, ctypes.c_double, vp, u32, ctypes.c_double,
                                       ctypes.c_double],
        "sldg_timeline": [vp, dp, ctypes.POINTER(ctypes.c_int), ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                          ctypes.c_int],
        "sldg_advect_pair": [vp, ctypes.c_double, dp, u32, ctypes.c_double, dp, u32],
        "sldg_advect_pair_device": [vp, ctypes.c_double, vp, u32, ctypes.c_double, vp, u32],
        "sldg_mass": [vp, dp],
        "sldg_shard_info": [vp, i64p, i64p],
        "sldg_sync": [vp],
        "sldg_set_stream": [vp, vp],
        "sldg_get_stream": [vp, ctypes.POINTER(vp)],
        "sldg_fill_random": [vp, ctypes.c_uint64],
        "sldg_fill_separable": [vp, ctypes.c_int, dp],
        "sldg_profile": [vp, ctypes.c_int],
        "sldg_kernel_time": [vp, ctypes.c_int, dp, i64p, dp, ctypes.c_int],
        "sldg_nccl_unique_id": [vp],
        "sldg_halo_widths": [i64, i64, i64p, i64p],
        "sldg_halo_plan": [i64, ctypes.c_int, ctypes.c_int, i64, i64, i64, i64p, i64, i64p],
        "sldg_layer_owner": [i64, ctypes.c_int, i64, ctypes.POINTER(ctypes.c_int), i64p],
        "sldg_transpose_plan": [i64, i64, ctypes.c_int, ctypes.c_int, i64p],
        "sldg_transpose_count": [vp, i64p],
        "sldg_peer_halo_check": [vp, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, i64],
        "sldg_advect_vnodes": [vp, ctypes.c_int, ctypes.c_int, dp],
        "sldg_advect_vnodes_device": [vp, ctypes.c_int, ctypes.c_int, vp],
        "sldg_vp_create": [vp, ctypes.c_int, ctypes.POINTER(vp)],
        "sldg_vp_destroy": [vp],
        "sldg_vp_density": [vp, dp],
        "sldg_vp_field": [vp, dp, dp, dp, dp],
        "sldg_vp_step": [vp, ctypes.c_double, dp],
        "sldg_vp_set_nodal": [vp, ctypes.c_int],
        "sldg_graph_begin": [vp],
        "sldg_graph_end": [vp, ctypes.POINTER(vp)],
        "sldg_graph_launch": [vp],
        "sldg_graph_destroy": [vp],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = ctypes.c_int
    L.sldg_memory_bytes.argtypes = [vp]
    L.sldg_memory_bytes.restype = ctypes.c_size_t
    L.sldg_last_error.argtypes = []
    L.sldg_last_error.restype = ctypes.c_char_p
    L.sldg_launch_count.argtypes = [vp]
    L.sldg_launch_count.restype = ctypes.c_int64
    L.sldg_sweep_kernel.argtypes = [vp, ctypes.c_int]
    L.sldg_sweep_kernel.restype = ctypes.c_char_p
    _lib = L
    return L


def _check(st: int):
    if st != SLDG_OK:
        raise SldgError(st, lib().sldg_last_error().decode(errors="replace"))


def _dp(a: np.ndarray):
    return a.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def nccl_unique_id() -> bytes:
    buf = ctypes.create_string_buffer(128)
    _check(lib().sldg_nccl_unique_id(buf))
    return buf.raw


def halo_widths(imin: int, imax: int):
    a, b = ctypes.c_int64(), ctypes.c_int64()
    _check(lib().sldg_halo_widths(imin, imax, ctypes.byref(a), ctypes.byref(b)))
    return a.value, b.value


def halo_plan(n: int, world: int, rank: int, pad: int, left: int, right: int):
    """[(kind, peer, slot, src)] -- the transfer plan sldg_advect runs for a sharded sweep."""
    cnt = ctypes.c_int64()
    _check(lib().sldg_halo_plan(n, world, rank, pad, left, right, None, 0, ctypes.byref(cnt)))
    buf = (ctypes.c_int64 * max(1, 4 * cnt.value))()
    _check(lib().sldg_halo_plan(n, world, rank, pad, left, right, buf, cnt.value, ctypes.byref(cnt)))
    return [tuple(buf[4 * i:4 * i + 4]) for i in range(cnt.value)]


def transpose_plan(n_outer: int, n_slab: int, world: int, rank: int):
    """[(send_layer_first, send_layer_count, send_slab_first, send_slab_count, recv_layer_first,
    recv_layer_count, recv_slab_first, recv_slab_count)] per peer -- the transpose path's plan."""
    buf = (ctypes.c_int64 * (8 * world))()
    _check(lib().sldg_transpose_plan(n_outer, n_slab, world, rank, buf))
    return [tuple(buf[8 * p:8 * p + 8]) for p in range(world)]


def layer_owner(n: int, world: int, layer: int):
    o, loc = ctypes.c_int(), ctypes.c_int64()
    _check(lib().sldg_layer_owner(n, world, layer, ctypes.byref(o), ctypes.byref(loc)))
    return o.value, loc.value


def peer_halo_check(cells, k: int, precision: str, world: int, pad: int, gran: int = 2 << 20):
    """sldg_peer_halo_check: None if SLDG_DIST_PEER_HALO accepts the layout, else the reason."""
    cells = [int(c) for c in cells]
    gd = GridDesc(len(cells), (ctypes.c_int64 * MAX_DIM)(*(cells + [1] * (MAX_DIM - len(cells)))))
    prec = {"mixed": SLDG_MIXED, "fp64": SLDG_FP64}[precision]
    st = lib().sldg_peer_halo_check(ctypes.byref(gd), int(k), prec, int(world), int(pad), int(gran))
    if st == 0:
        return None
    if st == 5:
        return lib().sldg_last_error().decode()
    _check(st)


class Grid:
    """Owns one sldg_grid handle.  Method names follow the C ABI (sldg_<name>)."""

    def __init__(self, cells, k: int, lo=None, hi=None, precision: str = "mixed",
                 rank: int = 0, world: int = 1, unique_id: bytes | None = None, max_halo: int = 0,
                 force_halo: bool = False, force_transpose: bool = False, nccl_self: bool = False,
                 peer_halo: bool = False, peer_via_fd: bool = False):
        cells = [int(c) for c in cells]
        self.D = len(cells)
        self.cells = cells
        self.k = int(k)
        self.K = self.k ** self.D
        self.precision = precision
        lo = list(lo) if lo is not None else [0.0] * self.D
        hi = list(hi) if hi is not None else [1.0] * self.D
        gd = GridDesc(self.D, (ctypes.c_int64 * MAX_DIM)(*(cells + [1] * (MAX_DIM - self.D))))
        dom = Domain((ctypes.c_double * MAX_DIM)(*(lo + [0.0] * (MAX_DIM - self.D))),
                     (ctypes.c_double * MAX_DIM)(*(hi + [1.0] * (MAX_DIM - self.D))))
        n_double = None
        if isinstance(precision, int):  # the paper's "# double": number of leading fp64 slots
            n_double = precision
            prec = SLDG_MIXED
        else:
            prec = {"mixed": SLDG_MIXED, "fp64": SLDG_FP64}[precision]
        dist_p = None
        self._uid = None
        if world > 1 or force_halo or force_transpose or nccl_self or peer_halo:
            uid = None
            if world > 1:
                self._uid = ctypes.create_string_buffer(unique_id, 128)
                uid = ctypes.cast(self._uid, ctypes.c_void_p)
            flags = ((SLDG_DIST_FORCE_HALO if force_halo else 0) | (SLDG_DIST_FORCE_TRANSPOSE if force_transpose else 0)
                     | (SLDG_DIST_NCCL_SELF if nccl_self else 0) | (SLDG_DIST_PEER_HALO if peer_halo else 0)
                     | (SLDG_DIST_PEER_VIA_FD if peer_via_fd else 0))
            self._dist = Dist(rank, world, uid, None, max_halo, flags)
            dist_p = ctypes.byref(self._dist)
        h = ctypes.c_void_p()
        if n_double is None:
            _check(lib().sldg_create(ctypes.byref(gd), self.k, ctypes.byref(dom), prec, dist_p, ctypes.byref(h)))
        else:  # general layout: slots q < n_double in fp64 (sldg_create_ex)
            _check(lib().sldg_create_ex(ctypes.byref(gd), self.k, ctypes.byref(dom), int(n_double), dist_p,
                                        ctypes.byref(h)))
        self.h = h
        self._dependents = weakref.WeakSet()
        fl, nl = ctypes.c_int64(), ctypes.c_int64()
        _check(lib().sldg_shard_info(self.h, ctypes.byref(fl), ctypes.byref(nl)))
        self.first_layer, self.n_layers = fl.value, nl.value
        per_layer = 1
        for c in cells[:-1] if self.D > 1 else []:
            per_layer *= c
        self.local_cells = (nl.value * per_layer) if self.D > 1 else cells[0]

    # -- lifecycle
    def destroy(self):
        for dep in list(getattr(self, "_dependents", ())):
            dep.destroy()
        if getattr(self, "h", None):
            lib().sldg_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    # -- data
    def set_coeffs(self, c: np.ndarray, first_cell: int = 0):
        c = np.ascontiguousarray(c, dtype=np.float64)
        n = c.size // self.K
        _check(lib().sldg_set_coeffs(self.h, _dp(c), int(first_cell), n))

    def get_coeffs(self, first_cell: int = 0, n_cells: int | None = None) -> np.ndarray:
        if n_cells is None:
            n_cells = self.local_cells - first_cell
        out = np.empty((n_cells, self.K), dtype=np.float64)
        _check(lib().sldg_get_coeffs(self.h, _dp(out), int(first_cell), int(n_cells)))
        return out

    def advect(self, dim: int, shift: float = 0.0, field=None, field_mask: int = 0):
        if field is None:
            _check(lib().sldg_advect(self.h, int(dim), float(shift), None, ctypes.c_uint32(field_mask)))
        else:
            f = np.ascontiguousarray(field, dtype=np.float64)
            want = 1
            for e in range(self.D):
                if int(field_mask) >> e & 1:
                    want *= self.cells[e]
            if f.size != want:  # the C side reads exactly `want` doubles from this buffer
                raise SldgError(SLDG_EINVAL, f"shift field has {f.size} entries, field_mask {field_mask:#x} needs {want}")
            _check(lib().sldg_advect(self.h, int(dim), float(shift), _dp(f), ctypes.c_uint32(field_mask)))

    def advect_vnodes(self, dim: int, vdim: int, nodal_nu):
        """x-sweep along dim with one CFL number per Gauss node of every v-cell of vdim (NEXT-3)."""
        f = np.ascontiguousarray(nodal_nu, dtype=np.float64)
        if not 0 <= int(vdim) < self.D or f.size != self.cells[int(vdim)] * self.k:
            raise SldgError(SLDG_EINVAL, f"nodal field has {f.size} entries, needs n[vdim] * k")
        _check(lib().sldg_advect_vnodes(self.h, int(dim), int(vdim), _dp(f)))

    def advect_vnodes_device(self, dim: int, vdim: int, d_nodal_ptr: int):
        _check(lib().sldg_advect_vnodes_device(self.h, int(dim), int(vdim), ctypes.c_void_p(d_nodal_ptr)))

    def advect_device(self, dim: int, d_field_ptr: int, field_mask: int, shift: float = 0.0):
        _check(lib().sldg_advect_device(self.h, int(dim), float(shift), ctypes.c_void_p(d_field_ptr),
                                        ctypes.c_uint32(field_mask)))

    def advect_device_bounded(self, dim: int, d_field_ptr: int, field_mask: int, nu_min: float, nu_max: float,
                              shift: float = 0.0):
        """advect_device with a caller bound nu_min <= every entry <= nu_max: a sharded sweep sizes
        its halo from the bound (no host synchronisation; graph-capturable)."""
        _check(lib().sldg_advect_device_bounded(self.h, int(dim), float(shift), ctypes.c_void_p(d_field_ptr),
                                                ctypes.c_uint32(field_mask), float(nu_min), float(nu_max)))

    def advect_pair(self, shift0: float = 0.0, field0=None, mask0: int = 0, shift1: float = 0.0, field1=None,
                    mask1: int = 0):
        """advect(0, shift0, field0, mask0) then advect(1, shift1, field1, mask1), in one pass over
        HBM when the fields allow (sldg_advect_pair)."""
        def arr(f, mask):
            if f is None:
                return None
            f = np.ascontiguousarray(f, dtype=np.float64)
            want = 1
            for e in range(self.D):
                if int(mask) >> e & 1:
                    want *= self.cells[e]
            if f.size != want:
                raise SldgError(SLDG_EINVAL, f"shift field has {f.size} entries, field_mask {mask:#x} needs {want}")
            return f
        a0, a1 = arr(field0, mask0), arr(field1, mask1)
        _check(lib().sldg_advect_pair(self.h, float(shift0), None if a0 is None else _dp(a0), ctypes.c_uint32(mask0),
                                      float(shift1), None if a1 is None else _dp(a1), ctypes.c_uint32(mask1)))

    def advect_pair_device(self, d_field0_ptr: int, mask0: int, d_field1_ptr: int, mask1: int,
                           shift0: float = 0.0, shift1: float = 0.0):
        _check(lib().sldg_advect_pair_device(self.h, float(shift0), ctypes.c_void_p(d_field0_ptr or None),
                                             ctypes.c_uint32(mask0), float(shift1),
                                             ctypes.c_void_p(d_field1_ptr or None), ctypes.c_uint32(mask1)))

    def timeline(self, reset: bool = True):
        """[(kind, t0_ms, t1_ms)] of the profiled sweeps (kind = dim) and halo exchanges (-1)."""
        n = ctypes.c_int()
        _check(lib().sldg_timeline(self.h, None, None, 0, ctypes.byref(n), 0))
        t = np.zeros(2 * max(1, n.value))
        kinds = (ctypes.c_int * max(1, n.value))()
        _check(lib().sldg_timeline(self.h, _dp(t), kinds, n.value, ctypes.byref(n), int(reset)))
        return [(int(kinds[i]), float(t[2 * i]), float(t[2 * i + 1])) for i in range(n.value)]

    def mass(self) -> float:
        m = ctypes.c_double()
        _check(lib().sldg_mass(self.h, ctypes.byref(m)))
        return m.value

    def sync(self):
        _check(lib().sldg_sync(self.h))

    def fill_random(self, seed: int):
        _check(lib().sldg_fill_random(self.h, ctypes.c_uint64(seed)))

    def fill_separable(self, terms):
        """terms: list (per term) of lists (per dim) of [n_d, k] tables (GLOBAL n_d)."""
        flat = np.concatenate([np.ascontiguousarray(t, dtype=np.float64).reshape(-1)
                               for term in terms for t in term])
        _check(lib().sldg_fill_separable(self.h, len(terms), _dp(flat)))

    def memory_bytes(self) -> int:
        return int(lib().sldg_memory_bytes(self.h))

    # -- streams / instrumentation
    def stream(self) -> int:
        s = ctypes.c_void_p()
        _check(lib().sldg_get_stream(self.h, ctypes.byref(s)))
        return s.value or 0

    def set_stream(self, stream_ptr: int | None):
        _check(lib().sldg_set_stream(self.h, ctypes.c_void_p(stream_ptr or 0)))

    def profile(self, enable: bool):
        _check(lib().sldg_profile(self.h, int(bool(enable))))

    def kernel_time(self, dim: int = -1, reset: bool = False):
        """(ms, launches, algorithmic bytes) of the sweep kernels along dim (-1: all)."""
        ms, n, b = ctypes.c_double(), ctypes.c_int64(), ctypes.c_double()
        _check(lib().sldg_kernel_time(self.h, int(dim), ctypes.byref(ms), ctypes.byref(n), ctypes.byref(b),
                                      int(reset)))
        return ms.value, n.value, b.value

    def launch_count(self) -> int:
        return int(lib().sldg_launch_count(self.h))

    def graph_begin(self):
        """Start capturing asynchronous calls into a CUDA graph (sldg_graph_begin)."""
        _check(lib().sldg_graph_begin(self.h))

    def graph_end(self) -> "Graph":
        h = ctypes.c_void_p()
        _check(lib().sldg_graph_end(self.h, ctypes.byref(h)))
        gr = Graph(h)
        self._dependents.add(gr)
        return gr

    def transpose_count(self) -> int:
        n = ctypes.c_int64()
        _check(lib().sldg_transpose_count(self.h, ctypes.byref(n)))
        return n.value

    def sweep_kernel(self, dim: int) -> str:
        return lib().sldg_sweep_kernel(self.h, int(dim)).decode()


class VlasovPoisson:
    """Vlasov-Poisson driver on a Grid whose dims are [x_1..x_dx, v_1..v_dx] (sldg_vp_*; NEXT-2)."""

    def __init__(self, grid: "Grid", dx: int):
        self.grid = grid
        self.dx = int(dx)
        self.k = grid.k
        self.nx = [int(n) for n in grid.cells[: self.dx]]
        self.Nx = int(np.prod(self.nx))
        self.Kx = self.k ** self.dx
        h = ctypes.c_void_p()
        _check(lib().sldg_vp_create(grid.h, self.dx, ctypes.byref(h)))
        self.h = h
        grid._dependents.add(self)  # destroyed before the grid (sldg_vp_* hold the grid pointer)

    def destroy(self):
        if self.h:
            lib().sldg_vp_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass

    def density(self) -> np.ndarray:
        out = np.empty((self.Nx, self.Kx))
        _check(lib().sldg_vp_density(self.h, _dp(out)))
        return out

    def field(self, rho=None):
        """(E at x-cell centres [dx, Nx], E Legendre coefficients [Nx, k+1] (dx = 1) or None,
        electric energy); from the grid's f, or from a given density [Nx, k^dx]."""
        e = np.empty((self.dx, self.Nx))
        coef = np.empty((self.Nx, self.k + 1)) if self.dx == 1 else None
        w = np.empty(1)
        r = None if rho is None else np.ascontiguousarray(rho, dtype=np.float64).reshape(-1)
        _check(lib().sldg_vp_field(self.h, None if r is None else _dp(r), _dp(e),
                                   None if coef is None else _dp(coef), _dp(w)))
        return e, coef, float(w[0])

    def set_nodal(self, on: bool = True):
        """x sweeps by the Gauss-node velocity treatment (NEXT-3) instead of the cell centre."""
        _check(lib().sldg_vp_set_nodal(self.h, int(bool(on))))

    def field_async(self):
        """density + field solve of the grid's f into device buffers only (no host copy)."""
        _check(lib().sldg_vp_field(self.h, None, None, None, None))

    def step(self, dt: float, energy: bool = False):
        """One Strang step; returns the mid-step electric energy when energy=True."""
        if energy:
            w = np.empty(1)
            _check(lib().sldg_vp_step(self.h, float(dt), _dp(w)))
            return float(w[0])
        _check(lib().sldg_vp_step(self.h, float(dt), None))
        return None


class Graph:
    """A captured sequence of asynchronous grid calls (sldg_graph_*)."""

    def __init__(self, h):
        self.h = h

    def launch(self):
        _check(lib().sldg_graph_launch(self.h))

    def destroy(self):
        if self.h:
            lib().sldg_graph_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.destroy()
        except Exception:
            pass
