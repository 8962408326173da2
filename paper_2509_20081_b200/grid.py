"""Dense voxel grid, device resident (reference grid.py:1-213).

``VoxelGrid`` keeps the reference's public surface — ``dims``,
``voxel_size``, ``origin``, ``h_max``/``t_occ`` provenance and the three
C-order field arrays ``mask`` (u32), ``sign`` (u8), ``hits`` (u8) — but the
authoritative voxel store lives in HBM, owned by libdbtsdf (see
csrc/engine.cuh): an 8-byte record per voxel (mask | sign, hits, pending
shadow visits), a 16-bit length cache and a 1-bit stamp certificate —
10.125 B/voxel. The numpy field arrays are a host mirror:

* they are materialised (downloaded) the first time ``mask``/``sign``/``hits``
  is touched;
* while a mirror exists, every engine call first uploads it (the caller may
  have written into it, as the reference's callers do) and every mutating
  call downloads into the same array objects in place, so references held by
  the caller see the update exactly as with the reference's in-place numpy
  arrays;
* ``release_host()`` drops the mirror; from then on the grid lives only in
  HBM (the production / benchmark mode: no per-scan grid transfers).

Queries (``observed_array``, ``signed_distance_field``, ``signed_distance``,
``to_records``) run the device readout kernels (``__popc``/``__clz`` decode).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _native
from .errors import ConfigurationError, CorruptionError, ResourceError

FULL_MASK = 0xFFFFFFFF
MAX_DISTANCE_CELLS = 32

SIGN_OCCUPIED = 0
SIGN_FREE = 1

BYTES_PER_VOXEL = 8

# Serialized voxel record (grid.py:30-34): mask (4, LE), sign (1), hits (1), 2 reserved.
VOXEL_DTYPE = np.dtype([("mask", "<u4"), ("sign", "u1"), ("hits", "u1"), ("reserved", "<u2")])

DEFAULT_MEMORY_CAP = 8 << 30  # bytes of voxel payload (reference accounting: 8 B/voxel)


def owned_planes(nx: int, slab=(0, None), interleave=None) -> np.ndarray:
    """Global x of the planes a grid stores, in storage order: the slab
    [x0, x1), or the interleaved blocks (width, parts, part) of [0, nx)."""
    if interleave is None:
        x0, x1 = slab[0], nx if slab[1] is None else slab[1]
        return np.arange(x0, x1, dtype=np.int64)
    w, p, r = interleave
    x = np.arange(nx, dtype=np.int64)
    return x[(x // w) % p == r]


class _GridHandle:
    def __init__(self, ptr):
        self.ptr = ptr

    def __del__(self):
        try:
            _native.lib().dbt_grid_destroy(self.ptr)
        except Exception:  # interpreter shutdown
            pass


class VoxelGrid:
    """Fixed-size axis-aligned grid; structure immutable after construction,
    voxel contents updated in place by the integrator (grid.py:39-58)."""

    def __init__(self, dims, voxel_size, origin, *, device: int | None = None, slab=None, interleave=None):
        """slab=(x0, x1): own the contiguous x-planes [x0, x1); interleave=
        (width, parts, part): own the planes whose block x // width is
        congruent to part mod parts (multi-GPU sharding, sharded.py)."""
        self.dims = tuple(int(d) for d in dims)
        self.voxel_size = float(voxel_size)
        self.origin = np.asarray(origin, dtype=np.float64).copy()
        self.h_max = 255
        self.t_occ = 2
        self.device = _native.default_device() if device is None else int(device)
        dims_a = np.array(self.dims, dtype=np.int64)
        org = np.ascontiguousarray(self.origin)
        out = ctypes.c_void_p()
        L = _native.lib()
        if interleave is not None:
            w, p, r = (int(v) for v in interleave)
            self.slab = (0, self.dims[0])
            self.interleave = (w, p, r)
            _native.check(L.dbt_grid_create_interleaved(dims_a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                                        self.voxel_size,
                                                        org.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                                        self.device, w, p, r, ctypes.byref(out)))
        else:
            x0, x1 = (0, self.dims[0]) if slab is None else (int(slab[0]), int(slab[1]))
            self.slab = (x0, x1)
            self.interleave = None
            _native.check(L.dbt_grid_create(dims_a.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                                            self.voxel_size, org.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                                            self.device, x0, x1, ctypes.byref(out)))
        self._handle = _GridHandle(out)
        self.owned_x = owned_planes(self.dims[0], self.slab, self.interleave)
        self._host = None  # (mask, sign, hits) mirror when exposed

    # ---- handle / mirror protocol -------------------------------------
    @property
    def handle(self):
        return self._handle.ptr

    @property
    def local_dims(self):
        return (len(self.owned_x), self.dims[1], self.dims[2])

    @property
    def num_voxels(self) -> int:
        nx, ny, nz = self.dims
        return nx * ny * nz

    def _expose(self):
        if self._host is None:
            shp = self.local_dims
            host = (np.empty(shp, np.uint32), np.empty(shp, np.uint8), np.empty(shp, np.uint8))
            _native.check(_native.lib().dbt_grid_download(self.handle, *(_native.ptr(a) for a in host)))
            self._host = host
        return self._host

    def push_host(self):
        """Upload the host mirror (if any) before an engine call."""
        if self._host is not None:
            m, s, h = self._host
            for a in self._host:
                if not a.flags.c_contiguous:
                    raise ConfigurationError("grid field arrays must stay C-contiguous")
            _native.check(_native.lib().dbt_grid_upload(self.handle, _native.ptr(m), _native.ptr(s), _native.ptr(h)))

    def pull_host(self):
        """Refresh the host mirror in place after a mutating engine call."""
        if self._host is not None:
            _native.check(_native.lib().dbt_grid_download(self.handle, *(_native.ptr(a) for a in self._host)))

    def release_host(self):
        """Drop the host mirror: the grid then lives only in HBM."""
        self.push_host()
        self._host = None

    def download_range(self, x_begin: int, x_end: int):
        """(mask, sign, hits) of global x-planes [x_begin, x_end) without
        touching the host mirror (streams grids too large to download whole)."""
        self.push_host()
        shp = (x_end - x_begin, self.dims[1], self.dims[2])
        out = (np.empty(shp, np.uint32), np.empty(shp, np.uint8), np.empty(shp, np.uint8))
        _native.check(_native.lib().dbt_grid_download_range(self.handle, int(x_begin), int(x_end),
                                                            *(_native.ptr(a) for a in out)))
        return out

    def synchronize(self):
        _native.check(_native.lib().dbt_synchronize(self.handle))

    def device_bytes(self) -> int:
        d = (ctypes.c_int64 * 3)()
        s = (ctypes.c_int64 * 2)()
        b = ctypes.c_int64()
        _native.check(_native.lib().dbt_grid_info(self.handle, d, s, ctypes.byref(b)))
        return int(b.value)

    # ---- reference field arrays -------------------------------------------
    def _set_field(self, i, value):
        arr = self._expose()[i]
        arr[...] = value

    mask = property(lambda self: self._expose()[0], lambda self, v: self._set_field(0, v))
    sign = property(lambda self: self._expose()[1], lambda self, v: self._set_field(1, v))
    hits = property(lambda self: self._expose()[2], lambda self, v: self._set_field(2, v))

    def __repr__(self):
        return f"VoxelGrid(dims={self.dims}, voxel_size={self.voxel_size}, origin={self.origin.tolist()}, device={self.device})"


def new_grid(dims, voxel_size: float, origin=(0.0, 0.0, 0.0), memory_cap: int = DEFAULT_MEMORY_CAP,
             device: int | None = None) -> VoxelGrid:
    """Allocate a fresh grid with every voxel unobserved (grid.py:61-89).

    ConfigurationError for degenerate dims/voxel_size; ResourceError when the
    reference payload (8 B/voxel) exceeds ``memory_cap`` or the device is out
    of memory. The device store itself takes 10.125 B/voxel (8-byte record,
    16-bit length cache, 1-bit stamp certificate).
    """
    dims = tuple(int(d) for d in dims)
    if len(dims) != 3 or any(d < 1 for d in dims):
        raise ConfigurationError(f"grid dims must be three positive counts, got {dims}")
    if not voxel_size > 0.0:
        raise ConfigurationError(f"voxel_size must be positive, got {voxel_size}")
    payload = dims[0] * dims[1] * dims[2] * BYTES_PER_VOXEL
    if payload > memory_cap:
        raise ResourceError(f"grid payload {payload} bytes exceeds memory cap {memory_cap}")
    return VoxelGrid(dims, voxel_size, origin, device=device)


def memory_bytes(grid: VoxelGrid) -> int:
    """Voxel payload size nx*ny*nz*8 bytes (grid.py:92-94)."""
    return grid.num_voxels * BYTES_PER_VOXEL


def world_to_voxel(grid: VoxelGrid, p):
    """Integer voxel indices of a world point; None when out of bounds (grid.py:97-104)."""
    idx = np.floor((np.asarray(p, dtype=np.float64) - grid.origin) / grid.voxel_size)
    ix, iy, iz = (int(v) for v in idx)
    nx, ny, nz = grid.dims
    if 0 <= ix < nx and 0 <= iy < ny and 0 <= iz < nz:
        return ix, iy, iz
    return None


def world_to_voxel_array(grid: VoxelGrid, points: np.ndarray) -> np.ndarray:
    """Vectorised floor indexing, no bounds check (grid.py:107-111)."""
    return np.floor((points - grid.origin[np.newaxis, :]) / grid.voxel_size).astype(np.int64)


def voxel_center(grid: VoxelGrid, ix, iy, iz) -> np.ndarray:
    return grid.origin + (np.array([ix, iy, iz], dtype=np.float64) + 0.5) * grid.voxel_size


def is_run_mask(mask) -> bool:
    """True iff mask is a contiguous low-bit run (incl. 0 and all-ones)."""
    m = int(mask) & FULL_MASK
    return (m & (m + 1)) & FULL_MASK == 0


def decode_distance(mask, checked: bool = True) -> int:
    """Population count of a run mask = truncated distance in cells (grid.py:124-129)."""
    m = int(mask) & FULL_MASK
    if checked and not is_run_mask(m):
        raise CorruptionError(f"distance mask {m:#010x} is not a low-bit run")
    return m.bit_count()


def run_mask(k: int) -> int:
    """Run mask with k active low bits, k in [0, 32] (grid.py:132-136)."""
    if not 0 <= k <= 32:
        raise ConfigurationError(f"run length {k} outside [0, 32]")
    return FULL_MASK >> (32 - k) if k > 0 else 0


def gather(grid: VoxelGrid, idx) -> tuple:
    """(mask, sign, hits) of the voxels at global indices idx (n,3), read on
    the device without downloading the grid."""
    idx = np.ascontiguousarray(np.asarray(idx, dtype=np.int64).reshape(-1, 3))
    n = idx.shape[0]
    m = np.empty(n, np.uint32)
    s = np.empty(n, np.uint8)
    h = np.empty(n, np.uint8)
    grid.push_host()
    _native.check(_native.lib().dbt_grid_gather(grid.handle, _native.ptr(idx), n, _native.ptr(m), _native.ptr(s),
                                                 _native.ptr(h)))
    return m, s, h


def is_observed(grid: VoxelGrid, ix, iy, iz) -> bool:
    m, _, h = gather(grid, [(ix, iy, iz)])
    return not (int(m[0]) == FULL_MASK and int(h[0]) == 0)


def signed_distance(grid: VoxelGrid, ix, iy, iz):
    """Signed distance in metres at a voxel, None when unobserved (grid.py:145-158)."""
    nx, ny, nz = grid.dims
    if not (0 <= ix < nx and 0 <= iy < ny and 0 <= iz < nz):
        raise IndexError(f"voxel index ({ix},{iy},{iz}) outside dims {grid.dims}")
    m, s, h = gather(grid, [(ix, iy, iz)])
    if int(m[0]) == FULL_MASK and int(h[0]) == 0:
        return None
    d = decode_distance(int(m[0]))
    sigma = -1.0 if int(s[0]) == SIGN_OCCUPIED else 1.0
    return sigma * d * grid.voxel_size


def observed_array(grid: VoxelGrid) -> np.ndarray:
    """Boolean array of voxels touched by at least one integration (grid.py:161-163)."""
    out = np.empty(grid.local_dims, np.uint8)
    grid.push_host()
    _native.check(_native.lib().dbt_observed(grid.handle, _native.ptr(out)))
    return out.view(np.bool_)


def popcount_array(masks) -> np.ndarray:
    """Per-voxel decoded distance. For a VoxelGrid this is the device readout;
    for a host mask array the reference's np.bitwise_count (grid.py:166-167)."""
    if isinstance(masks, VoxelGrid):
        out = np.empty(masks.local_dims, np.int32)
        masks.push_host()
        _native.check(_native.lib().dbt_popcount(masks.handle, _native.ptr(out)))
        return out
    return np.bitwise_count(np.asarray(masks)).astype(np.int32)


def signed_distance_field(grid: VoxelGrid):
    """Dense (field, observed); unobserved entries are +32*voxel_size
    placeholders to be gated by the observed array (grid.py:170-175)."""
    field_ = np.empty(grid.local_dims, np.float64)
    obs = np.empty(grid.local_dims, np.uint8)
    grid.push_host()
    _native.check(_native.lib().dbt_signed_distance_field(grid.handle, _native.ptr(field_), _native.ptr(obs)))
    return field_, obs.view(np.bool_)


def grid_counts(grid: VoxelGrid) -> tuple[int, int]:
    """(observed, occupied) voxel counts, reduced on the device (cli info)."""
    a, b = ctypes.c_int64(), ctypes.c_int64()
    grid.push_host()
    _native.check(_native.lib().dbt_grid_counts(grid.handle, ctypes.byref(a), ctypes.byref(b)))
    return int(a.value), int(b.value)


def to_records(grid: VoxelGrid) -> np.ndarray:
    """Serialized records in linear order ix + nx*(iy + ny*iz) (grid.py:178-185),
    transposed on the device from the voxel words."""
    rec = np.empty(grid.num_voxels, dtype=VOXEL_DTYPE)
    grid.push_host()
    _native.check(_native.lib().dbt_grid_to_records(grid.handle, _native.ptr(rec)))
    return rec


def from_records(rec: np.ndarray, dims, voxel_size, origin, h_max=255, t_occ=2, device: int | None = None) -> VoxelGrid:
    """Inverse of to_records (grid.py:188-202)."""
    dims = tuple(int(d) for d in dims)
    if rec.shape[0] != dims[0] * dims[1] * dims[2]:
        raise CorruptionError(f"record count {rec.shape[0]} does not match dims {dims}")
    g = new_grid(dims, voxel_size, origin, device=device)
    r = np.ascontiguousarray(rec)
    if r.dtype != VOXEL_DTYPE:
        r = r.astype(VOXEL_DTYPE)
    _native.check(_native.lib().dbt_grid_from_records(g.handle, _native.ptr(r)))
    g.h_max = int(h_max)
    g.t_occ = int(t_occ)
    return g


def grids_equal(a: VoxelGrid, b: VoxelGrid) -> bool:
    return (
        a.dims == b.dims
        and a.voxel_size == b.voxel_size
        and np.array_equal(a.origin, b.origin)
        and np.array_equal(a.mask, b.mask)
        and np.array_equal(a.sign, b.sign)
        and np.array_equal(a.hits, b.hits)
    )
