"""Parity oracle for the DB-TSDF scan-integration hot path.

TEST INFRASTRUCTURE ONLY — the checker, never the thing measured or shipped.
Only tests/, ``__graft_entry__.smoke()`` and bench.py's ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product package
(paper_2509_20081_b200) never imports it and has no CPU fallback.

Composition: preprocessing in numpy (oracle/prep.py, the reference's own numpy
calls restated) + stamping in C (oracle/dbtsdf_oracle.c, the reference's serial
sorted-order ``_stamp`` loop restated, compiled to oracle/liboracle.so by
paper_2509_20081_b200/build.py). Parity is pinned against outputs of the
reference itself: tests/golden/make_golden.py imports /root/reference in the
build container and stores hashes of the final grids (tests/golden/golden.json);
tests/test_oracle_golden.py checks this oracle reproduces every one.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

from . import prep

_HERE = Path(__file__).resolve().parent
_LIB = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_u8p = ctypes.POINTER(ctypes.c_uint8)
_u32p = ctypes.POINTER(ctypes.c_uint32)
_i32p = ctypes.POINTER(ctypes.c_int32)
_dp = ctypes.POINTER(ctypes.c_double)


def lib():
    """Load oracle/liboracle.so (built from oracle/*.c on demand)."""
    global _LIB
    if _LIB is None:
        path = _HERE / "liboracle.so"
        if not path.exists() or any(p.stat().st_mtime > path.stat().st_mtime for p in _HERE.glob("*.c")):
            from paper_2509_20081_b200 import build as _build  # build recipe only

            _build.build_oracle()
        L = ctypes.CDLL(str(path))
        L.orc_transform.argtypes = [_dp, ctypes.c_int64, _dp, _dp]
        L.orc_transform.restype = None
        L.orc_prepare.argtypes = [_dp, ctypes.c_int64, _dp, ctypes.c_int, _dp, ctypes.c_double, _i64p,
                                  ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, _i64p, _u8p, _i64p]
        L.orc_prepare.restype = None
        L.orc_bin_index_array.argtypes = [_dp, ctypes.c_int64, ctypes.c_int, ctypes.c_int, _i64p, _i64p]
        L.orc_bin_index_array.restype = None
        L.orc_stamp.argtypes = [_u32p, _u8p, _u8p, _i64p, ctypes.c_int, _u32p, _i32p, _i64p, _i64p, _u8p,
                                _i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                _i64p]
        L.orc_stamp.restype = ctypes.c_int64
        L.orc_stamp_slab.argtypes = [_u32p, _u8p, _u8p, _i64p, ctypes.c_int64, ctypes.c_int64, ctypes.c_int, _u32p,
                                     _i32p, _i64p, _i64p, _u8p, _i64p, ctypes.c_int64, ctypes.c_int, ctypes.c_int,
                                     ctypes.c_int, ctypes.c_int, _i64p]
        L.orc_stamp_slab.restype = ctypes.c_int64
        _LIB = L
    return _LIB


def _ptr(a, t):
    return a.ctypes.data_as(t)


@dataclass
class OracleBank:
    size: int
    b_az: int
    b_el: int
    distance_kernel: np.ndarray  # uint32 (K,K,K)
    shadow_xyz: np.ndarray  # int32 (total,3)
    shadow_start: np.ndarray  # int64 (n_bins+1)

    @property
    def half_extent(self):
        return self.size // 2

    @classmethod
    def build(cls, size=21, b_az=40, b_el=40, shadow_radius=3.0, shadow_model="hemisphere",
              cone_half_angle_deg=30.0):
        dk, xyz, start = prep.bank_tables(size, b_az, b_el, shadow_radius, shadow_model, cone_half_angle_deg)
        return cls(size, b_az, b_el, dk, np.ascontiguousarray(xyz), start)

    @classmethod
    def from_bank(cls, bank):
        """From any KernelBank-like object (distance_kernel, shadow_offsets)."""
        offs = bank.shadow_offsets
        counts = np.array([len(o) for o in offs], dtype=np.int64)
        start = np.zeros(len(offs) + 1, dtype=np.int64)
        np.cumsum(counts, out=start[1:])
        xyz = np.concatenate([np.asarray(o).reshape(-1, 3) for o in offs]).astype(np.int32)
        return cls(int(bank.size), int(bank.b_az), int(bank.b_el),
                   np.ascontiguousarray(bank.distance_kernel, dtype=np.uint32), np.ascontiguousarray(xyz), start)


@dataclass
class OracleGrid:
    """Reference voxel store (grid.py:39-89): three C-order arrays."""

    dims: tuple
    voxel_size: float
    origin: np.ndarray
    mask: np.ndarray = None
    sign: np.ndarray = None
    hits: np.ndarray = None
    slab: tuple = None  # (x0, x1) owned x-range; arrays hold only that slab

    def __post_init__(self):
        self.dims = tuple(int(d) for d in self.dims)
        self.origin = np.asarray(self.origin, dtype=np.float64)
        if self.slab is None:
            self.slab = (0, self.dims[0])
        shp = (self.slab[1] - self.slab[0], self.dims[1], self.dims[2])
        if self.mask is None:
            self.mask = np.full(shp, prep.FULL_MASK, dtype=np.uint32)
            self.sign = np.ones(shp, dtype=np.uint8)
            self.hits = np.zeros(shp, dtype=np.uint8)


@dataclass
class OracleStats:
    points_in: int = 0
    points_discarded: int = 0
    voxels_written: int = 0
    points_applied: int = 0
    extra: dict = field(default_factory=dict)


def stamp(grid: OracleGrid, bank: OracleBank, centers, ok, bins, h_max=255, t_occ=2, first_return=False,
          threads=1):
    """integrator.py:255-285 via the C restatement. Returns (voxels_written, applied)."""
    L = lib()
    centers = np.ascontiguousarray(centers, dtype=np.int64)
    ok = np.ascontiguousarray(ok, dtype=np.uint8)
    bins = np.ascontiguousarray(bins, dtype=np.int64)
    dims = np.array(grid.dims, dtype=np.int64)
    applied = ctypes.c_int64(0)
    for a in (grid.mask, grid.sign, grid.hits):
        assert a.flags.c_contiguous
    written = L.orc_stamp_slab(_ptr(grid.mask, _u32p), _ptr(grid.sign, _u8p), _ptr(grid.hits, _u8p),
                          _ptr(dims, _i64p), int(grid.slab[0]), int(grid.slab[1]), int(bank.size), _ptr(bank.distance_kernel, _u32p), _ptr(bank.shadow_xyz, _i32p),
                          _ptr(bank.shadow_start, _i64p), _ptr(centers, _i64p), _ptr(ok, _u8p), _ptr(bins, _i64p),
                          int(len(ok)), int(h_max), int(t_occ), int(bool(first_return)), int(threads),
                          ctypes.byref(applied))
    return int(written), int(applied.value)


def integrate_frame(grid: OracleGrid, bank: OracleBank, points, pose, h_max=255, t_occ=2, downsample=1,
                    first_return=False, threads=1, c_prep=False) -> OracleStats:
    """integrator.py:207-287 with compensation "none".

    c_prep=False: numpy preprocessing (bit-identical to the reference on the
    same host); c_prep=True: the C restatement (libm transcendentals), used
    by the timed CPU baseline.
    """
    pts = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    st = OracleStats()
    if pts.shape[0] == 0:
        return st
    if downsample > 1:
        pts = pts[::downsample]
    pose = np.asarray(pose, dtype=np.float64)
    r = bank.half_extent
    if c_prep:
        L = lib()
        pts = np.ascontiguousarray(pts)
        pose_c = np.ascontiguousarray(pose)
        pm = np.empty_like(pts)
        L.orc_transform(_ptr(pts, _dp), len(pts), _ptr(pose_c, _dp), _ptr(pm, _dp))
        sensor = np.ascontiguousarray(pose[:3, 3])
        centers = np.empty((len(pts), 3), np.int64)
        ok = np.empty(len(pts), np.uint8)
        bins = np.empty(len(pts), np.int64)
        dims = np.array(grid.dims, dtype=np.int64)
        L.orc_prepare(_ptr(pm, _dp), len(pts), _ptr(sensor, _dp), 0, _ptr(grid.origin, _dp), float(grid.voxel_size),
                      _ptr(dims, _i64p), r, bank.b_az, bank.b_el, 0, _ptr(centers, _i64p), _ptr(ok, _u8p),
                      _ptr(bins, _i64p))
        ok = ok.astype(bool)
    else:
        pm = prep.transform(pts, pose)
        centers, ok, bins = prep.prepare(pm, pose[:3, 3], grid.origin, grid.voxel_size, grid.dims, r, bank.b_az,
                                         bank.b_el)
    st.points_in = len(pts)
    st.points_discarded = st.points_in - int(np.count_nonzero(ok))
    st.voxels_written, st.points_applied = stamp(grid, bank, centers, ok, bins, h_max, t_occ, first_return,
                                                 threads)
    return st


def integrate_points_map(grid: OracleGrid, bank: OracleBank, p_map, sensor, h_max=255, t_occ=2):
    """Sequence of integrate_point calls (integrator.py:163-189). Each call is
    independent and the final grid is order-free, so they are stamped as one
    batch. Returns the per-point outcome (True = applied)."""
    p_map = np.asarray(p_map, dtype=np.float64).reshape(-1, 3)
    sensor = np.asarray(sensor, dtype=np.float64).reshape(-1, 3)
    rays = p_map - sensor
    # integrate_point's own discard uses the 1-D norm (integrator.py:174)
    deg = np.array([np.linalg.norm(r) < grid.voxel_size for r in rays], dtype=bool)
    r = bank.half_extent
    centers = prep.world_to_voxel_array(grid.origin, grid.voxel_size, p_map)
    d = np.array(grid.dims)
    ok = ~deg & np.all(centers >= r, axis=1) & np.all(centers <= d - 1 - r, axis=1)
    bins = np.zeros(len(p_map), dtype=np.int64)
    for i in np.nonzero(ok)[0]:  # integrate_point bins one ray at a time (integrator.py:183)
        b_a, b_e = prep.bin_index_array(rays[i][None, :], bank.b_az, bank.b_el)
        bins[i] = int(b_a[0]) * bank.b_el + int(b_e[0])
    stamp(grid, bank, centers, ok, bins, h_max, t_occ, False, 1)
    return ok


def os_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1
