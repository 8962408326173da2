"""Fuse posed scans into the voxel grid on the GPU (reference integrator.py:1-287).

Same API and semantics as the reference: ``ScanFrame``, ``IntegrationParams``,
``FrameStats``, ``motion_compensate``, ``integrate_point``,
``integrate_frame``. The per-return work — transform to the map frame,
degenerate/boundary discards, direction binning, first-return dedup, the K^3
mask AND and the shadow hit/sign update — runs in libdbtsdf
(csrc/integrate.cu); Python only validates inputs and moves buffers.

Differences that are not semantic:

* ``threads`` is accepted for signature compatibility; the device decides.
* ``FrameStats.voxels_written`` counts mask cells changed by the concurrent
  stamping; the reference counts changes in its serial sorted order
  (integrator.py:266-285). Both are <= applied * K^3 and 0 for an empty
  scan; the grids themselves are identical.
* Extra, non-compared FrameStats fields report device counters.
"""

from __future__ import annotations

import ctypes
import os
import time
from dataclasses import dataclass, field

import numpy as np
from scipy.spatial.transform import Rotation, Slerp

from . import _native
from .errors import ConfigurationError
from .grid import VoxelGrid
from .kernels import KernelBank
from .transforms import _rot_z, check_rotation

COMPENSATION_MODES = ("none", "yaw", "se3")


class ScanFrame:
    """One LiDAR sweep: sensor-frame points plus the end-of-sweep pose (4x4,
    map frame); ``prev_pose``/``timestamps`` only for motion compensation
    (integrator.py:30-52). ``points`` reads as float64 like the reference;
    float32 input is kept as is and shipped to the device at 12 B/point (the
    widening to float64 is exact and happens on the device)."""

    def __init__(self, points, pose, timestamps=None, prev_pose=None):
        self.points = points
        self.pose = np.asarray(pose, dtype=np.float64)
        check_rotation(self.pose)
        self.prev_pose = None
        if prev_pose is not None:
            self.prev_pose = np.asarray(prev_pose, dtype=np.float64)
            check_rotation(self.prev_pose)
        self.timestamps = None
        if timestamps is not None:
            self.timestamps = np.asarray(timestamps, dtype=np.float64).ravel()
            if self.timestamps.shape[0] != self.n_points:
                raise ConfigurationError("timestamp count does not match point count")

    @property
    def points(self) -> np.ndarray:
        if self._f64 is None:
            self._f64 = self._f32.astype(np.float64)
        return self._f64

    @points.setter
    def points(self, value):
        a = np.asarray(value)
        if a.dtype == np.float32:
            self._f32 = np.ascontiguousarray(a.reshape(-1, 3))
            self._f64 = None
        else:
            self._f32 = None
            self._f64 = np.ascontiguousarray(np.asarray(a, dtype=np.float64).reshape(-1, 3))

    @property
    def n_points(self) -> int:
        return (self._f32 if self._f32 is not None else self._f64).shape[0]

    def device_payload(self):
        """(contiguous array, dtype code) to ship: float32 when the scan came
        in as float32, else float64."""
        if self._f32 is not None:
            return self._f32, _native.DBT_F32
        return self._f64, _native.DBT_F64


@dataclass
class IntegrationParams:
    h_max: int = 255
    t_occ: int = 2
    compensation: str = "none"
    downsample: int = 1
    first_return_per_voxel: bool = False
    # FrameStats.voxels_written as the reference's serial count (stamps in
    # ascending centre order) instead of the concurrent change count; costs
    # ~ms per scan (exact.cu). Default from $DBT_EXACT_VOXELS_WRITTEN.
    exact_voxels_written: bool = field(default_factory=lambda: os.environ.get("DBT_EXACT_VOXELS_WRITTEN") == "1")

    def __post_init__(self):
        if not 1 <= self.t_occ <= self.h_max <= 255:
            raise ConfigurationError(f"need 1 <= T ({self.t_occ}) <= H_max ({self.h_max}) <= 255")
        if self.compensation not in COMPENSATION_MODES:
            raise ConfigurationError(f"compensation must be one of {COMPENSATION_MODES}")
        if self.downsample < 1:
            raise ConfigurationError("downsample factor must be >= 1")

    def native(self, flags: int = 0, downsample: int | None = None):
        if self.exact_voxels_written:
            flags |= _native.FLAG_EXACT_WRITTEN
        return _native.make_params(self.h_max, self.t_occ, self.downsample if downsample is None else downsample,
                                   self.first_return_per_voxel, flags)


@dataclass
class FrameStats:
    points_in: int = 0
    points_discarded: int = 0
    voxels_written: int = 0
    elapsed_ms: float = 0.0
    # device counters (not part of equality, absent from the reference)
    points_applied: int = field(default=0, compare=False)
    unique_centers: int = field(default=0, compare=False)
    centers_skipped: int = field(default=0, compare=False)
    bin_fallbacks: int = field(default=0, compare=False)
    device_ms: float = field(default=0.0, compare=False)
    rows_swept: int = field(default=0, compare=False)

    @classmethod
    def from_native(cls, s: _native.Stats, elapsed_ms: float | None = None) -> "FrameStats":
        # ctypes int64 / double fields already read as Python int / float;
        # filling __dict__ directly skips the dataclass __init__ (per-call cost)
        o = object.__new__(cls)
        o.__dict__.update(points_in=s.points_in, points_discarded=s.points_discarded,
                          voxels_written=s.voxels_written,
                          elapsed_ms=s.elapsed_ms if elapsed_ms is None else float(elapsed_ms),
                          points_applied=s.points_applied, unique_centers=s.unique_centers,
                          centers_skipped=s.centers_skipped, bin_fallbacks=s.bin_fallbacks,
                          device_ms=s.device_ms, rows_swept=s.rows_swept)
        return o


def _scan_times(scan: ScanFrame) -> np.ndarray:
    if scan.timestamps is not None:
        return scan.timestamps
    n = scan.n_points
    return np.linspace(0.0, 1.0, n) if n > 1 else np.zeros(n)


def deskew_params(scan: ScanFrame, mode: str) -> "_native.Deskew":
    """The point-independent part of motion_compensate (integrator.py:91-123)
    for the device deskew (dbt_integrate_frame_deskew): computed here with
    scipy exactly as the reference computes it; the per-point part (pose at
    the point's time, the move to the end-of-sweep frame) runs on the device
    (csrc/deskew.cuh)."""
    if mode not in ("yaw", "se3"):
        raise ConfigurationError(f"no device deskew for compensation {mode!r}")
    if scan.prev_pose is None:
        raise ConfigurationError("motion compensation requires prev_pose")
    T0, T1 = scan.prev_pose, scan.pose
    d = _native.Deskew()
    if mode == "se3":
        rots = Rotation.from_matrix(np.stack([T0[:3, :3], T1[:3, :3]]))
        s = Slerp([0.0, 1.0], rots)
        rv = s.rotvecs[0] if hasattr(s, "rotvecs") else (rots[:-1].inv() * rots[1:]).as_rotvec()[0]
        d.mode = _native.DESKEW_SE3
        d.q[:] = [float(v) for v in s.rotations[0].as_quat(canonical=False)]
        d.rv[:] = [float(v) for v in rv]
    else:
        y0 = Rotation.from_matrix(T0[:3, :3]).as_euler("zyx")[0]
        y1 = Rotation.from_matrix(T1[:3, :3]).as_euler("zyx")[0]
        dy = (y1 - y0 + np.pi) % (2 * np.pi) - np.pi
        tilt = _rot_z(-y1) * Rotation.from_matrix(T1[:3, :3])
        d.mode = _native.DESKEW_YAW
        d.q[:] = [float(v) for v in np.asarray(tilt.as_quat(canonical=False)).reshape(4)]
        d.y0, d.dy = float(y0), float(dy)
    d.t0[:] = [float(v) for v in T0[:3, 3]]
    d.t1[:] = [float(v) for v in T1[:3, 3]]
    d.r1[:] = [float(v) for v in np.asarray(T1[:3, :3], np.float64).reshape(9)]
    return d


def motion_compensate(scan: ScanFrame, mode: str) -> ScanFrame:
    """Deskew to the end-of-sweep sensor frame (integrator.py:91-123). Host
    side (scipy Slerp/Rotation, as the reference); "none" is the identity."""
    if mode not in COMPENSATION_MODES:
        raise ConfigurationError(f"unknown compensation mode {mode!r}")
    if mode == "none" or scan.n_points == 0:
        return scan
    if scan.prev_pose is None:
        raise ConfigurationError("motion compensation requires prev_pose")
    ts = np.clip(_scan_times(scan), 0.0, 1.0)
    T0, T1 = scan.prev_pose, scan.pose
    trans = (1.0 - ts)[:, None] * T0[:3, 3] + ts[:, None] * T1[:3, 3]
    if mode == "se3":
        rots = Slerp([0.0, 1.0], Rotation.from_matrix(np.stack([T0[:3, :3], T1[:3, :3]])))(ts)
    else:  # yaw-only: heading lerp along the shortest arc, end tilt kept
        y0 = Rotation.from_matrix(T0[:3, :3]).as_euler("zyx")[0]
        y1 = Rotation.from_matrix(T1[:3, :3]).as_euler("zyx")[0]
        dy = (y1 - y0 + np.pi) % (2 * np.pi) - np.pi
        tilt = _rot_z(-y1) * Rotation.from_matrix(T1[:3, :3])
        rots = _rot_z(y0 + ts * dy) * tilt
    mats = rots.as_matrix()
    p_map = np.einsum("nij,nj->ni", mats, scan.points) + trans
    p_end = (p_map - T1[:3, 3]) @ T1[:3, :3]
    return ScanFrame(points=p_end, pose=scan.pose, timestamps=scan.timestamps, prev_pose=scan.prev_pose)


def _pose_arg(pose: np.ndarray):
    p = pose if (pose.dtype == np.float64 and pose.flags.c_contiguous) else np.ascontiguousarray(pose, np.float64)
    return p, _native.ptr(p)


def integrate_point(grid: VoxelGrid, bank: KernelBank, p_map, sensor_pos, params: IntegrationParams) -> str:
    """Fuse one map-frame return; "applied" or "discarded" (integrator.py:163-189)."""
    p_map = np.asarray(p_map, dtype=np.float64).reshape(3)
    sensor_pos = np.asarray(sensor_pos, dtype=np.float64).reshape(3)
    # the reference's degenerate test uses the 1-D norm (dot-based); apply it
    # here verbatim and tell the device to skip its axis-1 variant
    if np.linalg.norm(p_map - sensor_pos) < grid.voxel_size:
        return "discarded"
    out = integrate_points(grid, bank, p_map[None, :], sensor_pos[None, :], params, _skip_norm=True)
    return "applied" if out[0] else "discarded"


def integrate_points(grid: VoxelGrid, bank: KernelBank, p_map, sensor_pos, params: IntegrationParams,
                     _skip_norm: bool = False) -> np.ndarray:
    """Batched integrate_point: n map-frame returns with per-return sensor
    positions in one launch; returns a bool array (True = applied). Equal to
    calling integrate_point for each in any order (the grid is order-free);
    the degenerate test here is the axis-1 norm of integrate_frame."""
    p_map = np.ascontiguousarray(np.asarray(p_map, dtype=np.float64).reshape(-1, 3))
    sensor = np.ascontiguousarray(np.broadcast_to(np.asarray(sensor_pos, dtype=np.float64).reshape(-1, 3),
                                                  p_map.shape))
    n = p_map.shape[0]
    outcome = np.zeros(n, np.int8)
    if n == 0:
        return outcome.astype(bool)
    grid.h_max = params.h_max
    grid.t_occ = params.t_occ
    grid.push_host()
    flags = _native.FLAG_MAP_FRAME | (_native.FLAG_SKIP_NORM_CHECK if _skip_norm else 0)
    prm = _native.make_params(params.h_max, params.t_occ, 1, False, flags)
    st = _native.Stats()
    _native.check(_native.lib().dbt_integrate_points_map(grid.handle, bank.device_handle(grid.device),
                                                         _native.ptr(p_map), _native.ptr(sensor), n,
                                                         ctypes.byref(prm), ctypes.byref(st), _native.ptr(outcome)))
    grid.pull_host()
    return outcome.astype(bool)


def integrate_frame(grid: VoxelGrid, bank: KernelBank, scan: ScanFrame, params: IntegrationParams,
                    threads: int = 1) -> FrameStats:
    """Fuse one scan (integrator.py:207-287): the points cross the host link
    once (pinned scans are read zero-copy by the preprocessing kernel;
    pageable ones are first copied by a host thread pool into pinned, mapped
    staging and then read the same way), then the device launch sequence and
    one D2H copy of the counters. compensation "yaw"/"se3" deskews on the
    device (deskew_params + csrc/deskew.cuh)."""
    t0 = time.perf_counter()
    if scan.n_points == 0:
        return FrameStats()
    downsample = params.downsample
    if params.compensation != "none" and device_deskew_available():
        # deskew on the device (csrc/deskew.cuh): the point-independent part
        # here with scipy, the per-point part in the preprocessing kernel
        dk = deskew_params(scan, params.compensation)
        grid.h_max = params.h_max
        grid.t_occ = params.t_occ
        pts, dtype = scan.device_payload()
        pose, pose_p = _pose_arg(scan.pose)
        ts = scan.timestamps
        prm = params.native(downsample=downsample)
        st = _native.Stats()
        grid.push_host()
        _native.check(_native.lib().dbt_integrate_frame_deskew(
            grid.handle, bank.device_handle(grid.device), _native.ptr(pts), dtype, pts.shape[0],
            None if ts is None else _native.ptr(ts), pose_p, ctypes.byref(dk), ctypes.byref(prm), ctypes.byref(st)))
        grid.pull_host()
        return FrameStats.from_native(st, (time.perf_counter() - t0) * 1e3)
    if params.compensation != "none":
        # the C library could not be matched (device_deskew_available): deskew
        # on the host exactly as the reference, then ship float64
        if downsample > 1:
            keep = slice(None, None, downsample)
            scan = ScanFrame(points=scan.points[keep], pose=scan.pose,
                             timestamps=None if scan.timestamps is None else scan.timestamps[keep],
                             prev_pose=scan.prev_pose)
            downsample = 1
        scan = motion_compensate(scan, params.compensation)
    grid.h_max = params.h_max
    grid.t_occ = params.t_occ
    pts, dtype = scan.device_payload()
    pose, pose_p = _pose_arg(scan.pose)
    prm = params.native(downsample=downsample)
    st = _native.Stats()
    grid.push_host()
    _native.check(_native.lib().dbt_integrate_frame(grid.handle, bank.device_handle(grid.device), _native.ptr(pts),
                                                    dtype, pts.shape[0], pose_p, ctypes.byref(prm), ctypes.byref(st)))
    grid.pull_host()
    return FrameStats.from_native(st, (time.perf_counter() - t0) * 1e3)


class PendingFrame:
    """A queued integrate_frame_async call: ``result()`` waits for it and
    returns its FrameStats (idempotent). Keeps the scan's points alive until
    then (the device copy reads them asynchronously)."""

    def __init__(self, grid: VoxelGrid, ticket: int | None, keep=None, stats: FrameStats | None = None):
        self._grid, self._ticket, self._keep, self._stats = grid, ticket, keep, stats

    def done(self) -> bool:
        return self._stats is not None

    def result(self) -> FrameStats:
        if self._stats is None:
            st = _native.Stats()
            _native.check(_native.lib().dbt_frame_wait(self._grid.handle, self._ticket, ctypes.byref(st)))
            self._stats = FrameStats.from_native(st, st.elapsed_ms)
            self._keep = None
        return self._stats


def integrate_frame_async(grid: VoxelGrid, bank: KernelBank, scan: ScanFrame, params: IntegrationParams) -> PendingFrame:
    """integrate_frame without waiting (dbt_integrate_frame_async): the scan
    is copied to the device on a copy stream and its launch sequence queued;
    consecutive calls pipeline, so the next scan's host work and host->device
    copy overlap this scan's kernels. Collect FrameStats with ``.result()``
    (at most 4 calls may be outstanding: the fifth call waits for the
    oldest). The grid's host mirror is dropped; reading grid.mask/sign/hits
    orders after every queued call. Motion-compensated scans run
    synchronously (integrate_frame)."""
    if params.compensation != "none" or scan.n_points == 0:
        return PendingFrame(grid, None, stats=integrate_frame(grid, bank, scan, params))
    grid.h_max = params.h_max
    grid.t_occ = params.t_occ
    grid.push_host()
    grid._host = None
    pts, dtype = scan.device_payload()
    pose, pose_p = _pose_arg(scan.pose)
    prm = params.native()
    ticket = ctypes.c_int64()
    _native.check(_native.lib().dbt_integrate_frame_async(grid.handle, bank.device_handle(grid.device),
                                                          _native.ptr(pts), dtype, pts.shape[0], pose_p,
                                                          ctypes.byref(prm), ctypes.byref(ticket)))
    return PendingFrame(grid, ticket.value, keep=(pts, pose))


_DESKEW_OK = None


def device_deskew_available() -> bool:
    """The device deskew reproduces the C library's sin/cos bit for bit
    (csrc/libm_emu.cuh); the engine checks that against this process's libm
    once. False (host deskew through scipy) on another libm build."""
    global _DESKEW_OK
    if _DESKEW_OK is None:
        if os.environ.get("DBT_HOST_DESKEW") == "1":
            _DESKEW_OK = False
        else:
            ok = ctypes.c_int32()
            _native.check(_native.lib().dbt_deskew_available(ctypes.byref(ok)))
            _DESKEW_OK = bool(ok.value)
    return _DESKEW_OK


def integrate_frames(grid: VoxelGrid, bank: KernelBank, scans, params: IntegrationParams) -> list:
    """Several scans in one launch sequence (batched config-5 path). Per-frame
    downsampling, discards and first-return are preserved; the final grid is
    the one sequential integrate_frame calls produce (order-free updates).
    Compensated scans are deskewed on the host first."""
    scans = list(scans)
    if params.exact_voxels_written:
        # the serial count is per scan: one launch each
        return [integrate_frame(grid, bank, s, params) for s in scans]
    if params.compensation != "none" and device_deskew_available():
        # device deskew: one launch per scan (the per-scan pose interpolation
        # constants travel as kernel parameters)
        return [integrate_frame(grid, bank, s, params) for s in scans]
    if params.compensation != "none":
        prepped = []
        for s in scans:
            if params.downsample > 1 and s.n_points:
                k = slice(None, None, params.downsample)
                s = ScanFrame(points=s.points[k], pose=s.pose,
                              timestamps=None if s.timestamps is None else s.timestamps[k], prev_pose=s.prev_pose)
            prepped.append(motion_compensate(s, params.compensation))
        scans, downsample = prepped, 1
    else:
        downsample = params.downsample
    if not scans:
        return []
    t0 = time.perf_counter()
    payloads = [s.device_payload() for s in scans]
    dtype = _native.DBT_F32 if all(d == _native.DBT_F32 for _, d in payloads) else _native.DBT_F64
    np_dt = np.float32 if dtype == _native.DBT_F32 else np.float64
    # one pointer per scan: no host concatenation (pinned scans are read
    # zero-copy by the device, pageable ones staged scan by scan)
    arrays = [p if p.dtype == np_dt else p.astype(np_dt) for p, _ in payloads]
    ptrs = (ctypes.c_void_p * len(arrays))(*[a.ctypes.data for a in arrays])
    counts = np.array([a.shape[0] for a in arrays], dtype=np.int64)
    poses = np.ascontiguousarray(np.stack([s.pose for s in scans]).reshape(-1))
    grid.h_max = params.h_max
    grid.t_occ = params.t_occ
    prm = params.native(downsample=downsample)
    out = (_native.Stats * len(scans))()
    grid.push_host()
    _native.check(_native.lib().dbt_integrate_scans(
        grid.handle, bank.device_handle(grid.device), ptrs, dtype,
        counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(scans),
        ctypes.c_void_p(poses.ctypes.data), ctypes.byref(prm), out))
    grid.pull_host()
    el = (time.perf_counter() - t0) * 1e3
    return [FrameStats.from_native(out[i], el if i == 0 else 0.0) for i in range(len(scans))]
