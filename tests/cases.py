"""Parity cases shared by tests/golden/make_golden.py (which runs the
reference on them) and the oracle / GPU parity tests (which must reproduce
the stored hashes). Inputs are regenerated from seeds; their hashes are stored
with the golden outputs so generator drift on another host is reported as
such, not as a kernel mismatch.

Each case: grid (dims, voxel_size, origin), optional non-fresh initial
state, bank parameters, integration params and a list of frames
(sensor-frame points + pose) or of integrate_point hits (map-frame point +
sensor position).
"""

from __future__ import annotations

import hashlib
import math
import os
import sys
from dataclasses import dataclass, field

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import workloads  # noqa: E402

FULL = 0xFFFFFFFF


def sha(a) -> str:
    a = np.ascontiguousarray(a)
    h = hashlib.sha256()
    h.update(str(a.dtype).encode())
    h.update(str(a.shape).encode())
    h.update(a.reshape(-1).view(np.uint8).data if a.size else b"")  # the raw bytes, no copy
    return h.hexdigest()[:32]


def yaw_pose(yaw, t):
    T = np.eye(4)
    c, s = math.cos(yaw), math.sin(yaw)
    T[:3, :3] = [[c, -s, 0], [s, c, 0], [0, 0, 1]]
    T[:3, 3] = t
    return T


@dataclass
class Case:
    name: str
    dims: tuple
    voxel_size: float
    origin: tuple
    bank: dict
    params: dict = field(default_factory=dict)
    frames: list = field(default_factory=list)   # [(points, pose)]
    hits: tuple | None = None                    # (p_map (n,3), sensor (n,3)) for integrate_point
    init: tuple | None = None                    # (mask, sign, hits) non-fresh start
    slow: bool = False                           # large grid: skip in quick runs

    def input_hash(self) -> str:
        h = hashlib.sha256()
        for p, pose in self.frames:
            h.update(np.ascontiguousarray(p).tobytes())
            h.update(np.ascontiguousarray(pose).tobytes())
        if self.hits is not None:
            h.update(np.ascontiguousarray(self.hits[0]).tobytes())
            h.update(np.ascontiguousarray(self.hits[1]).tobytes())
        if self.init is not None:
            for a in self.init:
                h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()[:32]


def _random_state(rng, dims, h_hi=256):
    k = rng.integers(0, 33, size=dims)
    mask = np.where(k > 0, (FULL >> (32 - np.maximum(k, 1))).astype(np.uint64), 0).astype(np.uint32)
    hits = rng.integers(0, h_hi, size=dims).astype(np.uint8)
    sign = rng.integers(0, 2, size=dims).astype(np.uint8)
    return mask, sign, hits


def _random_hits(rng, n, dims, vs, margin=11):
    lo = margin * vs
    his = [(d - margin) * vs for d in dims]
    pts = rng.uniform([lo] * 3, his, size=(n, 3))
    dirs = rng.normal(size=(n, 3))
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    return pts, pts - dirs


def small_cases() -> list:
    cases = []
    eye = np.eye(4)
    b3 = dict(size=21, shadow_radius=3)
    # test_integrator-style random frames (uniform in [1.2, 2.9]^3, 41^3 grid)
    rng = np.random.default_rng(11)
    pts = rng.uniform(1.2, 2.9, size=(500, 3))
    cases.append(Case("frame500_default", (41, 41, 41), 0.1, (0, 0, 0), b3, {}, [(pts, eye)]))
    cases.append(Case("frame500_first_return", (41, 41, 41), 0.1, (0, 0, 0), b3,
                      {"first_return_per_voxel": True}, [(pts, eye)]))
    cases.append(Case("frame500_downsample3", (41, 41, 41), 0.1, (0, 0, 0), b3, {"downsample": 3}, [(pts, eye)]))
    # rotated + translated poses over several frames (FMA-chain transform)
    rng = np.random.default_rng(21)
    frames = []
    for k in range(4):
        p = rng.uniform(-1.2, 1.2, size=(400, 3)).astype(np.float32)
        frames.append((p, yaw_pose(rng.uniform(0, 2 * np.pi), (3.2, 3.1, 3.0))))
    cases.append(Case("yaw_frames_f32", (64, 64, 64), 0.1, (0, 0, 0), dict(size=21, shadow_radius=2), {"t_occ": 1},
                      frames))
    # non-fresh start: random run masks, hits 0..255 (incl. > h_max), random signs
    for model, hm, t in (("hemisphere", 7, 3), ("cone", 200, 2), ("hemisphere", 255, 1)):
        rng = np.random.default_rng(31 + hm)
        dims = (48, 48, 48)
        init = _random_state(rng, dims)
        frames = [(rng.uniform(1.15, 3.6, size=(300, 3)), yaw_pose(0.3 * k, (0.05 * k, 0.02, -0.01))) for k in range(3)]
        cases.append(Case(f"nonfresh_{model}_h{hm}_t{t}", dims, 0.1, (0, 0, 0),
                          dict(size=21, shadow_radius=3 if model == "cone" else 2, shadow_model=model,
                               cone_half_angle_deg=40.0), {"h_max": hm, "t_occ": t}, frames, init=init))
    # arbitrary state the reference accepts: any 32-bit mask (not only low-bit
    # runs), any sign byte, any hit count
    rng = np.random.default_rng(77)
    dims = (48, 48, 48)
    init = (rng.integers(0, 2**32, size=dims, dtype=np.uint64).astype(np.uint32),
            rng.integers(0, 256, size=dims).astype(np.uint8), rng.integers(0, 256, size=dims).astype(np.uint8))
    frames = [(rng.uniform(1.15, 3.6, size=(300, 3)), yaw_pose(0.2 * k, (0.03 * k, 0.0, 0.0))) for k in range(2)]
    cases.append(Case("arbitrary_state", dims, 0.1, (0, 0, 0), dict(size=21, shadow_radius=2), {"h_max": 250, "t_occ": 4},
                      frames, init=init))
    # other kernel sizes
    rng = np.random.default_rng(41)
    p = rng.uniform(0.45, 2.75, size=(300, 3))
    cases.append(Case("k9_bins8", (32, 32, 32), 0.1, (0, 0, 0), dict(size=9, b_az=8, b_el=8, shadow_radius=2), {},
                      [(p, eye)]))
    p = rng.uniform(1.2, 5.2, size=(300, 3))
    cases.append(Case("k23_wide", (64, 64, 64), 0.1, (0, 0, 0), dict(size=23, shadow_radius=4), {"t_occ": 1},
                      [(p, eye)]))
    # reference acceptance C1 shape: integrate_point hits, random directions
    rng = np.random.default_rng(42)
    pm, sens = _random_hits(rng, 10_000, (64, 64, 64), 0.1)
    cases.append(Case("c1_points10k", (64, 64, 64), 0.1, (0, 0, 0), b3, {"t_occ": 2}, hits=(pm, sens)))
    # boundary + degenerate + NaN/inf returns mixed in
    rng = np.random.default_rng(51)
    p = rng.uniform(-0.5, 4.6, size=(400, 3))
    p[:5] = [[0.0, 0.0, 0.001], [np.nan, 1, 1], [np.inf, 1, 1], [1e30, 0, 0], [0.05, 0.0, 0.0]]
    cases.append(Case("edge_returns", (41, 41, 41), 0.1, (0, 0, 0), b3, {}, [(p, yaw_pose(0.0, (2.0, 2.0, 2.0)))]))
    cases.append(Case("empty_scan", (41, 41, 41), 0.1, (0, 0, 0), b3, {}, [(np.zeros((0, 3)), eye)]))
    return cases


def config_cases(include_slow=True) -> list:
    cases = []
    w = workloads.get(1)
    cases.append(Case("cfg1_scan0", w.dims, w.voxel_size, w.origin, dict(size=21, shadow_radius=w.shadow_radius), {},
                      [(w.scan(0), w.poses[0])]))
    w = workloads.get(2)
    cases.append(Case("cfg2_scans0-2", w.dims, w.voxel_size, w.origin, dict(size=21, shadow_radius=w.shadow_radius),
                      {}, [(w.scan(k), w.poses[k]) for k in range(3)]))
    cases.append(Case("cfg2_scan0_rs3", w.dims, w.voxel_size, w.origin, dict(size=21, shadow_radius=3), {},
                      [(w.scan(0), w.poses[0])]))
    if include_slow:
        w = workloads.get(3)
        cases.append(Case("cfg3_scans0-1", w.dims, w.voxel_size, w.origin, dict(size=21, shadow_radius=w.shadow_radius),
                          {}, [(w.scan(k), w.poses[k]) for k in range(2)], slow=True))
        # config-4 scene/sensor at 0.02 m on a 1000x1000x400 window (the full
        # 6.4e9-voxel grid needs 38 GB of reference host arrays)
        w4 = workloads.get(4)
        cases.append(Case("cfg4_window_scan0", (1000, 1000, 400), w4.voxel_size, (0.0, 90.0, -0.22),
                          dict(size=21, shadow_radius=w4.shadow_radius), {}, [(w4.scan(0), w4.poses[0])], slow=True))
    return cases


@dataclass
class DeskewCase:
    """Motion-compensated frames (compensation "se3" / "yaw",
    integrator.py:91-123): frames are (points, pose, prev_pose, timestamps
    or None)."""
    name: str
    dims: tuple
    voxel_size: float
    origin: tuple
    bank: dict
    params: dict
    frames: list

    def input_hash(self) -> str:
        h = hashlib.sha256()
        for p, pose, prev, ts in self.frames:
            for a in (p, pose, prev) + (() if ts is None else (ts,)):
                h.update(np.ascontiguousarray(a).tobytes())
        return h.hexdigest()[:32]


def _euler_pose(yaw, pitch, roll, t):
    cy, sy, cp, sp, cr, sr = (math.cos(yaw), math.sin(yaw), math.cos(pitch), math.sin(pitch), math.cos(roll),
                              math.sin(roll))
    Rz = np.array([[cy, -sy, 0], [sy, cy, 0], [0, 0, 1]])
    Ry = np.array([[cp, 0, sp], [0, 1, 0], [-sp, 0, cp]])
    Rx = np.array([[1, 0, 0], [0, cr, -sr], [0, sr, cr]])
    T = np.eye(4)
    T[:3, :3] = Rz @ Ry @ Rx
    T[:3, 3] = t
    return T


def deskew_cases() -> list:
    """Seeded sweeps with motion during the sweep: heading wraps across +-pi,
    tilted poses, tiny rotations (Slerp's small-angle branch), explicit
    timestamps (some outside [0, 1]: clipped) and point-order timestamps,
    float32 and float64 points, downsampling."""
    out = []
    dims, vs, org = (64, 64, 64), 0.1, (0.0, 0.0, 0.0)
    c = (3.2, 3.2, 3.2)
    b = dict(size=21, shadow_radius=2)

    def sweep(rng, n, f32):
        p = rng.uniform(-1.4, 1.4, size=(n, 3))
        return p.astype(np.float32) if f32 else p

    for mode in ("se3", "yaw"):
        rng = np.random.default_rng(71 if mode == "se3" else 72)
        frames = []
        for k in range(3):
            y0 = rng.uniform(-math.pi, math.pi)
            y1 = y0 + rng.uniform(-0.6, 0.6) + (2 * math.pi if k == 1 else 0.0)  # k = 1 wraps
            T0 = _euler_pose(y0, rng.normal() * 0.05, rng.normal() * 0.05, np.add(c, rng.normal(size=3) * 0.1))
            T1 = _euler_pose(y1, rng.normal() * 0.05, rng.normal() * 0.05, np.add(c, rng.normal(size=3) * 0.1))
            frames.append((sweep(rng, 1500, k == 2), T1, T0, None))
        out.append(DeskewCase(f"deskew_{mode}_linspace", dims, vs, org, b, {"compensation": mode}, frames))
        frames = []
        for k in range(3):
            y0 = rng.uniform(-math.pi, math.pi)
            T0 = _euler_pose(y0, 0.02, -0.03, np.add(c, rng.normal(size=3) * 0.1))
            dyaw = 1e-5 if k == 0 else rng.uniform(-0.4, 0.4)  # k = 0: small-angle Slerp
            T1 = _euler_pose(y0 + dyaw, 0.02 + (0 if k == 0 else 0.03), -0.03, np.add(c, rng.normal(size=3) * 0.1))
            n = 1800
            ts = np.sort(rng.uniform(-0.05, 1.05, n))
            frames.append((sweep(rng, n, k != 1), T1, T0, ts))
        out.append(DeskewCase(f"deskew_{mode}_ts_ds2", dims, vs, org, b, {"compensation": mode, "downsample": 2},
                              frames))
    # config 2's trajectory with the previous scan's pose as the sweep start
    w = workloads.get(2)
    frames = [(w.scan(k), w.poses[k], w.poses[k - 1], None) for k in (1, 2, 3)]
    out.append(DeskewCase("deskew_cfg2_scans1-3_se3", w.dims, w.voxel_size, w.origin,
                          dict(size=21, shadow_radius=w.shadow_radius), {"compensation": "se3"}, frames))
    # config 3's street trajectory (262 k returns per scan), yaw mode with
    # per-return times in firing order (azimuth-major sweep)
    w = workloads.get(3)
    frames = []
    for k in (1, 2):
        pts = w.scan(k)
        frames.append((pts, w.poses[k], w.poses[k - 1], np.linspace(0.0, 1.0, len(pts))[::-1].copy()))
    out.append(DeskewCase("deskew_cfg3_scans1-2_yaw", w.dims, w.voxel_size, w.origin,
                          dict(size=21, shadow_radius=w.shadow_radius), {"compensation": "yaw"}, frames))
    return out


def bank_specs() -> list:
    return [
        dict(size=21, shadow_radius=1),
        dict(size=21, shadow_radius=2),
        dict(size=21, shadow_radius=3),
        dict(size=21, shadow_radius=3, shadow_model="cone", cone_half_angle_deg=30.0),
        dict(size=21, shadow_radius=2, shadow_model="cone", cone_half_angle_deg=40.0),
        dict(size=9, b_az=8, b_el=8, shadow_radius=2),
        dict(size=3, b_az=1, b_el=1, shadow_radius=1),
        dict(size=23, shadow_radius=4),
    ]


def bank_key(spec: dict) -> str:
    return ",".join(f"{k}={spec[k]}" for k in sorted(spec))


def bank_hashes(bank) -> dict:
    offs = [np.asarray(o, dtype=np.int64).reshape(-1, 3) for o in bank.shadow_offsets]
    counts = np.array([len(o) for o in offs], dtype=np.int64)
    return {
        "distance_kernel": sha(np.asarray(bank.distance_kernel, dtype=np.uint32)),
        "shadow_counts": sha(counts),
        "shadow_offsets": sha(np.concatenate(offs)),
        "bin_dirs": sha(np.asarray(bank.bin_dirs, dtype=np.float64)),
    }


def bin_dir_sets() -> dict:
    """Direction sets whose (b_a, b_e) from the reference bin_index_array are
    stored: random normals (test_kernels.py:32-37 shape) and bin centres."""
    rng = np.random.default_rng(3)
    out = {"normal200": rng.normal(size=(200, 3)), "normal100k": rng.normal(size=(100_000, 3))}
    centres = []
    for ba in range(40):
        for be in range(40):
            a = (ba + 0.5) * 2 * math.pi / 40
            e = (be + 0.5) * math.pi / 40 - math.pi / 2
            centres.append([math.cos(e) * math.cos(a), math.cos(e) * math.sin(a), math.sin(e)])
    out["bin_centres"] = np.array(centres)
    out["axes"] = np.array([[1, 0, 0], [0, 0, 1], [0, -1, 0], [-1, 0, 0], [0, 1, 0], [0, 0, -1], [1, 1, 0],
                            [-1, -1, 0], [1, -1, 0], [3, 4, 0], [1, 1, 1]], dtype=np.float64)
    return out


# --------------------------------------------------------------------------
# Trajectories: the regime the bench times (many launches into one grid, so
# stamp certificates, culling, lazy shadow folds and PDL ordering carry state
# across scans). The reference's grid hashes are stored after EVERY scan, so
# a GPU run can be compared scan by scan or at the end of any batch split.


@dataclass
class Trajectory:
    name: str
    config: int
    scans: tuple          # (first, last + 1)
    dims: tuple
    voxel_size: float
    origin: tuple
    bank: dict
    slow: bool = False    # multi-GB grids / minutes of ray casting

    def workload(self):
        return workloads.get(self.config)

    def scan_ids(self):
        return list(range(*self.scans))


def trajectories() -> list:
    w2, w3, w4 = workloads.get(2), workloads.get(3), workloads.get(4)
    return [
        # config 2 in full: the 100-scan trajectory
        Trajectory("cfg2_traj100", 2, (0, 100), w2.dims, w2.voxel_size, w2.origin,
                   dict(size=21, shadow_radius=w2.shadow_radius)),
        # config 3 prefix, also the config-5 batched case (batches of 8 / 32 / 128)
        Trajectory("cfg3_traj128", 3, (0, 128), w3.dims, w3.voxel_size, w3.origin,
                   dict(size=21, shadow_radius=w3.shadow_radius), slow=True),
        # config-4 scene/sensor at 0.02 m on the 1000x1000x400 window (the
        # reference's host arrays for the full grid are 38 GB); scans 0-29
        # cover the bench's prefill + timed window
        Trajectory("cfg4_window_traj30", 4, (0, 30), (1000, 1000, 400), w4.voxel_size, (0.0, 90.0, -0.22),
                   dict(size=21, shadow_radius=w4.shadow_radius), slow=True),
    ]


def scan_hash(pts, pose) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pts).reshape(-1).view(np.uint8).data if len(pts) else b"")
    h.update(np.ascontiguousarray(pose).tobytes())
    return h.hexdigest()[:32]
