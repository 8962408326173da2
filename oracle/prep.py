"""numpy restatement of the reference preprocessing and kernel-bank tables.

TEST INFRASTRUCTURE ONLY: imported by tests/, ``__graft_entry__.smoke()`` and
bench.py's CPU-baseline leg as the parity checker; never by the product
package. Each function cites the reference line it restates
(/root/reference/pkg/src/bitsdf). numpy calls are the same ones the reference
makes, so on a given host the results (incl. numpy's SIMD arctan2/arcsin
rounding) are bit-identical to the reference's.
"""

from __future__ import annotations

import math

import numpy as np

TWO_PI = 2.0 * math.pi  # kernels.py:28
FULL_MASK = 0xFFFFFFFF


def run_mask(k: int) -> int:
    """grid.py:132-136: k low bits set, k in [0, 32]."""
    return FULL_MASK >> (32 - k) if k > 0 else 0


def transform(points: np.ndarray, pose: np.ndarray) -> np.ndarray:
    """integrator.py:232 — map-frame points ``points @ R.T + t``."""
    points = np.asarray(points, dtype=np.float64).reshape(-1, 3)
    return points @ pose[:3, :3].T + pose[:3, 3]


def bin_index_array(dirs: np.ndarray, b_az: int, b_el: int):
    """kernels.py:49-57 — (b_a, b_e) int64 arrays for (n,3) nonzero vectors."""
    norms = np.linalg.norm(dirs, axis=1)
    az = np.arctan2(dirs[:, 1], dirs[:, 0])
    az = np.where(az < 0.0, az + TWO_PI, az)
    el = np.arcsin(np.clip(dirs[:, 2] / norms, -1.0, 1.0))
    b_a = np.clip((az / TWO_PI * b_az).astype(np.int64), 0, b_az - 1)
    b_e = np.clip(((el + np.pi / 2) / np.pi * b_el).astype(np.int64), 0, b_el - 1)
    return b_a, b_e


def world_to_voxel_array(origin, voxel_size, points):
    """grid.py:107-111 — floor((p - origin) / voxel_size) as int64."""
    origin = np.asarray(origin, dtype=np.float64)
    return np.floor((points - origin[np.newaxis, :]) / voxel_size).astype(np.int64)


def prepare(pts_map, sensor, origin, voxel_size, dims, half_extent, b_az, b_el):
    """integrator.py:192-204 (_prepare_chunk): centres (n,3) int64, ok (n,)
    bool and flat bins b_a*b_el+b_e (n,) int64 (0 where not ok)."""
    rays = pts_map - sensor
    norms = np.linalg.norm(rays, axis=1)
    ok = norms >= voxel_size
    centers = world_to_voxel_array(origin, voxel_size, pts_map)
    r = half_extent
    d = np.array(dims)
    ok &= np.all(centers >= r, axis=1) & np.all(centers <= d - 1 - r, axis=1)
    b_a = np.zeros(len(pts_map), dtype=np.int64)
    b_e = np.zeros(len(pts_map), dtype=np.int64)
    if np.any(ok):
        b_a[ok], b_e[ok] = bin_index_array(rays[ok], b_az, b_el)
    return centers, ok, b_a * b_el + b_e


def bin_direction(b_a: int, b_e: int, b_az: int, b_el: int) -> np.ndarray:
    """kernels.py:60-68 — unit vector at the bin's angular centre."""
    a = (b_a + 0.5) * TWO_PI / b_az
    e = (b_e + 0.5) * math.pi / b_el - math.pi / 2
    return np.array([math.cos(e) * math.cos(a), math.cos(e) * math.sin(a), math.sin(e)])


def _offset_cube(half: int):
    """kernels.py:81-87 — lexicographic (K^3,3) offsets and their L2 norms."""
    rng = np.arange(-half, half + 1)
    ox, oy, oz = np.meshgrid(rng, rng, rng, indexing="ij")
    offs = np.stack([ox.ravel(), oy.ravel(), oz.ravel()], axis=1)
    return offs, np.linalg.norm(offs.astype(np.float64), axis=1)


def bank_tables(size=21, b_az=40, b_el=40, shadow_radius=3.0, shadow_model="hemisphere",
                cone_half_angle_deg=30.0):
    """kernels.py:151-193 (+ :90-119 build_shadow_mask) as flat tables.

    Returns (distance_kernel uint32 (K,K,K), shadow_xyz int32 (total,3),
    shadow_start int64 (n_bins+1)) with bins in flat order b_a*b_el+b_e.
    """
    half = size // 2
    offs, norms = _offset_cube(half)
    runs = np.ceil(norms).astype(np.int64)
    runs[norms == 0.0] = 0
    runs = np.minimum(runs, 32)
    lut = np.array([run_mask(int(k)) for k in range(33)], dtype=np.uint32)
    dk = lut[runs].reshape(size, size, size)
    inside = norms <= shadow_radius
    cos_half = math.cos(math.radians(cone_half_angle_deg))
    lists = []
    for ba in range(b_az):
        for be in range(b_el):
            d = bin_direction(ba, be, b_az, b_el)
            dot = offs @ d
            if shadow_model == "hemisphere":
                keep = inside & (dot >= 0.0)
            elif shadow_model == "cone":
                keep = inside & ((norms == 0.0) | (dot >= norms * cos_half))
            else:
                raise ValueError(f"unknown shadow model {shadow_model!r}")
            keep |= norms == 0.0
            lists.append(offs[keep])
    counts = np.array([len(x) for x in lists], dtype=np.int64)
    start = np.zeros(len(lists) + 1, dtype=np.int64)
    np.cumsum(counts, out=start[1:])
    xyz = np.concatenate(lists).astype(np.int32) if lists else np.zeros((0, 3), np.int32)
    return dk, xyz, start
