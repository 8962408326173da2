"""DBTSDF01 grid snapshots straight from the device layout (reference
io.py:449-486).

File: 8-byte magic ``DBTSDF01``, a 52-byte little-endian header
(nx, ny, nz u32; voxel_size, origin x/y/z f64; h_max, t_occ u8; 6 pad bytes),
then one 8-byte record {mask u32, sign u8, hits u8, reserved u16} per voxel
in linear order ix + nx*(iy + ny*iz). The F-order record stream of z-planes
[z0, z1) is one contiguous block, so both directions stream in z-chunks
through ``dbt_grid_to/from_records_range`` (the device transposes its C-order
records tile by tile): no full host copy of the grid, which for config 4 would
be 51 GB.
"""

from __future__ import annotations

import struct
from pathlib import Path

import numpy as np

from . import _native
from .errors import ConfigurationError, CorruptionError
from .grid import VOXEL_DTYPE, VoxelGrid, new_grid

SNAPSHOT_MAGIC = b"DBTSDF01"
_HEADER = struct.Struct("<3I4d2B6x")  # io.py:32
_CHUNK_BYTES = 256 << 20


def _planes_per_chunk(grid_dims) -> int:
    plane = grid_dims[0] * grid_dims[1] * 8
    return max(1, _CHUNK_BYTES // plane)


def save_grid(grid: VoxelGrid, path) -> None:
    """io.py:449-459: magic, header, voxel records in linear-index order."""
    path = Path(path)
    if grid.slab != (0, grid.dims[0]) or grid.interleave is not None:
        raise ConfigurationError("a snapshot needs the whole grid, not one slab")
    nx, ny, nz = grid.dims
    header = _HEADER.pack(nx, ny, nz, float(grid.voxel_size), *[float(o) for o in grid.origin],
                          int(grid.h_max), int(grid.t_occ))
    grid.push_host()
    zs = _planes_per_chunk(grid.dims)
    buf = np.empty(min(zs, nz) * nx * ny, dtype=VOXEL_DTYPE)
    L = _native.lib()
    with open(path, "wb") as f:
        f.write(SNAPSHOT_MAGIC)
        f.write(header)
        for z in range(0, nz, zs):
            z1 = min(z + zs, nz)
            part = buf[:(z1 - z) * nx * ny]
            _native.check(L.dbt_grid_to_records_range(grid.handle, z, z1, _native.ptr(part)))
            part.tofile(f)


def load_grid(path, device: int | None = None, memory_cap: int | None = None) -> VoxelGrid:
    """io.py:462-486: validate magic, header and payload length like the
    reference (CorruptionError), then stream the records onto the device."""
    path = Path(path)
    size = path.stat().st_size
    with open(path, "rb") as f:
        if f.read(8) != SNAPSHOT_MAGIC:
            f.seek(0)
            raise CorruptionError(f"{path}: bad snapshot magic {f.read(8)!r}")
        head = f.read(_HEADER.size)
        if len(head) < _HEADER.size:
            raise CorruptionError(f"{path}: snapshot header truncated")
        nx, ny, nz, voxel_size, ox, oy, oz, h_max, t_occ = _HEADER.unpack(head)
        if min(nx, ny, nz) < 1 or voxel_size <= 0:
            raise CorruptionError(f"{path}: degenerate snapshot header")
        n = nx * ny * nz
        body = size - 8 - _HEADER.size
        if body < n * 8:
            raise CorruptionError(f"{path}: snapshot payload short ({body} < {n * 8} bytes)")
        kw = {} if memory_cap is None else {"memory_cap": memory_cap}
        g = new_grid((nx, ny, nz), voxel_size, (ox, oy, oz), device=device, **kw)
        g.h_max, g.t_occ = int(h_max), int(t_occ)
        zs = _planes_per_chunk((nx, ny, nz))
        L = _native.lib()
        for z in range(0, nz, zs):
            z1 = min(z + zs, nz)
            part = np.fromfile(f, dtype=VOXEL_DTYPE, count=(z1 - z) * nx * ny)
            _native.check(L.dbt_grid_from_records_range(g.handle, z, z1, _native.ptr(part)))
    return g
