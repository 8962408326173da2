"""Zero-isosurface extraction on the device (reference: mesher.py:26-110).

``extract_mesh(grid, iso)`` returns the reference's TriangleMesh bit for bit
(vertex order = sorted lattice-edge keys, triangle order = table slot, then
cell in C order; float64 vertices with the reference's operation order). The
work runs in libdbtsdf.so (csrc/mesh.cu) on the grid's device; only the
finished arrays cross PCIe.

The marching-cubes lookup tables ship with the package
(``data/mc_tables.npz``, the classic edge / triangle tables in the layout of
_mc_tables.py:9-324); the engine takes them as an input, so an ``.npz`` named
by ``$DBT_MC_TABLES`` or any mapping / module passed as ``tables=`` holding
EDGE_TABLE, TRI_TABLE, CORNER_OFFSETS, EDGE_BASE and EDGE_AXIS replaces them.
The reference package is not needed.
"""

from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from . import _native
from .errors import ConfigurationError
from .grid import VoxelGrid

_TABLE_FIELDS = (("EDGE_TABLE", 256), ("TRI_TABLE", 256 * 16), ("CORNER_OFFSETS", 24), ("EDGE_BASE", 36),
                 ("EDGE_AXIS", 12))


class McTables(ctypes.Structure):
    """dbt_mc_tables (include/dbtsdf.h)."""

    _fields_ = [("edge_table", ctypes.c_int32 * 256), ("tri_table", ctypes.c_int32 * (256 * 16)),
                ("corner_offsets", ctypes.c_int32 * 24), ("edge_base", ctypes.c_int32 * 36),
                ("edge_axis", ctypes.c_int32 * 12)]


@dataclass
class TriangleMesh:
    """mesher.py:26-34."""

    vertices: np.ndarray  # (v, 3) float64, world meters
    triangles: np.ndarray  # (f, 3) int64
    normals: np.ndarray | None = None  # (v, 3) unit vectors when present

    @property
    def is_empty(self) -> bool:
        return self.vertices.shape[0] == 0


def empty_mesh() -> TriangleMesh:
    """mesher.py:37-40."""
    return TriangleMesh(vertices=np.zeros((0, 3)), triangles=np.zeros((0, 3), dtype=np.int64))


_PKG_TABLES = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data", "mc_tables.npz")


def _table_source(source):
    """Default: the tables shipped with the package (data/mc_tables.npz: the
    classic Lorensen-Cline / Bourke marching-cubes edge and triangle tables in
    the order the reference's _mc_tables.py:9-324 lists them, with its corner
    and edge numbering); $DBT_MC_TABLES or tables= override them."""
    if source is None:
        return np.load(os.environ.get("DBT_MC_TABLES") or _PKG_TABLES)
    if isinstance(source, (str, os.PathLike)):
        return np.load(source)
    return source


_cache: dict = {}


def load_mc_tables(source=None) -> McTables:
    """Pack the five tables into the C struct (validated again by the engine)."""
    src = _table_source(source)
    key = id(src)
    hit = _cache.get(key)
    if hit is not None and hit[0] is src:
        return hit[1]
    t = McTables()
    for (name, n), (field, _) in zip(_TABLE_FIELDS, McTables._fields_):
        try:
            arr = src[name] if hasattr(src, "__getitem__") and not hasattr(src, name) else getattr(src, name)
        except (KeyError, AttributeError) as e:
            raise ConfigurationError(f"marching-cubes table {name} missing") from e
        a = np.ascontiguousarray(np.asarray(arr), dtype=np.int32).ravel()
        if a.size != n:
            raise ConfigurationError(f"marching-cubes table {name} has {a.size} entries, expected {n}")
        ctypes.memmove(getattr(t, field), a.ctypes.data, 4 * n)
    _cache[key] = (src, t)
    return t


class DeviceMesh:
    """Owning handle of a mesh kept in HBM (dbt_mesh*)."""

    def __init__(self, ptr, nv: int, nf: int):
        self.ptr, self.n_vertices, self.n_triangles = ptr, nv, nf

    def download(self) -> TriangleMesh:
        if self.n_triangles == 0:
            return empty_mesh()
        v = np.empty((self.n_vertices, 3), np.float64)
        f = np.empty((self.n_triangles, 3), np.int64)
        _native.check(_native.lib().dbt_mesh_download(self.ptr, _native.ptr(v), _native.ptr(f)))
        return TriangleMesh(vertices=v, triangles=f)

    def normals(self) -> np.ndarray:
        """Area-weighted unit vertex normals computed on the device."""
        _native.check(_native.lib().dbt_mesh_normals(self.ptr))
        out = np.empty((self.n_vertices, 3), np.float64)
        _native.check(_native.lib().dbt_mesh_download_normals(self.ptr, _native.ptr(out)))
        return out

    def device_pointers(self):
        v, f = ctypes.c_void_p(), ctypes.c_void_p()
        _native.check(_native.lib().dbt_mesh_device_buffers(self.ptr, ctypes.byref(v), ctypes.byref(f)))
        return v.value, f.value

    def close(self):
        if self.ptr:
            _native.lib().dbt_mesh_destroy(self.ptr)
            self.ptr = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # interpreter shutdown
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def extract_mesh_device(grid: VoxelGrid, iso: float = 0.0, tables=None) -> DeviceMesh:
    """Marching cubes left in device memory (for device-side consumers)."""
    t = load_mc_tables(tables)
    grid.push_host()
    out = ctypes.c_void_p()
    nv, nf = ctypes.c_int64(), ctypes.c_int64()
    _native.check(_native.lib().dbt_mesh_extract(grid.handle, float(iso), ctypes.byref(t), ctypes.byref(out),
                                                 ctypes.byref(nv), ctypes.byref(nf)))
    return DeviceMesh(out.value, int(nv.value), int(nf.value))


def extract_mesh(grid: VoxelGrid, iso: float = 0.0, tables=None) -> TriangleMesh:
    """Deterministic marching cubes at the given iso level in meters
    (mesher.py:43-110)."""
    with extract_mesh_device(grid, iso, tables) as m:
        return m.download()


def vertex_normals(mesh: TriangleMesh, device: int | None = None) -> TriangleMesh:
    """Attach area-weighted unit vertex normals (mesher.py:113-127), computed
    on the device bit-exactly; vertices with no incident non-degenerate
    triangle keep a zero normal."""
    if mesh.is_empty:
        return TriangleMesh(mesh.vertices, mesh.triangles, np.zeros((0, 3)))
    v = np.ascontiguousarray(mesh.vertices, dtype=np.float64)
    f = np.ascontiguousarray(mesh.triangles, dtype=np.int64)
    if v.ndim != 2 or v.shape[1] != 3 or f.ndim != 2 or f.shape[1] != 3:
        raise ConfigurationError("vertices and triangles must be (n, 3) arrays")
    dev = _native.default_device() if device is None else int(device)
    out = ctypes.c_void_p()
    _native.check(_native.lib().dbt_mesh_from_host(dev, _native.ptr(v), v.shape[0], _native.ptr(f), f.shape[0],
                                                   ctypes.byref(out)))
    with DeviceMesh(out.value, v.shape[0], f.shape[0]) as m:
        return TriangleMesh(mesh.vertices, mesh.triangles, m.normals())
