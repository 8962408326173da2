"""B200-native DB-TSDF scan integration (drop-in for the reference ``bitsdf``
integrate/query API, reference pkg/src/bitsdf/__init__.py:4-32).

The compute path is libdbtsdf.so (hand-written sm_100a CUDA, C ABI in
include/dbtsdf.h); this package is the host-side mirror of the reference
interface, plus the first consumer of the query path: device marching cubes
(``extract_mesh``). Metrics / file IO / CLI are outside this
build's scope.
"""

from .errors import (
    BitsdfError,
    ConfigurationError,
    CorruptionError,
    EvaluationError,
    FormatError,
    ResourceError,
)
from .grid import (
    VoxelGrid,
    decode_distance,
    memory_bytes,
    new_grid,
    observed_array,
    popcount_array,
    signed_distance,
    signed_distance_field,
    to_records,
    from_records,
)
from .integrator import (
    FrameStats,
    IntegrationParams,
    ScanFrame,
    integrate_frame,
    integrate_frames,
    integrate_frame_async,
    PendingFrame,
    integrate_point,
    integrate_points,
)
from .kernels import KernelBank, build_kernel_bank
from .mesher import TriangleMesh, empty_mesh, extract_mesh, extract_mesh_device, load_mc_tables, vertex_normals
from .snapshot import SNAPSHOT_MAGIC, load_grid, save_grid

__version__ = "0.1.0"

__all__ = [
    "VoxelGrid",
    "new_grid",
    "decode_distance",
    "signed_distance",
    "memory_bytes",
    "observed_array",
    "popcount_array",
    "signed_distance_field",
    "to_records",
    "from_records",
    "KernelBank",
    "build_kernel_bank",
    "ScanFrame",
    "IntegrationParams",
    "FrameStats",
    "integrate_frame",
    "integrate_frames",
    "integrate_frame_async",
    "PendingFrame",
    "integrate_point",
    "integrate_points",
    "TriangleMesh",
    "empty_mesh",
    "extract_mesh",
    "extract_mesh_device",
    "load_mc_tables",
    "vertex_normals",
    "SNAPSHOT_MAGIC",
    "save_grid",
    "load_grid",
    "BitsdfError",
    "ConfigurationError",
    "ResourceError",
    "FormatError",
    "CorruptionError",
    "EvaluationError",
    "__version__",
]
