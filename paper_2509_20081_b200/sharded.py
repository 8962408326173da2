"""Multi-GPU slab sharding of the voxel grid.

One process per GPU (torchrun). Rank r owns the contiguous x-slab
[x0_r, x1_r) of the global grid and allocates only that slab. Every voxel
update (mask AND, saturating hit count, occupied sign) is local to its voxel
and commutative, so a return's K^3 stamp splits exactly across slabs: there is
no halo exchange and no reduction of grid data. The only collective on the
data path is the broadcast of each launch's raw points (float32 xyz, 12 B per
return) from the rank that read them, over NCCL / NVLink; every rank then runs
the identical deterministic preprocessing against the GLOBAL grid dims
(discards, bins, first-return) and stamps only the part of each cube inside
its slab (csrc/integrate.cu clips the dx range per centre). FrameStats:
points_in / points_discarded are identical on every rank; the changed-cell
counts are summed with one all-reduce.

The functions below take a ``torch.distributed`` process group and work with
any backend (NCCL on the GPU box, gloo in the CPU tests).

``ReplicatedGrid`` is the data-parallel alternative for grids that fit one
GPU (config 2's is 87 MB of masks, even config 4's 51 GB fits 180 GB): each
rank integrates its own scans into a whole replica with no per-scan
collective, and an exact merge (three all-reduces) combines the replicas
when the global map is needed.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _native
from .errors import ConfigurationError
from .grid import VoxelGrid
from .integrator import FrameStats, IntegrationParams
from .kernels import KernelBank

DTYPE_CODES = {"float32": _native.DBT_F32, "float64": _native.DBT_F64}


def slab_bounds(nx: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous, disjoint x-slabs covering [0, nx); sizes differ by <= 1."""
    if not 0 <= rank < world:
        raise ValueError("rank outside [0, world)")
    return nx * rank // world, nx * (rank + 1) // world


def owner_of(x: int, nx: int, world: int) -> int:
    """Rank whose slab holds global plane x."""
    for r in range(world):
        a, b = slab_bounds(nx, world, r)
        if a <= x < b:
            return r
    raise ValueError("x outside the grid")


def broadcast_batch(points, counts, poses, dist, group=None, src: int = 0, device=None):
    """Broadcast one launch's scans from ``src``.

    points: torch tensor (n, 3) float32/float64 on ``src`` (ignored elsewhere);
    counts: int64 per-scan point counts, poses: (S, 4, 4) float64 — numpy on
    ``src``. Returns (points tensor on ``device``, counts ndarray, poses ndarray)
    on every rank. Metadata travels as one small int64/float64 tensor pair;
    the point payload is one broadcast of the raw buffer.
    """
    import torch

    rank = dist.get_rank(group)
    dev = torch.device("cpu") if device is None else torch.device(device)
    if rank == src:
        hdr = torch.tensor([int(points.shape[0]), 0 if points.dtype == torch.float32 else 1, len(counts)],
                           dtype=torch.int64, device=dev)
    else:
        hdr = torch.zeros(3, dtype=torch.int64, device=dev)
    dist.broadcast(hdr, src, group=group)
    n, code, S = (int(v) for v in hdr.tolist())
    if rank == src:
        meta_i = torch.as_tensor(np.asarray(counts, dtype=np.int64), device=dev)
        meta_f = torch.as_tensor(np.asarray(poses, dtype=np.float64).reshape(S, 16), device=dev)
        payload = points.to(dev).contiguous()
    else:
        meta_i = torch.zeros(S, dtype=torch.int64, device=dev)
        meta_f = torch.zeros((S, 16), dtype=torch.float64, device=dev)
        payload = torch.empty((n, 3), dtype=torch.float32 if code == 0 else torch.float64, device=dev)
    dist.broadcast(meta_i, src, group=group)
    dist.broadcast(meta_f, src, group=group)
    dist.broadcast(payload, src, group=group)
    return payload, meta_i.cpu().numpy(), meta_f.cpu().numpy().reshape(S, 4, 4)


def reduce_stats(stats: list, dist, group=None, device=None) -> list:
    """Sum the per-rank changed-cell counts (the only rank-dependent field)."""
    import torch

    dev = torch.device("cpu") if device is None else torch.device(device)
    t = torch.tensor([s.voxels_written for s in stats], dtype=torch.int64, device=dev)
    dist.all_reduce(t, group=group)
    out = []
    for s, w in zip(stats, t.cpu().tolist()):
        out.append(FrameStats(s.points_in, s.points_discarded, int(w), s.elapsed_ms, s.points_applied,
                              s.unique_centers, s.centers_skipped, s.bin_fallbacks, s.device_ms))
    return out


def _replica_stream(st):
    """Stream argument of the dbt_replica_* calls: NULL there means the
    grid's own stream, so torch's legacy default stream (handle 0) is passed
    as cudaStreamLegacy (0x1). Otherwise the pack/apply kernels would run on
    the grid's non-blocking stream, unordered with the collectives torch
    enqueues on the default stream."""
    return ctypes.c_void_p(st.cuda_stream or 1)


def _launch_device(grid: VoxelGrid, bank: KernelBank, points, dtype, counts, poses, prm, stream):
    """dbt_integrate_device on ``grid`` (asynchronous on ``stream``). A host
    mirror the caller may have written is uploaded first; afterwards it is
    dropped (it would be stale, and a later push_host would overwrite the
    device integration with it): the next read of grid.mask/sign/hits
    downloads the current grid."""
    grid.push_host()
    grid._host = None
    _native.check(_native.lib().dbt_integrate_device(
        grid.handle, bank.device_handle(grid.device), ctypes.c_void_p(points.data_ptr()), dtype,
        counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), len(counts),
        ctypes.c_void_p(poses.ctypes.data), ctypes.byref(prm), ctypes.c_void_p(stream.cuda_stream)))


class ShardedGrid:
    """This rank's share of a globally-sized grid, device resident: the
    contiguous slab ``slab_bounds`` gives, or (interleave=width) the x-blocks
    of ``width`` planes dealt round-robin over the ranks, which balances the
    1/r^2 return density around the sensor across ranks."""

    def __init__(self, dims, voxel_size, origin, rank: int, world: int, device: int | None = None,
                 interleave: int | None = None):
        self.dims = tuple(int(d) for d in dims)
        self.rank, self.world = rank, world
        if interleave:
            self.slab = (0, self.dims[0])
            self.local = VoxelGrid(self.dims, voxel_size, origin, device=device,
                                   interleave=(int(interleave), world, rank))
        else:
            self.slab = slab_bounds(self.dims[0], world, rank)
            self.local = VoxelGrid(self.dims, voxel_size, origin, device=device, slab=self.slab)

    @property
    def owned_x(self) -> np.ndarray:
        """Global x of this rank's planes, in storage order."""
        return self.local.owned_x

    def integrate_device(self, bank: KernelBank, points, counts, poses, params: IntegrationParams, stream=None):
        """Stamp this rank's slab from device-resident points (torch CUDA
        tensor). Asynchronous on ``stream`` (a torch.cuda.Stream or None for
        the current torch stream); read stats with ``stats``."""
        import torch

        dtype = _native.DBT_F32 if points.dtype == torch.float32 else _native.DBT_F64
        counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
        poses = np.ascontiguousarray(np.asarray(poses, dtype=np.float64).reshape(-1))
        st = torch.cuda.current_stream() if stream is None else stream
        prm = params.native()
        self._last_scans = len(counts)
        _launch_device(self.local, bank, points, dtype, counts, poses, prm, st)

    def stats(self) -> list:
        out = (_native.Stats * self._last_scans)()
        _native.check(_native.lib().dbt_stats_read(self.local.handle, out, self._last_scans))
        return [FrameStats.from_native(out[i]) for i in range(self._last_scans)]


class ReplicatedGrid:
    """Data-parallel replicas: every rank holds the whole grid (device
    resident) and integrates its OWN scans — no collective per scan. ``merge``
    makes all replicas equal to the grid that every rank's scans produce
    together (exact: see csrc/replica.cu): the ranks OR their dirty-brick
    flags, and the 16^3 bricks within a kernel radius of any rank's returns
    are reduced (MIN of the mask bit lengths and signs, float16 SUM of the
    hit deltas: 4 B per voxel of those bricks only). Until then each replica
    holds a valid partial map; reads that need the global map merge first.

    The scans between two merges must share (h_max, t_occ), as the hit-count
    combine depends on them."""

    def __init__(self, dims, voxel_size, origin, dist, group=None, device: int | None = None):
        self.dims = tuple(int(d) for d in dims)
        self.dist, self.group = dist, group
        self.local = VoxelGrid(self.dims, voxel_size, origin, device=device)
        self._params = None
        self._bufs = None
        self.mark()

    def mark(self):
        """Start a merge interval from the current records (after creation,
        reset or any host write). A host mirror is uploaded and then dropped:
        a later upload of it would replace the records and void the merge
        base (reading grid.mask/sign/hits again downloads a fresh one)."""
        self.local.push_host()
        self.local._host = None
        _native.check(_native.lib().dbt_replica_mark(self.local.handle))
        self._params = None

    def reset(self):
        _native.check(_native.lib().dbt_grid_reset(self.local.handle))
        self.mark()

    def _note_params(self, params: IntegrationParams):
        key = (params.h_max, params.t_occ)
        if self._params is None:
            self._params = key
        elif self._params != key:
            raise ConfigurationError("replica scans between two merges must share h_max and t_occ")

    def integrate_device(self, bank: KernelBank, points, counts, poses, params: IntegrationParams, stream=None):
        """Stamp this rank's scans (device tensor) into its replica,
        asynchronously on ``stream`` (torch.cuda.Stream or None = current)."""
        import torch

        self._note_params(params)
        dtype = _native.DBT_F32 if points.dtype == torch.float32 else _native.DBT_F64
        counts = np.ascontiguousarray(np.asarray(counts, dtype=np.int64))
        poses = np.ascontiguousarray(np.asarray(poses, dtype=np.float64).reshape(-1))
        st = torch.cuda.current_stream() if stream is None else stream
        prm = params.native()
        self._last_scans = len(counts)
        _launch_device(self.local, bank, points, dtype, counts, poses, prm, st)

    def integrate_frame(self, bank: KernelBank, scan, params: IntegrationParams) -> FrameStats:
        """integrate_frame on this rank's replica (synchronous; local stats)."""
        from .integrator import integrate_frame

        self._note_params(params)
        return integrate_frame(self.local, bank, scan, params)

    def stats(self) -> list:
        out = (_native.Stats * self._last_scans)()
        _native.check(_native.lib().dbt_stats_read(self.local.handle, out, self._last_scans))
        return [FrameStats.from_native(out[i]) for i in range(self._last_scans)]

    def _agreed_params(self, dev, reach: int = 0):
        """(h_max, t_occ) every rank that integrated since the last merge used,
        and the largest kernel radius any rank integrated with (collective).
        Ranks without scans take the parameters from the others, so all
        replicas fold the hit deltas identically; disagreement raises on
        every rank."""
        import torch

        have = self._params is not None
        h, t = self._params if have else (0, 0)
        v = torch.tensor([h if have else 1 << 20, t if have else 1 << 20, -h if have else 1 << 20,
                          -t if have else 1 << 20, -int(reach)], dtype=torch.int64, device=dev)
        self.dist.all_reduce(v, op=self.dist.ReduceOp.MIN, group=self.group)
        lo_h, lo_t, hi_h, hi_t, nreach = (int(x) for x in v.tolist())
        if lo_h == 1 << 20:  # no rank integrated: no deltas to fold
            return 255, 2, -nreach
        if (lo_h, lo_t) != (-hi_h, -hi_t):
            raise ConfigurationError("replica scans between two merges must share h_max and t_occ across ranks")
        return lo_h, lo_t, -nreach

    def merge(self, stream=None, sparse: bool = True):
        """All ranks: combine the replicas (collective). Returns when the
        merged records are enqueued on ``stream`` (current torch stream by
        default).

        sparse (default): only the 16^3 bricks within a kernel radius of a
        return some rank applied since the last merge travel — the ranks OR
        their dirty-brick flags (1 B per brick), then reduce 4 B per voxel of
        the selected bricks. sparse=False reduces the whole grid."""
        import torch

        dev = torch.device("cuda", self.local.device)
        st = torch.cuda.current_stream(dev) if stream is None else stream
        L = _native.lib()
        self.local.push_host()
        if not sparse:
            self._merge_dense(dev, st)
        else:
            nb, reach = ctypes.c_int64(), ctypes.c_int32()
            _native.check(L.dbt_replica_bricks(self.local.handle, ctypes.byref(nb), ctypes.byref(reach)))
            flags = torch.empty(int(nb.value), dtype=torch.uint8, device=dev)
            _native.check(L.dbt_replica_dirty(self.local.handle, ctypes.c_void_p(flags.data_ptr()),
                                              _replica_stream(st)))
            with torch.cuda.stream(st):
                self.dist.all_reduce(flags, op=self.dist.ReduceOp.MAX, group=self.group)
            h_max, t_occ, reach_all = self._agreed_params(dev, reach.value)
            n_sel = ctypes.c_int64()
            _native.check(L.dbt_replica_select(self.local.handle, ctypes.c_void_p(flags.data_ptr()), int(reach_all),
                                               ctypes.byref(n_sel), _replica_stream(st)))
            cells = int(n_sel.value) * 4096
            self.last_merge_voxels = cells
            if cells:
                ms = torch.empty(2 * cells, dtype=torch.uint8, device=dev)
                dl = torch.empty(cells, dtype=torch.float16, device=dev)
                _native.check(L.dbt_replica_pack_bricks(self.local.handle, ctypes.c_void_p(ms.data_ptr()),
                                                        ctypes.c_void_p(dl.data_ptr()), _replica_stream(st)))
                with torch.cuda.stream(st):
                    self.dist.all_reduce(ms, op=self.dist.ReduceOp.MIN, group=self.group)
                    self.dist.all_reduce(dl, op=self.dist.ReduceOp.SUM, group=self.group)
                _native.check(L.dbt_replica_apply_bricks(self.local.handle, ctypes.c_void_p(ms.data_ptr()),
                                                         ctypes.c_void_p(dl.data_ptr()), int(h_max), int(t_occ),
                                                         _replica_stream(st)))
                # the reduction buffers must outlive the enqueued apply
                ms.record_stream(st)
                dl.record_stream(st)
            else:
                _native.check(L.dbt_replica_apply_bricks(self.local.handle, None, None, int(h_max), int(t_occ),
                                                         _replica_stream(st)))
        self.local.pull_host()
        self._params = None

    def _merge_dense(self, dev, st):
        import torch

        n = self.dims[0] * self.dims[1] * self.dims[2]
        if self._bufs is None:
            self._bufs = (torch.empty(n, dtype=torch.uint8, device=dev), torch.empty(n, dtype=torch.uint8, device=dev),
                          torch.empty(n, dtype=torch.float16, device=dev))
        mk, sg, dl = self._bufs
        L = _native.lib()
        _native.check(L.dbt_replica_pack(self.local.handle, ctypes.c_void_p(mk.data_ptr()),
                                         ctypes.c_void_p(sg.data_ptr()), ctypes.c_void_p(dl.data_ptr()),
                                         _replica_stream(st)))
        with torch.cuda.stream(st):
            self.dist.all_reduce(mk, op=self.dist.ReduceOp.MIN, group=self.group)
            self.dist.all_reduce(sg, op=self.dist.ReduceOp.MIN, group=self.group)
            self.dist.all_reduce(dl, op=self.dist.ReduceOp.SUM, group=self.group)
        h_max, t_occ, _ = self._agreed_params(dev)
        self.last_merge_voxels = n
        _native.check(L.dbt_replica_apply(self.local.handle, ctypes.c_void_p(mk.data_ptr()),
                                          ctypes.c_void_p(sg.data_ptr()), ctypes.c_void_p(dl.data_ptr()),
                                          int(h_max), int(t_occ), _replica_stream(st)))
