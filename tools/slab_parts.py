"""What each rank of the slab mode does at N GPUs, on one GPU: the config-2
trajectory integrated into each interleaved part (bench.py's block width dealt
over N ranks), device-resident, L2 flushed per step. Prints the slowest part's
per-scan time and the implied all-rank throughput (the per-step NCCL point
broadcast, 786 KB, is not included)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import workloads
from paper_2509_20081_b200 import _native, build_kernel_bank
from paper_2509_20081_b200.grid import VoxelGrid

w = workloads.get(2); L = _native.lib()
scans = [torch.from_numpy(w.scan(k)).cuda() for k in range(w.n_scans)]
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
prm = _native.make_params()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for N in (1, 2, 4, 8):
    worst, applied = 0.0, 0
    for r in range(N):
        g = VoxelGrid(w.dims, w.voxel_size, w.origin, interleave=(min(64, w.dims[0] // (2 * N)), N, r)) if N > 1 else VoxelGrid(w.dims, w.voxel_size, w.origin)
        tot = 0.0
        for k in range(w.n_scans):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cnt = np.array([scans[k].shape[0]], np.int64); pose = np.ascontiguousarray(w.poses[k].reshape(-1))
            a.record()
            _native.check(L.dbt_integrate_device(g.handle, bank.device_handle(0), ctypes.c_void_p(scans[k].data_ptr()),
                                                 0, cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1,
                                                 ctypes.c_void_p(pose.ctypes.data), ctypes.byref(prm), ctypes.c_void_p(0)))
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
            if r == 0:
                st = (_native.Stats * 1)(); L.dbt_stats_read(g.handle, st, 1)
                applied += st[0].points_in - st[0].points_discarded
        worst = max(worst, tot)
        del g
    print(f"N={N}: slowest part {worst / w.n_scans * 1e3:.1f} us/scan, {applied / (worst / 1e3) / 1e6:.0f} M applied/s "
          f"all ranks (broadcast excluded)", flush=True)
