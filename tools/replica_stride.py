"""What one rank of the replica mode does at N GPUs, on one GPU: integrate
its contiguous segment of the config-2 trajectory (bench.py's split: every
pass divided into N segments, reset per pass) into a whole replica,
device-resident, L2 flushed per step like bench.py. Prints the per-scan time
and applied returns/s for every rank's segment at N = 1, 2, 4, 8, plus the
pack + apply time of a merge (the all-reduce itself needs N GPUs)."""
import ctypes, sys
import numpy as np, torch
sys.path.insert(0, ".")
import workloads
from paper_2509_20081_b200 import IntegrationParams, _native, build_kernel_bank
from paper_2509_20081_b200.grid import VoxelGrid

w = workloads.get(2); L = _native.lib()
scans = [torch.from_numpy(w.scan(k)).cuda() for k in range(w.n_scans)]
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
prm = _native.make_params()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
g = VoxelGrid(w.dims, w.voxel_size, w.origin)
def seg_time(mine):
    for rep in range(2):
        L.dbt_grid_reset(g.handle)
        torch.cuda.synchronize()
        tot, applied = 0.0, 0
        for k in mine:
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cnt = np.array([scans[k].shape[0]], np.int64); pose = np.ascontiguousarray(w.poses[k].reshape(-1))
            a.record()
            _native.check(L.dbt_integrate_device(g.handle, bank.device_handle(0), ctypes.c_void_p(scans[k].data_ptr()),
                                                 0, cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1,
                                                 ctypes.c_void_p(pose.ctypes.data), ctypes.byref(prm),
                                                 ctypes.c_void_p(0)))
            b.record()
            torch.cuda.synchronize()
            tot += a.elapsed_time(b)
            st = (_native.Stats * 1)(); L.dbt_stats_read(g.handle, st, 1)
            applied += st[0].points_in - st[0].points_discarded
    return tot, applied


for N in (1, 2, 4, 8):
    res = [seg_time(list(range(r * w.n_scans // N, (r + 1) * w.n_scans // N))) for r in range(N)]
    worst = max(t for t, _ in res)
    total = sum(a for _, a in res)
    print(f"N={N}: segments of {w.n_scans // N} scans, slowest rank {worst:.2f} ms per pass, "
          f"{total / (worst / 1e3) / 1e6:.0f} M applied/s all ranks (merge excluded)", flush=True)
# merge kernels (pack + apply) on this grid
n = int(np.prod(w.dims))
mk = torch.empty(n, dtype=torch.uint8, device="cuda"); sg = torch.empty(n, dtype=torch.uint8, device="cuda")
dl = torch.empty(n, dtype=torch.float16, device="cuda")
_native.check(L.dbt_replica_mark(g.handle))
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    _native.check(L.dbt_replica_pack(g.handle, ctypes.c_void_p(mk.data_ptr()), ctypes.c_void_p(sg.data_ptr()), ctypes.c_void_p(dl.data_ptr()),
                       ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    _native.check(L.dbt_replica_apply(g.handle, ctypes.c_void_p(mk.data_ptr()), ctypes.c_void_p(sg.data_ptr()), ctypes.c_void_p(dl.data_ptr()),
                        255, 2, ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
b.record(); torch.cuda.synchronize()
print(f"pack+apply {a.elapsed_time(b) / 10:.3f} ms for {n * 4 / 1e6:.0f} MB of reduce buffers")
