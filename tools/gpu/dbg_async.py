"""Diagnostic: per-call host times of integrate_frame_async vs integrate_frame."""
import sys, time, ctypes
import numpy as np
sys.path.insert(0, ".")
import workloads
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, integrate_frame_async, new_grid, _native
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.get(cfg)
L = _native.lib()
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin, memory_cap=1 << 40)
scans = {}
for k in range(30):
    s = w.scan(k)
    buf = ctypes.c_void_p()
    _native.check(L.dbt_host_alloc(s.nbytes, ctypes.byref(buf)))
    arr = np.ctypeslib.as_array((ctypes.c_float * s.size).from_address(buf.value)).reshape(s.shape)
    arr[...] = s
    scans[k] = arr
p = IntegrationParams()
for k in range(10):
    integrate_frame(g, bank, ScanFrame(points=scans[k], pose=w.poses[k]), p)
g.synchronize()
t = []
pend = []
t0 = time.perf_counter()
for k in range(10, 30):
    a = time.perf_counter()
    pend.append(integrate_frame_async(g, bank, ScanFrame(points=scans[k], pose=w.poses[k]), p))
    b = time.perf_counter()
    c = b
    if len(pend) > 2:
        r = pend.pop(0).result()
        c = time.perf_counter()
    t.append((round((b - a) * 1e6), round((c - b) * 1e6)))
for f in pend:
    f.result()
print("async total per step us", (time.perf_counter() - t0) / 20 * 1e6)
print("issue/collect us per call", t)
L.dbt_grid_reset(g.handle)
for k in range(10):
    integrate_frame(g, bank, ScanFrame(points=scans[k], pose=w.poses[k]), p)
g.synchronize()
t0 = time.perf_counter()
for k in range(10, 30):
    integrate_frame(g, bank, ScanFrame(points=scans[k], pose=w.poses[k]), p)
print("sync per step us", (time.perf_counter() - t0) / 20 * 1e6)
