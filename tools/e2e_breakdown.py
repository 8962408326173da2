"""Where the end-to-end time of integrate_frame goes (config 2, pinned f32
scans, L2 flushed between steps like bench.py): Python ScanFrame
construction, the C call (host wall, elapsed_ms) and the device span from
the H2D copy to the counter read-back (device_ms)."""
import os
os.environ.setdefault("DBT_DEVICE_MS", "1")  # FrameStats.device_ms on every call (timing events)
import ctypes
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, _native, build_kernel_bank, integrate_frame, new_grid  # noqa

w = workloads.get(2)
L = _native.lib()
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin)
n = 40
scans = [w.scan(k) for k in range(n)]
pinned = []
for s in scans:
    buf = ctypes.c_void_p()
    _native.check(L.dbt_host_alloc(s.nbytes, ctypes.byref(buf)))
    arr = np.ctypeslib.as_array((ctypes.c_float * s.size).from_address(buf.value)).reshape(s.shape)
    arr[...] = s
    pinned.append((buf, arr))
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
params = IntegrationParams()
rows = []
for rep in range(2):
    L.dbt_grid_reset(g.handle)
    for k in range(n):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        sf = ScanFrame(points=pinned[k][1], pose=w.poses[k])
        t1 = time.perf_counter()
        st = integrate_frame(g, bank, sf, params)
        t2 = time.perf_counter()
        # the C entry point alone (same scan again: its stamps are certified,
        # so this measures the fixed per-call cost on a redundant scan)
        pts, dt_ = sf.device_payload()
        pose = np.ascontiguousarray(sf.pose.reshape(-1))
        prm = params.native()
        cst = _native.Stats()
        t3 = time.perf_counter()
        _native.check(L.dbt_integrate_frame(g.handle, bank.device_handle(0), _native.ptr(pts), dt_, pts.shape[0],
                                            ctypes.c_void_p(pose.ctypes.data),
                                            ctypes.byref(prm), ctypes.byref(cst)))
        t4 = time.perf_counter()
        if rep == 1 and k >= 10:
            rows.append(((t1 - t0) * 1e6, (t2 - t1) * 1e6, st.elapsed_ms * 1e3, st.device_ms * 1e3,
                         (t4 - t3) * 1e6, cst.elapsed_ms * 1e3, cst.device_ms * 1e3))
r = np.array(rows).mean(axis=0)
print(f"per step us: ScanFrame {r[0]:.1f}  integrate_frame {r[1]:.1f}  (python-side total {r[2]:.1f})  "
      f"device span H2D..D2H {r[3]:.1f}  total {r[0] + r[1]:.1f}")
print(f"redundant re-integration via ctypes: wall {r[4]:.1f}  C-side wall {r[5]:.1f}  device span {r[6]:.1f}")
