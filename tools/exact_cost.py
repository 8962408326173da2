"""Cost of DBT_FLAG_EXACT_WRITTEN (the reference's serial voxels_written) on a
config's trajectory: device ms per scan with and without it, per kernel."""
import os
os.environ.setdefault("DBT_DEVICE_MS", "1")  # FrameStats.device_ms on every call (timing events)
import ctypes, json, sys
import numpy as np
sys.path.insert(0, ".")
import workloads
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, _native, build_kernel_bank, integrate_frame, new_grid

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 2
n_scans = int(sys.argv[2]) if len(sys.argv) > 2 else 40
w = workloads.get(cfg); L = _native.lib()
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin, memory_cap=1 << 44)
scans = [w.scan(k) for k in range(n_scans)]
for exact in (False, True):
    L.dbt_grid_reset(g.handle)
    p = IntegrationParams(exact_voxels_written=exact)
    L.dbt_profile_enable(g.handle, 1); L.dbt_profile_reset(g.handle)
    dev, written = [], []
    for k in range(n_scans):
        st = integrate_frame(g, bank, ScanFrame(points=scans[k], pose=w.poses[k]), p)
        dev.append(st.device_ms); written.append(st.voxels_written)
    names = ctypes.create_string_buffer(32 * 16); ms = (ctypes.c_double * 16)(); cnt = (ctypes.c_int64 * 16)(); nk = ctypes.c_int32()
    L.dbt_profile_read(g.handle, names, ms, cnt, 16, ctypes.byref(nk))
    ks = {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): round(ms[i] / max(cnt[i], 1), 4) for i in range(nk.value)}
    L.dbt_profile_enable(g.handle, 0)
    print(json.dumps({"config": cfg, "exact": exact, "scans": n_scans, "device_ms_per_scan": round(float(np.mean(dev)), 4),
                      "voxels_written_total": int(sum(written)), "kernels_ms": ks}), flush=True)
