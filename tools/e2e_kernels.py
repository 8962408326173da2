import os
os.environ.setdefault("DBT_DEVICE_MS", "1")  # FrameStats.device_ms on every call (timing events)
import ctypes, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import workloads
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, _native, build_kernel_bank, integrate_frame, new_grid
w = workloads.get(2); L = _native.lib()
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin)
scans = [w.scan(k) for k in range(60)]
pinned = []
for s in scans:
    buf = ctypes.c_void_p(); _native.check(L.dbt_host_alloc(s.nbytes, ctypes.byref(buf)))
    arr = np.ctypeslib.as_array((ctypes.c_float * s.size).from_address(buf.value)).reshape(s.shape); arr[...] = s
    pinned.append(arr)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
p = IntegrationParams()
for mode in ("pinned", "pageable"):
    L.dbt_grid_reset(g.handle)
    for k in range(20):
        integrate_frame(g, bank, ScanFrame(points=pinned[k] if mode == "pinned" else scans[k], pose=w.poses[k]), p)
    L.dbt_profile_enable(g.handle, 1); L.dbt_profile_reset(g.handle)
    dev = []
    for k in range(20, 60):
        flush.zero_(); torch.cuda.synchronize()
        st = integrate_frame(g, bank, ScanFrame(points=pinned[k] if mode == "pinned" else scans[k], pose=w.poses[k]), p)
        dev.append(st.device_ms * 1e3)
    names = ctypes.create_string_buffer(32 * 16); ms = (ctypes.c_double * 16)(); cnt = (ctypes.c_int64 * 16)(); nk = ctypes.c_int32()
    L.dbt_profile_read(g.handle, names, ms, cnt, 16, ctypes.byref(nk))
    ks = {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): round(ms[i] / max(cnt[i], 1) * 1e3, 1) for i in range(nk.value)}
    L.dbt_profile_enable(g.handle, 0)
    print(mode, "device span us", round(float(np.mean(dev)), 1), ks)

# pinned scans: zero-copy vs one DMA copy (FLAG_STAGE_COPY), C entry point
for flags, name in ((0, "zero-copy"), (_native.FLAG_STAGE_COPY, "dma")):
    prm = _native.make_params(flags=flags)
    L.dbt_grid_reset(g.handle)
    L.dbt_profile_enable(g.handle, 1); L.dbt_profile_reset(g.handle)
    dev, wall = [], []
    for k in range(60):
        flush.zero_(); torch.cuda.synchronize()
        pose = np.ascontiguousarray(w.poses[k].reshape(-1)); st = _native.Stats()
        t0 = time.perf_counter()
        _native.check(L.dbt_integrate_frame(g.handle, bank.device_handle(0), ctypes.c_void_p(pinned[k].ctypes.data),
                                            _native.DBT_F32, len(pinned[k]), ctypes.c_void_p(pose.ctypes.data),
                                            ctypes.byref(prm), ctypes.byref(st)))
        if k >= 20:
            wall.append((time.perf_counter() - t0) * 1e6); dev.append(st.device_ms * 1e3)
    names = ctypes.create_string_buffer(32 * 16); ms = (ctypes.c_double * 16)(); cnt = (ctypes.c_int64 * 16)(); nk = ctypes.c_int32()
    L.dbt_profile_read(g.handle, names, ms, cnt, 16, ctypes.byref(nk))
    ks = {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): round(ms[i] / max(cnt[i], 1) * 1e3, 1) for i in range(nk.value)}
    L.dbt_profile_enable(g.handle, 0)
    print(name, "wall us", round(float(np.mean(wall)), 1), "device span us", round(float(np.mean(dev)), 1), ks)
