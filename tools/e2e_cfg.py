"""Where the end-to-end time of integrate_frame goes on a BASELINE config
(bench.py's window: prefill scans 0-9, scans 10-29 timed; L2 flushed):
host wall per call, the device span from the scan transfer to the counter
read-back (device_ms) and per-kernel CUDA-event times, for pinned scans read
zero-copy by prep, pinned scans staged by an H2D copy (FLAG_STAGE_COPY) and
pageable numpy scans.

usage: python tools/e2e_cfg.py [config=4]"""
import os
os.environ.setdefault("DBT_DEVICE_MS", "1")
import ctypes  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, _native, build_kernel_bank, integrate_frame, new_grid  # noqa

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.get(cfg)
L = _native.lib()
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin, memory_cap=1 << 42)
g.release_host()
scans = [w.scan(k) for k in range(30)]
pinned = []
for s in scans:
    buf = ctypes.c_void_p()
    _native.check(L.dbt_host_alloc(s.nbytes, ctypes.byref(buf)))
    arr = np.ctypeslib.as_array((ctypes.c_float * s.size).from_address(buf.value)).reshape(s.shape)
    arr[...] = s
    pinned.append(arr)
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")


def run(src, params, label):
    L.dbt_grid_reset(g.handle)
    for k in range(10):
        integrate_frame(g, bank, ScanFrame(points=src[k], pose=w.poses[k]), params)
    L.dbt_profile_enable(g.handle, 1)
    L.dbt_profile_reset(g.handle)
    wall, dev, ela = [], [], []
    for k in range(10, 30):
        flush.zero_()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = integrate_frame(g, bank, ScanFrame(points=src[k], pose=w.poses[k]), params)
        wall.append((time.perf_counter() - t0) * 1e6)
        dev.append(st.device_ms * 1e3)
        ela.append(st.elapsed_ms * 1e3)
    names = ctypes.create_string_buffer(32 * 16)
    ms = (ctypes.c_double * 16)()
    cn = (ctypes.c_int64 * 16)()
    nk = ctypes.c_int32()
    L.dbt_profile_read(g.handle, names, ms, cn, 16, ctypes.byref(nk))
    ks = {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): round(ms[i] / max(cn[i], 1) * 1e3, 1)
          for i in range(nk.value)}
    L.dbt_profile_enable(g.handle, 0)
    print(f"config {cfg} {label:28s} wall {np.mean(wall):7.1f} us  C call {np.mean(ela):7.1f}  device span "
          f"{np.mean(dev):7.1f}  kernels {ks}", flush=True)


run(pinned, IntegrationParams(), "pinned zero-copy")
run(scans, IntegrationParams(), "pageable numpy")
