"""Batched e2e (config-5 shape): 32 pinned scans per dbt_integrate_scans call,
zero-copy reads in preprocessing vs one DMA copy per scan (FLAG_STAGE_COPY)."""
import os
os.environ.setdefault("DBT_DEVICE_MS", "1")  # FrameStats.device_ms on every call (timing events)
import ctypes
import sys
import time

import numpy as np

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import _native, build_kernel_bank, new_grid  # noqa: E402

w = workloads.get(3)
L = _native.lib()
B = int(sys.argv[1]) if len(sys.argv) > 1 else 32
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin, memory_cap=1 << 42)
scans = [w.scan(k) for k in range(2 * B)]
pinned = []
for s in scans:
    buf = ctypes.c_void_p()
    _native.check(L.dbt_host_alloc(s.nbytes, ctypes.byref(buf)))
    arr = np.ctypeslib.as_array((ctypes.c_float * s.size).from_address(buf.value)).reshape(s.shape)
    arr[...] = s
    pinned.append(arr)
for flags, name in ((0, "zero-copy"), (_native.FLAG_STAGE_COPY, "dma-staged")):
    prm = _native.make_params(flags=flags)
    for rep in range(3):
        L.dbt_grid_reset(g.handle)
        t = []
        for j in range(2):
            ks = range(j * B, (j + 1) * B)
            ptrs = (ctypes.c_void_p * B)(*[pinned[k].ctypes.data for k in ks])
            counts = np.array([len(pinned[k]) for k in ks], np.int64)
            poses = np.ascontiguousarray(np.stack([w.poses[k] for k in ks]).reshape(-1))
            out = (_native.Stats * B)()
            t0 = time.perf_counter()
            _native.check(L.dbt_integrate_scans(g.handle, bank.device_handle(0), ptrs, _native.DBT_F32,
                                                counts.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), B,
                                                ctypes.c_void_p(poses.ctypes.data), ctypes.byref(prm), out))
            t.append((time.perf_counter() - t0) * 1e3)
        print(f"{name}: {t[0]:.2f} / {t[1]:.2f} ms per {B}-scan call (device {out[0].device_ms:.2f} ms)")

# the same through the public API (ScanFrame + integrate_frames)
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, integrate_frames  # noqa: E402

params = IntegrationParams()
import torch  # noqa: E402

flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
for rep in range(4):
    L.dbt_grid_reset(g.handle)
    t = []
    for j in range(2):
        ks = range(j * B, (j + 1) * B)
        if rep >= 2:  # L2 flushed before the call, like bench.py
            flush.zero_()
            torch.cuda.synchronize()
        t0 = time.perf_counter()
        frames = [ScanFrame(points=pinned[k], pose=w.poses[k]) for k in ks]
        t1 = time.perf_counter()
        sts = integrate_frames(g, bank, frames, params)
        t.append(((t1 - t0) * 1e3, (time.perf_counter() - t1) * 1e3))
    print(("flushed " if rep >= 2 else "") + "public API: ScanFrames %.2f ms + integrate_frames %.2f ms | %.2f + %.2f" % (t[0] + t[1]))
