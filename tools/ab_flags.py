"""A/B engine variants on the config-2 trajectory (device-resident, per-kernel
CUDA-event times): default vs engine flags given on the command line."""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import _native, build_kernel_bank  # noqa: E402
from paper_2509_20081_b200.grid import VoxelGrid  # noqa: E402

w = workloads.get(2)
scans = [torch.from_numpy(w.scan(k)).cuda() for k in range(30)]
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
L = _native.lib()
variants = {"default": 0, "fused": _native.FLAG_FUSE_SHADOW, "no_skip": _native.FLAG_NO_SKIP,
            "no_dedup": _native.FLAG_NO_DEDUP, "generic": _native.FLAG_GENERIC_SWEEP}
if len(sys.argv) > 1:
    variants = {k: v for k, v in variants.items() if k in sys.argv[1:]}
for name, flags in variants.items():
    g = VoxelGrid(w.dims, w.voxel_size, w.origin)
    prm = _native.make_params(flags=flags)
    L.dbt_profile_enable(g.handle, 1)
    ev = []
    for rep in range(2):
        L.dbt_grid_reset(g.handle)
        L.dbt_profile_reset(g.handle)
        for k, s in enumerate(scans):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            cnt = np.array([s.shape[0]], np.int64)
            pose = np.ascontiguousarray(w.poses[k].reshape(-1))
            a.record()
            _native.check(L.dbt_integrate_device(g.handle, bank.device_handle(0), ctypes.c_void_p(s.data_ptr()), 0,
                                                 cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1,
                                                 ctypes.c_void_p(pose.ctypes.data),
                                                 ctypes.byref(prm), ctypes.c_void_p(0)))
            b.record()
            ev.append((a, b))
        torch.cuda.synchronize()
    ms = sum(a.elapsed_time(b) for a, b in ev[len(scans):]) / len(scans)
    names = ctypes.create_string_buffer(32 * 16)
    kms = (ctypes.c_double * 16)()
    cnt_ = (ctypes.c_int64 * 16)()
    nk = ctypes.c_int32()
    L.dbt_profile_read(g.handle, names, kms, cnt_, 16, ctypes.byref(nk))
    ks = {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): round(kms[i] / max(cnt_[i], 1) * 1e3, 1)
          for i in range(nk.value)}
    print(f"{name:9s} step {ms * 1e3:7.1f} us  kernels(us) {ks}", flush=True)
