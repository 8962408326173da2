"""Profiling driver: integrate the first N scans of a BASELINE config
device-resident, flushing L2 (256 MB write) between scans like bench.py.

Usage: python tools/prof_cfg.py CONFIG N_SCANS [--window]
--window: config 4 on the 1000x1000x400 parity window instead of the full grid.
Prints per scan: device ms, voxels_written, unique centres, centres skipped.
"""
import sys

import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, new_grid  # noqa

cfg = int(sys.argv[1])
n = int(sys.argv[2])
w = workloads.get(cfg)
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
if "--window" in sys.argv:
    g = new_grid((1000, 1000, 400), w.voxel_size, (0.0, 90.0, -0.22))
else:
    g = new_grid(w.dims, w.voxel_size, w.origin, memory_cap=1 << 42)
scans = [ScanFrame(points=w.scan(k), pose=w.poses[k]) for k in range(n)]
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k, s in enumerate(scans):
    flush.fill_(k & 0xFF)
    torch.cuda.synchronize()
    st = integrate_frame(g, bank, s, IntegrationParams())
    print(k, round(st.device_ms, 3), st.points_applied, st.voxels_written, st.unique_centers, st.centers_skipped,
          flush=True)
