"""Profiling driver: integrate the first N config-2 scans device-resident.

Usage: python tools/prof_cfg2.py [n_scans] [--repeat]
Scans are generated up front; each integrate_frame call is one launch
sequence (prep, shadow, sweep). With --repeat the same scans are integrated
twice (second pass = fully redundant scans).
"""
import sys

import numpy as np

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, new_grid  # noqa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4
w = workloads.get(2)
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin)
scans = [ScanFrame(points=w.scan(k), pose=w.poses[k]) for k in range(n)]
passes = 2 if "--repeat" in sys.argv else 1
for p in range(passes):
    for k, s in enumerate(scans):
        st = integrate_frame(g, bank, s, IntegrationParams())
        print(p, k, round(st.device_ms, 3), st.voxels_written, st.unique_centers, st.centers_skipped, flush=True)
