"""Workload for ncu captures of the device mesher and the exact
voxels_written kernels: the config-2 grid after its 100-scan trajectory, then
extract_mesh_device (iso 0) + vertex normals twice; with --exact also one
scan integrated with exact_voxels_written."""
import os
import sys

import numpy as np

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import (IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame,  # noqa: E402
                                   integrate_frames, new_grid)
from paper_2509_20081_b200.mesher import extract_mesh_device  # noqa: E402

w = workloads.get(2)
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(w.dims, w.voxel_size, w.origin)
for k0 in range(0, 96, 16):
    integrate_frames(g, bank, [ScanFrame(points=w.scan(k), pose=w.poses[k]) for k in range(k0, k0 + 16)],
                     IntegrationParams())
tabs = dict(np.load(os.path.join("tests", "golden", "mc_tables.npz")))
for _ in range(2):
    with extract_mesh_device(g, 0.0, tabs) as m:
        n = m.normals()
        print("mesh", m.n_vertices, m.n_triangles, float(np.abs(n).sum()))
if "--exact" in sys.argv:
    for k in range(96, 98):
        st = integrate_frame(g, bank, ScanFrame(points=w.scan(k), pose=w.poses[k]),
                             IntegrationParams(exact_voxels_written=True))
        print("exact voxels_written", st.voxels_written)
