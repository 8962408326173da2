"""How much of the sweep's lowering work is redundant: config-4 scene on the
1000x1000x400 window grid (tests/cases.py), scans 0..N-1. Per scan: centres
swept, rows swept, lowering REDs issued (voxels_written, concurrent count),
the reference's serial count (exact_voxels_written, separate grid), and the
voxels whose mask actually changed (masks downloaded before / after)."""
import sys

import numpy as np

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, new_grid  # noqa

n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
cfg = int(sys.argv[2]) if len(sys.argv) > 2 else 4
w = workloads.get(cfg)
dims, org = ((1000, 1000, 400), (0.0, 90.0, -0.22)) if cfg == 4 else (w.dims, w.origin)
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
g = new_grid(dims, w.voxel_size, org, memory_cap=1 << 42)
ge = new_grid(dims, w.voxel_size, org, memory_cap=1 << 42)
g.release_host()
ge.release_host()
prev = g.download_range(0, dims[0])[0]
for k in range(n):
    s = ScanFrame(points=w.scan(k), pose=w.poses[k])
    st = integrate_frame(g, bank, s, IntegrationParams())
    se = integrate_frame(ge, bank, s, IntegrationParams(exact_voxels_written=True))
    cur = g.download_range(0, dims[0])[0]
    changed = int(np.count_nonzero(cur != prev))
    prev = cur
    print(f"scan {k}: applied {st.points_in - st.points_discarded} centres {st.unique_centers} rows {st.rows_swept} "
          f"REDs {st.voxels_written} serial {se.voxels_written} unique_changed {changed} "
          f"reds/changed {st.voxels_written / max(changed, 1):.2f} rows/centre {st.rows_swept / max(st.unique_centers, 1):.1f}",
          flush=True)
