"""Dump rays whose device bin differs from numpy's (knife-edge diagnosis)."""
import math
import sys

import numpy as np

sys.path.insert(0, ".")
import workloads  # noqa: E402
from oracle import prep  # noqa: E402
from paper_2509_20081_b200 import kernels as K  # noqa: E402

out = []
for cfg, ks in ((1, [0]), (2, [0, 1, 2]), (3, [0, 1, 2])):
    w = workloads.get(cfg)
    for k in ks:
        pts = w.scan(k).astype(np.float64)
        pose = w.poses[k]
        rays = prep.transform(pts, pose) - pose[:3, 3]
        rays = rays[np.linalg.norm(rays, axis=1) > 0]
        ra, re = prep.bin_index_array(rays, 40, 40)
        da, de = K.bin_index_array(rays, 40, 40)
        bad = np.nonzero((ra != da) | (re != de))[0]
        print(cfg, k, len(rays), "mismatch", len(bad))
        for i in bad:
            r = rays[i]
            n = np.linalg.norm(r)
            az = math.atan2(r[1], r[0])
            print("  ray", repr(r.tolist()), "numpy", int(ra[i]), int(re[i]), "dev", int(da[i]), int(de[i]),
                  "np_atan2", repr(float(np.arctan2(r[1], r[0]))), "np_asin", repr(float(np.arcsin(r[2] / n))))
            out.append(r)
np.save("gpurun_out/bad_rays.npy", np.array(out))
