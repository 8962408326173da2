import sys; sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tests")
import numpy as np, ctypes, torch
import cases
from paper_2509_20081_b200 import _native, build_kernel_bank, new_grid, integrate_frame, ScanFrame, IntegrationParams
from test_gpu_parity import TestReplicaMerge as T
import json
golden = json.load(open("/root/repo/tests/golden/golden.json"))
c = next(x for x in cases.small_cases() if x.name == "yaw_frames_f32")
ref = golden["cases"][c.name]
for sparse in (False, True):
    for reps in (1, 2, 3):
        gs = T().run(c, reps, 1, sparse=sparse)
        ok = []
        for g in gs:
            m, s, h = g.download_range(0, c.dims[0])
            ok.append((cases.sha(m) == ref["mask"], cases.sha(s) == ref["sign"], cases.sha(h) == ref["hits"]))
        print("sparse", sparse, "reps", reps, ok, flush=True)
