"""Marching-cubes timing: device extract_mesh on the
final grid of a config's trajectory vs the reference algorithm on the host
(oracle/mc_oracle.py = mesher.py restated in the reference's own numpy calls).

    python tools/bench_mesh.py [--config 2] [--reps 10] [--cpu]

One JSON line per config: device ms (kernels + scans + the two count
read-backs, mesh left in HBM), e2e ms (incl. the D2H of vertices/triangles),
normals ms, per-kernel ms from the engine's profiling hooks, HBM bytes the
flag/count/group passes must move, and the CPU time when --cpu.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workloads  # noqa: E402
from paper_2509_20081_b200 import (IntegrationParams, ScanFrame, _native, build_kernel_bank,  # noqa: E402
                                   integrate_frames, new_grid)
from paper_2509_20081_b200.mesher import extract_mesh, extract_mesh_device, vertex_normals  # noqa: E402

TABLES = os.path.join(ROOT, "tests", "golden", "mc_tables.npz")


def prof_read(L, g):
    names = ctypes.create_string_buffer(32 * 32)
    ms = (ctypes.c_double * 32)()
    cnt = (ctypes.c_int64 * 32)()
    nk = ctypes.c_int32()
    L.dbt_profile_read(g.handle, names, ms, cnt, 32, ctypes.byref(nk))
    return {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): (ms[i], int(cnt[i])) for i in range(nk.value)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, nargs="+", default=[2])
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--scans", type=int, default=0, help="scans to integrate first (0 = whole trajectory)")
    ap.add_argument("--cpu", action="store_true", help="also time the host restatement (oracle/mc_oracle.py)")
    a = ap.parse_args()
    L = _native.lib()
    tabs = dict(np.load(TABLES))
    for cfg in a.config:
        w = workloads.get(cfg)
        n_scans = a.scans or len(w.poses)
        bank = build_kernel_bank(shadow_radius=w.shadow_radius)
        g = new_grid(w.dims, w.voxel_size, w.origin, memory_cap=1 << 44)
        for k0 in range(0, n_scans, 16):
            integrate_frames(g, bank, [ScanFrame(points=w.scan(k), pose=w.poses[k])
                                       for k in range(k0, min(n_scans, k0 + 16))], IntegrationParams())
        g.synchronize()
        with extract_mesh_device(g, 0.0, tabs) as m:  # warm-up (folds pending visits)
            nv, nf = m.n_vertices, m.n_triangles
        dev = []
        L.dbt_profile_enable(g.handle, 1)
        L.dbt_profile_reset(g.handle)
        for _ in range(a.reps):
            t0 = time.perf_counter()
            m = extract_mesh_device(g, 0.0, tabs)
            dev.append((time.perf_counter() - t0) * 1e3)
            m.close()
        prof = prof_read(L, g)
        L.dbt_profile_enable(g.handle, 0)
        e2e = []
        for _ in range(max(2, a.reps // 2)):
            t0 = time.perf_counter()
            mesh = extract_mesh(g, 0.0, tabs)
            e2e.append((time.perf_counter() - t0) * 1e3)
        nrm = []
        with extract_mesh_device(g, 0.0, tabs) as m:
            for _ in range(max(2, a.reps // 2)):
                t0 = time.perf_counter()
                _native.check(L.dbt_mesh_normals(m.ptr))
                nrm.append((time.perf_counter() - t0) * 1e3)
        t0 = time.perf_counter()
        vertex_normals(mesh)
        nrm_e2e = (time.perf_counter() - t0) * 1e3
        nvox = int(np.prod(w.dims))
        out = {
            "config": cfg, "dims": list(w.dims), "voxels": nvox, "scans": n_scans, "n_vertices": nv, "n_triangles": nf,
            "device_ms": round(float(np.median(dev)), 3), "e2e_ms": round(float(np.median(e2e)), 3),
            "normals_device_ms": round(float(np.median(nrm)), 3), "normals_e2e_ms": round(nrm_e2e, 3),
            "kernels_ms": {k: round(v[0] / max(v[1], 1), 4) for k, v in prof.items()},
            # flags: read 8 B record + write 1 B; count + select: >= 1 B each; group: 1 B; vertices: 1 B
            "min_hbm_bytes": nvox * (8 + 1 + 1 + 1 + 1 + 1),
            "gvoxels_per_s": round(nvox / (np.median(dev) * 1e-3) / 1e9, 2),
        }
        if a.cpu:
            from oracle import mc_oracle

            mk, sg, ht = g.download_range(0, w.dims[0])
            t0 = time.perf_counter()
            v, f = mc_oracle.mesh(mk, sg, ht, w.voxel_size, w.origin, 0.0, tabs)
            out["cpu_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
            t0 = time.perf_counter()
            n = mc_oracle.normals(v, f)
            out["cpu_normals_ms"] = round((time.perf_counter() - t0) * 1e3, 1)
            out["cpu_equal"] = bool(np.array_equal(v.view(np.uint64), mesh.vertices.view(np.uint64))
                                    and np.array_equal(f, mesh.triangles))
            out["cpu_normals_equal"] = bool(np.array_equal(n.view(np.uint64),
                                                           vertex_normals(mesh).normals.view(np.uint64)))
        print(json.dumps(out), flush=True)
        del g


if __name__ == "__main__":
    main()
