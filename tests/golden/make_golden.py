"""Generate tests/golden/golden.json by running the REFERENCE implementation.

Runs only in the build container, where the reference is importable from
/root/reference/pkg/src (it does not exist on the GPU box). For every case in
tests/cases.py it integrates the seeded inputs with the reference's own
``integrate_frame`` / ``integrate_point`` and stores sha256 prefixes of the
final mask/sign/hits arrays plus the FrameStats, the input hashes, the kernel
bank table hashes (``build_kernel_bank``) and the reference's
``bin_index_array`` output on fixed direction sets.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py [--fast]
"""

from __future__ import annotations

import json
import platform
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from bitsdf.grid import new_grid  # noqa: E402  (reference)
from bitsdf.integrator import IntegrationParams, ScanFrame, integrate_frame, integrate_point  # noqa: E402
from bitsdf.kernels import bin_index_array, build_kernel_bank  # noqa: E402
from bitsdf import io as bio  # noqa: E402


def run_case(c: cases.Case) -> dict:
    bank = build_kernel_bank(**c.bank)
    g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 40)
    if c.init is not None:
        g.mask[...] = c.init[0]
        g.sign[...] = c.init[1]
        g.hits[...] = c.init[2]
    params = IntegrationParams(**c.params)
    stats = []
    t0 = time.perf_counter()
    for pts, pose in c.frames:
        st = integrate_frame(g, bank, ScanFrame(points=pts, pose=pose), params, threads=8)
        stats.append([st.points_in, st.points_discarded, st.voxels_written])
    applied = None
    if c.hits is not None:
        applied = 0
        for p, s in zip(*c.hits):
            applied += integrate_point(g, bank, p, s, params) == "applied"
    el = time.perf_counter() - t0
    out = {
        "input": c.input_hash(),
        "mask": cases.sha(g.mask),
        "sign": cases.sha(g.sign),
        "hits": cases.sha(g.hits),
        "stats": stats,
        "applied": applied,
        "observed": int(np.count_nonzero(~((g.mask == 0xFFFFFFFF) & (g.hits == 0)))),
        "occupied": int(np.count_nonzero(g.sign == 0)),
        "ref_seconds": round(el, 2),
    }
    if not c.slow:
        # the reference's own DBTSDF01 snapshot of the final grid (io.py:449-459)
        # with the case's h_max / t_occ in the header
        import hashlib
        import tempfile
        g.h_max, g.t_occ = params.h_max, params.t_occ
        with tempfile.TemporaryDirectory() as td:
            fp = Path(td) / "g.dbtsdf"
            bio.save_grid(g, fp)
            raw = fp.read_bytes()
        out["snapshot"] = {"bytes": len(raw), "sha": hashlib.sha256(raw).hexdigest()[:32]}
    print(f"{c.name}: {el:.1f}s stats={stats} applied={applied}", flush=True)
    return out


def main():
    fast = "--fast" in sys.argv
    out_path = HERE / "golden.json"
    gold = json.loads(out_path.read_text()) if out_path.exists() else {}
    gold["_meta"] = {
        "generator": "tests/golden/make_golden.py (reference bitsdf imported from /root/reference/pkg/src)",
        "numpy": np.__version__,
        "python": platform.python_version(),
        "machine": platform.processor() or platform.machine(),
    }
    gold.setdefault("banks", {})
    for spec in cases.bank_specs():
        gold["banks"][cases.bank_key(spec)] = cases.bank_hashes(build_kernel_bank(**spec))
    gold.setdefault("bins", {})
    for name, dirs in cases.bin_dir_sets().items():
        b_a, b_e = bin_index_array(dirs, 40, 40)
        gold["bins"][name] = {"input": cases.sha(dirs), "b_a": cases.sha(b_a.astype(np.int64)),
                              "b_e": cases.sha(b_e.astype(np.int64))}
    gold.setdefault("cases", {})
    if "--only-mesh" in sys.argv:
        # the reference's marching-cubes tables (inputs the device mesher takes
        # from its caller) and its extract_mesh output on final golden grids
        from bitsdf import _mc_tables as T
        from bitsdf.mesher import extract_mesh, vertex_normals
        np.savez(HERE / "mc_tables.npz", EDGE_TABLE=T.EDGE_TABLE, TRI_TABLE=T.TRI_TABLE,
                 CORNER_OFFSETS=T.CORNER_OFFSETS, EDGE_BASE=T.EDGE_BASE, EDGE_AXIS=T.EDGE_AXIS)
        wanted = ("frame500_default", "arbitrary_state", "nonfresh_cone_h200_t2", "k9_bins8", "cfg2_scans0-2")
        for c in cases.small_cases() + cases.config_cases(include_slow=False):
            if c.name not in wanted:
                continue
            bank = build_kernel_bank(**c.bank)
            g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 40)
            if c.init is not None:
                g.mask[...], g.sign[...], g.hits[...] = c.init
            params = IntegrationParams(**c.params)
            for pts, pose in c.frames:
                integrate_frame(g, bank, ScanFrame(points=pts, pose=pose), params, threads=8)
            assert cases.sha(g.mask) == gold["cases"][c.name]["mask"]
            out = {}
            for iso in (0.0, 0.1):
                m = extract_mesh(g, iso)
                out[repr(iso)] = {"vertices": cases.sha(np.ascontiguousarray(m.vertices, dtype=np.float64)),
                                  "triangles": cases.sha(np.ascontiguousarray(m.triangles, dtype=np.int64)),
                                  "n_vertices": int(m.vertices.shape[0]), "n_triangles": int(m.triangles.shape[0]),
                                  "normals": cases.sha(vertex_normals(m).normals)}
            gold["cases"][c.name]["mesh"] = out
            print(c.name, out, flush=True)
        out_path.write_text(json.dumps(gold, indent=1, sort_keys=True))
        print("wrote", out_path)
        return
    if "--only-deskew" in sys.argv:
        # motion-compensated frames through the reference's integrate_frame
        # (and the hash of its motion_compensate output per frame). The
        # reference's yaw mode calls Rotation.from_euler("z", angles) with a
        # 1-D angle array, which scipy >= 1.15 rejects (it wants (n, 1) for a
        # single axis); for that call only, the angles are reshaped to (n, 1)
        # — the same rotations older scipy versions built.
        from scipy.spatial.transform import Rotation
        from bitsdf.integrator import motion_compensate
        orig = Rotation.from_euler

        def from_euler_1d(seq, angles, degrees=False):
            a = np.asarray(angles)
            if len(seq) == 1 and a.ndim == 1:
                a = a[:, None]
            return orig(seq, a, degrees=degrees)

        Rotation.from_euler = staticmethod(from_euler_1d)
        gold.setdefault("deskew", {})
        for c in cases.deskew_cases():
            bank = build_kernel_bank(**c.bank)
            g = new_grid(c.dims, c.voxel_size, c.origin, memory_cap=1 << 40)
            params = IntegrationParams(**c.params)
            stats, moved = [], []
            t0 = time.perf_counter()
            for pts, pose, prev, ts in c.frames:
                st = integrate_frame(g, bank, ScanFrame(points=pts, pose=pose, timestamps=ts, prev_pose=prev), params,
                                     threads=8)
                stats.append([st.points_in, st.points_discarded, st.voxels_written])
                k = slice(None, None, params.downsample)
                sc = ScanFrame(points=np.asarray(pts, np.float64)[k], pose=pose,
                               timestamps=None if ts is None else ts[k], prev_pose=prev)
                moved.append(cases.sha(motion_compensate(sc, params.compensation).points))
            gold["deskew"][c.name] = {"input": c.input_hash(), "mask": cases.sha(g.mask), "sign": cases.sha(g.sign),
                                      "hits": cases.sha(g.hits), "stats": stats, "points": moved,
                                      "ref_seconds": round(time.perf_counter() - t0, 2)}
            print(c.name, gold["deskew"][c.name], flush=True)
        out_path.write_text(json.dumps(gold, indent=1, sort_keys=True))
        print("wrote", out_path)
        return
    if "--only-snapshots" in sys.argv:
        # add the snapshot hashes of the small cases; every other stored value
        # must come out unchanged
        for c in cases.small_cases():
            r = run_case(c)
            old = gold["cases"][c.name]
            for k in ("input", "mask", "sign", "hits", "stats", "applied"):
                assert old[k] == r[k], (c.name, k)
            old["snapshot"] = r["snapshot"]
        out_path.write_text(json.dumps(gold, indent=1, sort_keys=True))
        print("wrote", out_path)
        return
    all_cases = cases.small_cases() + cases.config_cases(include_slow=not fast)
    for c in all_cases:
        gold["cases"][c.name] = run_case(c)
        out_path.write_text(json.dumps(gold, indent=1, sort_keys=True))
    print("wrote", out_path)


if __name__ == "__main__":
    main()
