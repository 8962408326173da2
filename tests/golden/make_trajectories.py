"""Generate tests/golden/trajectories.json by running the REFERENCE
implementation over the multi-scan trajectories of tests/cases.py
(``trajectories()``): after every scan the sha256 prefixes of the
reference's mask / sign / hits arrays and its FrameStats are stored, plus the
hash of every input scan (generator drift on another host is then reported
as such, not as a kernel mismatch).

Runs only in the build container (the reference is importable from
/root/reference/pkg/src; it does not exist on the GPU box). The trajectories
run in parallel worker processes; config 3 / config-4 window take minutes.

    python tests/golden/make_trajectories.py [name ...]
"""

from __future__ import annotations

import json
import sys
import time
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))
sys.path.insert(0, str(HERE.parent.parent))
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402


def run(t: cases.Trajectory) -> dict:
    from bitsdf.grid import new_grid  # reference
    from bitsdf.integrator import IntegrationParams, ScanFrame, integrate_frame
    from bitsdf.kernels import build_kernel_bank

    w = t.workload()
    bank = build_kernel_bank(**t.bank)
    g = new_grid(t.dims, t.voxel_size, t.origin, memory_cap=1 << 40)
    params = IntegrationParams()
    out = {"config": t.config, "scans": list(t.scans), "dims": list(t.dims), "voxel_size": t.voxel_size,
           "origin": list(t.origin), "bank": t.bank, "per_scan": []}
    t0 = time.perf_counter()
    ref_s = 0.0
    for k in t.scan_ids():
        pts, pose = w.scan(k), w.poses[k]
        a = time.perf_counter()
        st = integrate_frame(g, bank, ScanFrame(points=pts, pose=pose), params, threads=2)
        ref_s += time.perf_counter() - a
        out["per_scan"].append({
            "scan": k, "input": cases.scan_hash(pts, pose),
            "stats": [st.points_in, st.points_discarded, st.voxels_written],
            "mask": cases.sha(g.mask), "sign": cases.sha(g.sign), "hits": cases.sha(g.hits)})
        print(f"{t.name} scan {k}: {st.points_in} in, {st.points_discarded} discarded, "
              f"{st.voxels_written} written, {time.perf_counter() - t0:.0f}s", flush=True)
    out["observed"] = int(np.count_nonzero(~((g.mask == 0xFFFFFFFF) & (g.hits == 0))))
    out["occupied"] = int(np.count_nonzero(g.sign == 0))
    out["ref_integrate_seconds"] = round(ref_s, 1)
    return out


def main():
    names = sys.argv[1:]
    todo = [t for t in cases.trajectories() if not names or t.name in names]
    out_path = HERE / "trajectories.json"
    gold = json.loads(out_path.read_text()) if out_path.exists() else {}
    import platform
    gold["_meta"] = {"generator": "tests/golden/make_trajectories.py (reference bitsdf from /root/reference/pkg/src)",
                     "numpy": np.__version__, "python": platform.python_version()}
    with ProcessPoolExecutor(max_workers=len(todo)) as ex:
        for t, r in zip(todo, ex.map(run, todo)):
            gold[t.name] = r
            out_path.write_text(json.dumps(gold, indent=1, sort_keys=True))
    print("wrote", out_path)


if __name__ == "__main__":
    main()
