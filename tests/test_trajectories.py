"""GPU parity over whole trajectories: the regime bench.py times.

The reference's grid hashes after EVERY scan of each trajectory of
tests/cases.py (``trajectories()``: config 2 in full, 100 scans; config 3
scans 0-127, also the config-5 batched case; the config-4 scene at 0.02 m
on its 1000x1000x400 window, scans 0-29) are stored in
tests/golden/trajectories.json by tests/golden/make_trajectories.py, which
imports the reference itself (integrator.py:207-287). Here the engine runs
the same scans through its default path — stamp certificates carried across
launches, neighbour-dominance culling, lazy shadow-visit folds, the PDL sweep
launch — and its downloaded grid must hash identically at every checkpoint:

* scan by scan through ``integrate_frame`` (synchronous calls);
* in batches of 8, 32 and 128 scans per launch (``integrate_frames``,
  config 5's batch sizes);
* device-resident launches queued back to back without a host sync
  (``dbt_integrate_device``, exactly what bench.py times);
* config 2 with ``exact_voxels_written``: every FrameStats field equals the
  reference's, scan by scan.
"""

import ctypes
import json
import os
from concurrent.futures import ProcessPoolExecutor
from pathlib import Path

import numpy as np
import pytest

import cases
from paper_2509_20081_b200 import (IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame,
                                   integrate_frames, new_grid)
from paper_2509_20081_b200 import _native

pytestmark = pytest.mark.gpu

GOLD = json.loads((Path(__file__).resolve().parent / "golden" / "trajectories.json").read_text())
TRAJ = {t.name: t for t in cases.trajectories()}
_SCANS = {}


def _scan(args):
    cfg, k = args
    import workloads

    return workloads.get(cfg).scan(k)


def scans_of(t: cases.Trajectory):
    """The trajectory's scans (ray cast once per session, in a process pool),
    checked against the input hashes the reference run stored."""
    if t.name not in _SCANS:
        w = t.workload()
        ids = t.scan_ids()
        if t.config <= 2:
            pts = [w.scan(k) for k in ids]
        else:
            with ProcessPoolExecutor(max_workers=min(len(ids), os.cpu_count() or 1)) as ex:
                pts = list(ex.map(_scan, [(t.config, k) for k in ids]))
        ref = GOLD[t.name]["per_scan"]
        for k, p, r in zip(ids, pts, ref):
            assert r["scan"] == k
            assert cases.scan_hash(p, w.poses[k]) == r["input"], f"generator drift at scan {k}"
        _SCANS[t.name] = [(p, w.poses[k]) for k, p in zip(ids, pts)]
    return _SCANS[t.name]


def fresh(t):
    g = new_grid(t.dims, t.voxel_size, t.origin, memory_cap=1 << 42)
    return g, build_kernel_bank(**t.bank)


def assert_grid(g, t, i, how):
    """Grid after scan index i (0-based within the trajectory) equals the
    reference's."""
    ref = GOLD[t.name]["per_scan"][i]
    m, s, h = g.download_range(0, t.dims[0])
    where = f"{t.name} after scan {ref['scan']} ({how})"
    assert cases.sha(m) == ref["mask"], f"mask differs from the reference {where}"
    assert cases.sha(s) == ref["sign"], f"sign differs from the reference {where}"
    assert cases.sha(h) == ref["hits"], f"hits differ from the reference {where}"


def checkpoints(t):
    n = len(t.scan_ids())
    # every scan on config 2 (21.7 M voxels); every 5th (config-4 window) or
    # 16th (config 3, 128 scans) + the last on the 4e8-voxel grids (each
    # check downloads and hashes 2.4 GB)
    step = 1 if t.config <= 2 else (5 if len(t.scan_ids()) <= 40 else 16)
    return sorted(set(range(step - 1, n, step)) | {n - 1})


@pytest.mark.parametrize("name", list(TRAJ))
def test_trajectory_scan_by_scan(name):
    t = TRAJ[name]
    frames = scans_of(t)
    g, bank = fresh(t)
    g.release_host()
    cps = set(checkpoints(t))
    ref = GOLD[name]["per_scan"]
    for i, (p, pose) in enumerate(frames):
        st = integrate_frame(g, bank, ScanFrame(points=p, pose=pose), IntegrationParams())
        assert [st.points_in, st.points_discarded] == ref[i]["stats"][:2], f"scan {ref[i]['scan']} counts"
        if i in cps:
            assert_grid(g, t, i, "integrate_frame, scan by scan")


@pytest.mark.parametrize("batch", [8, 32, 128])
@pytest.mark.parametrize("name", list(TRAJ))
def test_trajectory_batched(name, batch):
    t = TRAJ[name]
    frames = scans_of(t)
    g, bank = fresh(t)
    g.release_host()
    ref = GOLD[name]["per_scan"]
    n = len(frames)
    for b0 in range(0, n, batch):
        sts = integrate_frames(g, bank, [ScanFrame(points=p, pose=pose) for p, pose in frames[b0:b0 + batch]],
                               IntegrationParams())
        for j, st in enumerate(sts):
            assert [st.points_in, st.points_discarded] == ref[b0 + j]["stats"][:2]
        last = min(b0 + batch, n) - 1
        if t.config <= 2 or last == n - 1 or (last + 1) % 32 == 0:
            assert_grid(g, t, last, f"integrate_frames, {batch} scans per launch")


@pytest.mark.parametrize("name", ["cfg2_traj100", "cfg4_window_traj30"])
def test_trajectory_queued_device_launches(name):
    """bench.py's path: device-resident scans, launches queued back to back
    on one stream with no host synchronisation between scans (scratch reuse
    across in-flight launches, PDL, the concurrent shadow stream)."""
    import torch

    t = TRAJ[name]
    frames = scans_of(t)
    g, bank = fresh(t)
    g.release_host()
    L = _native.lib()
    dev = [torch.from_numpy(p).cuda() for p, _ in frames]
    stream = torch.cuda.Stream()
    prm = IntegrationParams().native()
    n = len(frames)
    stops = sorted({n // 2 - 1, n - 1})
    done = 0
    for stop in stops:
        for i in range(done, stop + 1):
            cnt = np.array([frames[i][0].shape[0]], np.int64)
            pose = np.ascontiguousarray(frames[i][1].reshape(-1))
            _native.check(L.dbt_integrate_device(g.handle, bank.device_handle(g.device),
                                                 ctypes.c_void_p(dev[i].data_ptr()), _native.DBT_F32,
                                                 cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1,
                                                 ctypes.c_void_p(pose.ctypes.data), ctypes.byref(prm),
                                                 ctypes.c_void_p(stream.cuda_stream)))
        stream.synchronize()
        assert_grid(g, t, stop, "queued dbt_integrate_device launches")
        done = stop + 1


def test_cfg2_trajectory_exact_frame_stats():
    """Every FrameStats field of the 100 config-2 scans equals the
    reference's, with the serial voxels_written (exact_voxels_written)."""
    t = TRAJ["cfg2_traj100"]
    frames = scans_of(t)
    g, bank = fresh(t)
    g.release_host()
    ref = GOLD[t.name]["per_scan"]
    prm = IntegrationParams(exact_voxels_written=True)
    for i, (p, pose) in enumerate(frames):
        st = integrate_frame(g, bank, ScanFrame(points=p, pose=pose), prm)
        assert [st.points_in, st.points_discarded, st.voxels_written] == ref[i]["stats"], f"scan {ref[i]['scan']}"
    assert_grid(g, t, len(frames) - 1, "exact_voxels_written")
