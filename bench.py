"""Benchmark: LiDAR points integrated per second (BASELINE.json metric).

Default workload: BASELINE config 4, the largest configuration that fits one
B200 — the config-3 street scene and 128x2048-beam sensor at 0.02 m voxels on
the full 4000x4000x400 grid (6.4e9 voxels, 58 GB of device state), K=21
kernel, 40x40 bins, shadow radius 2. `--config N` selects another BASELINE
config (1: room scan, 2: room trajectory, 3: street 2000x2000x100 @ 0.1 m,
5: config-3 scans, `--batch S` per launch).

Fixed scan window (independent of --steps / --warmup): the grid first holds
the trajectory's scans 0-9 (prefill, untimed); a step integrates the next
scan (the next S scans for --batch S, one launch) of the window, scans 10-29
(batches: max(2, 128 // S) batches from scan 10). After the last window
batch the grid is reset and refilled (untimed, between the step events), so
every pass over the window times the same grid states. Warm-up steps run the
same window, then the grid is reset and refilled before the timed region.
Config 1 has one scan: every step integrates it into a fresh grid. L2 is
flushed before every step (the config-4 grid is 58 GB anyway): a 256 MB
write, then a 256 MB read of a second buffer, so the flush's own dirty lines
are written back before the step events rather than by the step's kernels
(`--flush write` keeps the write-only flush).

  value : applied returns / device seconds, scans resident in HBM, CUDA
          events on the launch stream around each step (launch sequence incl.
          the concurrent shadow stream), max over ranks.
  e2e   : same metric through the public API with PINNED host float32
          scans: validation, the scan's host->device transfer, launches, the
          FrameStats read-back, host wall clock. Single scans per step
          (N = 1): integrate_frame_async calls pipelined two deep (the next
          scan's copy and host work overlap the current kernels), every
          FrameStats collected inside the timed region; `e2e_sync` is one
          synchronous integrate_frame per step (L2 flushed before each).
          Batches / N > 1: the synchronous calls. `e2e_pageable` repeats the
          synchronous pass with the plain numpy scans a stock caller passes,
          `e2e_pageable_async` the pipelined pass with them.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--config 4] [--batch 1] [--multi slab|replica]
--gpus N > 1 without torchrun re-launches itself under torch.distributed.run
(one process per GPU). N > 1 default: interleaved x-slabs, every rank stamps
only the part of each return's cube inside its planes; rank 0 holds the scans
and broadcasts each step's points over NCCL inside the timed region.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import socket
import subprocess
import sys
import threading
import time
from concurrent.futures import ProcessPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import workloads  # noqa: E402

METRIC = "LiDAR points integrated/sec (device-timed)"
UNIT = "points/s"
K_EDGE = 21
PREFILL = 10   # trajectory scans in the grid before the window
WINDOW = 20    # window scans (single-scan steps)
CPU_SCANS_PER_STEP = 4  # --impl reference: scans of a step's batch the CPU sample integrates


def b_alg(shadow_cells: float) -> float:
    """algorithmic bytes per applied return = 4*K^3 + 4*|S|
    (mask read for every cube cell + hits/sign read-write on shadow cells),
    defined on the reference's 4-byte mask layout."""
    return 4.0 * K_EDGE ** 3 + 4.0 * shadow_cells


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or platform.machine()


def plan(w, batch: int):
    """(prefill scan ids, window batches as lists of scan ids)."""
    if w.n_scans == 1:
        return [], [[0]]
    if batch == 1:
        return list(range(PREFILL)), [[PREFILL + j] for j in range(WINDOW)]
    nb = max(2, 128 // batch)
    return list(range(PREFILL)), [list(range(PREFILL + j * batch, PREFILL + (j + 1) * batch)) for j in range(nb)]


def window_desc(w, batch):
    pre, win = plan(w, batch)
    if not pre:
        return "scan 0 into a fresh grid every step"
    return (f"grid holds scans 0-{pre[-1]} (prefill, untimed); step j integrates window batch j mod {len(win)} "
            f"(scans {win[0][0]}-{win[-1][-1]}, {batch} scan(s) per launch); reset + prefill after every pass "
            f"(untimed) — independent of --steps/--warmup")


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 100 ms (nvidia-smi's
    own loop mode) during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None
        self._t = None

    def _reader(self):
        for line in self.proc.stdout:
            parts = [v.strip() for v in line.strip().split(",")]
            if len(parts) == 6:
                self.rows.append(parts)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._reader, daemon=True)
            self._t.start()
            time.sleep(0.3)  # first samples before the timed region starts
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
            self._t.join(timeout=5)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}

        def num(v):
            try:
                return float(v)
            except ValueError:
                return None

        sm = [x for x in (num(r[0]) for r in self.rows) if x is not None]
        mx = [x for x in (num(r[1]) for r in self.rows) if x is not None]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4) if r[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def _scan_job(args):
    config, k = args
    return workloads.get(config).scan(k)


def gen_scans(w, ids):
    """{scan id: float32 points} (ray casting in a process pool for the street
    scenes, ~2.6 s per config-3 scan)."""
    ids = sorted(set(ids))
    if w.config <= 2 or len(ids) <= 2:
        return {k: w.scan(k) for k in ids}
    with ProcessPoolExecutor(max_workers=min(len(ids), os.cpu_count() or 1)) as ex:
        return dict(zip(ids, ex.map(_scan_job, [(w.config, k) for k in ids])))


def diag_reorder(pts, pose, w, how):
    """Diagnostics: the scan's points permuted by their map-frame voxel
    (Morton / lexicographic) or at random. The grid result does not depend
    on the order; the sweep's memory locality does."""
    if how == "random":
        return pts[np.random.default_rng(0).permutation(len(pts))]
    if how.startswith("az"):
        # sensor-frame azimuth sectors, scan order kept inside a sector: the
        # beams that stamp overlapping cubes come close together in the list
        n = int(how[2:])
        sec = np.floor((np.arctan2(pts[:, 1].astype(np.float64), pts[:, 0]) / (2 * np.pi) + 0.5) * n).astype(np.int64) % n
        return np.ascontiguousarray(pts[np.argsort(sec, kind="stable")])
    m = pts.astype(np.float64) @ pose[:3, :3].T + pose[:3, 3]
    v = np.clip(np.floor((m - np.asarray(w.origin)) / w.voxel_size), 0, (1 << 20) - 1).astype(np.uint64)
    if how == "xyz":
        key = (v[:, 0] << np.uint64(42)) | (v[:, 1] << np.uint64(21)) | v[:, 2]
    else:
        key = np.zeros(len(v), np.uint64)
        for b in range(21):
            for a in range(3):
                key |= ((v[:, a] >> np.uint64(b)) & np.uint64(1)) << np.uint64(3 * b + (2 - a))
    return np.ascontiguousarray(pts[np.argsort(key, kind="stable")])


def cpu_grid_for(w):
    """Grid the CPU samples run on. Config 4's 6.4e9-voxel grid needs 38 GB
    of reference host arrays; per-scan CPU cost does not depend on grid size
    (BASELINE.md §2), so its sample uses the config-4 window
    of tests/cases.py (1000x1000x400 at the same origin offset)."""
    if w.config == 4:
        return (1000, 1000, 400), (0.0, 90.0, -0.22), "config-4 scene on its 1000x1000x400 window grid"
    return w.dims, w.origin, "same grid"


def cpu_baseline(w, batch, scans, budget_s=12.0, threads=None):
    """Oracle port (C preprocessing + C serial-order stamping, x-slab threads
    over all host cores) on the prefill + window scans in trajectory order
    until the time budget is spent. Returns applied returns / s."""
    import oracle

    threads = threads or oracle.os_threads()
    ob = oracle.OracleBank.build(size=K_EDGE, shadow_radius=w.shadow_radius)
    dims, origin, note = cpu_grid_for(w)
    g = oracle.OracleGrid(dims, w.voxel_size, origin)
    pre, win = plan(w, batch)
    order = pre + [k for b in win for k in b]
    applied = 0
    t0 = time.perf_counter()
    n = 0
    for k in order:
        st = oracle.integrate_frame(g, ob, scans[k], w.poses[k], threads=threads, c_prep=True)
        applied += st.points_in - st.points_discarded
        n += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return {"value": applied / el, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
            "sample": f"config-{w.config} scans {order[0]}..{order[n - 1]} ({n} scans, {applied} applied returns) "
                      f"in {el:.1f} s, {note}, oracle C port of the reference integrate_frame (libm "
                      f"transcendentals), {threads} threads (x-slab stamping) on {cpu_model()}"}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port of the Python reference, which cannot travel to the GPU box)
    on the same window, all host threads, one window batch per step."""
    if rank != 0:
        return
    import oracle

    w = workloads.get(args.config)
    B = max(1, args.batch)
    pre, win = plan(w, B)
    scans = gen_scans(w, pre + [k for b in win for k in b])
    threads = oracle.os_threads()
    ob = oracle.OracleBank.build(size=K_EDGE, shadow_radius=w.shadow_radius)
    dims, origin, note = cpu_grid_for(w)

    def fresh():
        g = oracle.OracleGrid(dims, w.voxel_size, origin)
        for k in pre:
            oracle.integrate_frame(g, ob, scans[k], w.poses[k], threads=threads, c_prep=True)
        return g

    g = fresh()
    applied, el = 0, 0.0
    for s in range(args.warmup + args.steps):
        if s == args.warmup or (s and s % len(win) == 0):
            g = fresh()
        j = (s - args.warmup) % len(win) if s >= args.warmup else s % len(win)
        t0 = time.perf_counter()
        a = 0
        # bounded sample: at most CPU_SCANS_PER_STEP scans of the step's batch
        for k in win[j][:CPU_SCANS_PER_STEP]:
            st = oracle.integrate_frame(g, ob, scans[k], w.poses[k], threads=threads, c_prep=True)
            a += st.points_in - st.points_discarded
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            applied += a
            el += dt
    value = applied / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
        "config": config_desc(w, B, l2=L2_CLEAN),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
                         "sample": f"{args.steps} timed window steps of config {args.config} (at most "
                                   f"{CPU_SCANS_PER_STEP} scans of each step's batch; {note}), oracle C port of the "
                                   f"reference integrate_frame, {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


L2_CLEAN = ("flushed before every step: 256 MB write, then a 256 MB read of another buffer (write-back of the "
            "flush's dirty lines outside the step)")


class L2Flush:
    """Evict L2 before a timed step: write a 256 MB buffer (> the 126 MB L2);
    mode "clean" then reads a second 256 MB buffer, so the dirty lines the
    write left are written back here, not by the next step's kernels."""

    def __init__(self, dev, mode):
        import torch
        self.mode = mode
        self.w = torch.empty(64 << 20, dtype=torch.float32, device=dev)
        self.r = torch.zeros(64 << 20, dtype=torch.float32, device=dev) if mode == "clean" else None

    def __call__(self):
        self.w.zero_()
        if self.r is not None:
            self.r.max()

    def desc(self):
        return L2_CLEAN if self.mode == "clean" else "flushed before every step (256 MB write)"


def config_desc(w, batch, interleave=0, multi="single", l2="flushed before every step (256 MB write)"):
    scene = "synthetic room" if w.config <= 2 else "synthetic street (ground, 40 buildings, 200 poles)"
    par = {"single": "single GPU",
           "replica": "data-parallel whole-grid replicas: each rank integrates a contiguous segment of the window, "
                      "one exact merge at the end of every pass (MIN/MIN/SUM all-reduces over the 16^3 bricks any rank touched), timed",
           "slab": f"x-interleaved slabs ({interleave}-plane blocks dealt round-robin over the ranks): every rank "
                   "stamps only the part of each return's cube inside its planes; points broadcast from rank 0 "
                   "over NCCL every step"}[multi]
    return {"workload": f"config {w.config}: {scene}, {w.beams}x{w.n_az} float32 returns/scan, {w.voxel_size} m "
                        f"voxels, grid {w.dims[0]}x{w.dims[1]}x{w.dims[2]}"
                        + (" (literal room grid padded by 11)" if w.config <= 2 else ""),
            "kernel": f"{K_EDGE}^3", "bins": "40x40", "shadow_radius": w.shadow_radius, "t_occ": 2, "h_max": 255,
            "scans_per_step": batch, "window": window_desc(w, batch),
            "l2": l2, "parallelism": par}


def relaunch(n: int) -> int:
    """--gpus N > 1 outside torchrun: one process per GPU under
    torch.distributed.run (127.0.0.1 rendezvous)."""
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def kernel_traffic(config: int, batch: int):
    """ncu per-launch DRAM/LTS figures of this workload's kernels
    (profiles/kernel_traffic.json, written by tools/ncu_traffic.py from a
    capture of this bench command on the current build)."""
    p = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p)).get("configs", {}).get(f"{config}x{batch}")
    return d


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--batch", type=int, default=1, help="scans per launch (config 5: 1/8/32/128)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true", help="diagnostics only: skip the end-to-end passes")
    ap.add_argument("--no-flush", action="store_true", help="diagnostics only: keep L2 warm between steps")
    ap.add_argument("--flush", default="clean", choices=["clean", "write"],
                    help="L2 flush before a step: write a 256 MB buffer, then (clean) read another 256 MB buffer so "
                         "the flush's dirty lines are written back before the step instead of inside it")
    ap.add_argument("--diag-order", default=None, choices=["morton", "xyz", "random", "az8", "az16", "az32", "az64", "az128", "az256"],
                    help="diagnostics only: reorder each scan's points (spatial locality of the sweep work list)")
    ap.add_argument("--interleave", type=int, default=None,
                    help="slab mode: x-block width of interleaved sharding (default 64, at most nx / 2N)")
    ap.add_argument("--multi", default="slab", choices=["replica", "slab"],
                    help="N > 1: x-interleaved slabs with a per-step point broadcast (default), or data-parallel "
                         "whole-grid replicas with one exact merge per window pass")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(relaunch(args.gpus))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    args.warmup = max(args.warmup, 3)

    import torch

    from paper_2509_20081_b200 import _native
    from paper_2509_20081_b200 import IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame, integrate_frames
    from paper_2509_20081_b200.grid import VoxelGrid
    from paper_2509_20081_b200.sharded import ReplicatedGrid, ShardedGrid

    backend = os.environ.get("BENCH_BACKEND", "nccl")
    if backend == "gloo":
        # functional checks of the N > 1 host logic on a box with fewer GPUs
        # than ranks (host-staged collectives; not a timing configuration)
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "gloo":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    w = workloads.get(args.config)
    B = max(1, args.batch)
    pre, win = plan(w, B)
    multi = args.multi if world > 1 else "single"
    replica = multi == "replica"
    holds_scans = rank == 0 or replica
    scans = gen_scans(w, pre + [k for b in win for k in b]) if holds_scans else {}
    if args.diag_order:
        scans = {k: diag_reorder(v, w.poses[k], w, args.diag_order) for k, v in scans.items()}
    bank = build_kernel_bank(size=K_EDGE, shadow_radius=w.shadow_radius)
    shadow_cells = float(np.mean([len(o) for o in bank.shadow_offsets]))
    params = IntegrationParams()
    L = _native.lib()
    dev = f"cuda:{local}"

    # ---------------- device-resident value --------------------------------
    if replica:
        ilv = 0
        sg = ReplicatedGrid(w.dims, w.voxel_size, w.origin, dist, device=local)
    else:
        # 64-plane blocks, narrower when the grid has too few for every rank
        ilv = args.interleave if args.interleave is not None else (
            min(64, max(1, w.dims[0] // (2 * world))) if world > 1 else 0)
        sg = ShardedGrid(w.dims, w.voxel_size, w.origin, rank, world, device=local, interleave=ilv or None)
    g_local = sg.local

    def to_dev(ids):
        poses = np.stack([w.poses[k] for k in ids])
        if holds_scans:
            counts = [len(scans[k]) for k in ids]
            pts = torch.from_numpy(np.concatenate([scans[k] for k in ids])).to(dev)
        else:
            counts, pts = [0] * len(ids), None
        if dist is not None and not replica:
            # every rank needs the counts to size the broadcast buffers
            c = torch.tensor(counts, dtype=torch.int64, device=dev)
            dist.broadcast(c, 0)
            counts = c.cpu().tolist()
        return pts, counts, poses

    pre_dev = [to_dev([k]) for k in pre]
    win_dev = [to_dev(b) for b in win]
    nw = len(win)
    # replicas: every pass over the window is split into W contiguous segments
    # (slab parts all integrate every batch: one segment, the whole window)
    W = world if replica else 1
    r_seg = rank if replica else 0
    seg = (r_seg * nw // W, (r_seg + 1) * nw // W)
    P = -(-nw // W)  # steps per pass (longest segment)

    def batch_of(s):
        """Window batch this rank integrates at step s of a pass, or None."""
        i = s % P
        return seg[0] + i if seg[0] + i < seg[1] else None

    flush = L2Flush(dev, args.flush)
    stream = torch.cuda.Stream(device=local)  # every timed op (flush, broadcast, engine) on this stream
    torch.cuda.set_stream(stream)

    def launch(item):
        pts, counts, poses = item
        if not replica:
            if rank != 0:
                pts = torch.empty((sum(counts), 3), dtype=torch.float32, device=dev)
            if dist is not None:
                dist.broadcast(pts, 0)
        sg.integrate_device(bank, pts, counts, poses, params, stream=stream)

    profiling = [False]

    def refill():
        """reset + prefill (untimed, queued on the stream; its launches are
        kept out of the per-kernel profile)."""
        if profiling[0]:
            L.dbt_profile_enable(g_local.handle, 0)
        L.dbt_grid_reset(g_local.handle)
        for item in pre_dev:
            launch(item)
        if replica:
            stream.synchronize()
            sg.mark()
        if profiling[0]:
            L.dbt_profile_enable(g_local.handle, 1)

    # applied returns of every window batch in its pass position (discards
    # do not depend on the grid state), so the timed pass needs no read-back
    applied_of = {}
    refill()
    for j in range(seg[0], seg[1]):
        launch(win_dev[j])
        applied_of[j] = sum(x.points_in - x.points_discarded for x in sg.stats())

    def run_pass(timed):
        """warmup + steps; timed: no host sync or profiling inside the region
        (launches queue ahead), else per-step stats and per-kernel events."""
        profiling[0] = not timed
        L.dbt_profile_enable(g_local.handle, 0 if timed else 1)
        refill()
        for s in range(args.warmup):
            if s and s % P == 0:
                if replica:
                    sg.merge(stream=stream)
                refill()
            if batch_of(s) is not None:
                launch(win_dev[batch_of(s)])
        if replica:
            sg.merge(stream=stream)
        torch.cuda.synchronize()
        refill()
        torch.cuda.synchronize()
        L.dbt_profile_reset(g_local.handle)
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        cnt = {"applied": 0, "swept": 0, "written": 0, "skipped": 0, "rows": 0}
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()
        launches0 = L.dbt_launch_count()
        merges = []

        def timed_merge():
            # the replicas' partial maps become the pass's global map: one
            # exact merge (three all-reduces over the packed grid), timed
            em = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            em[0].record(stream)
            sg.merge(stream=stream)
            em[1].record(stream)
            merges.append(em)

        for i in range(args.steps):
            if i and i % P == 0:
                if replica:
                    timed_merge()
                refill()  # untimed: between the step events
            if not args.no_flush:
                flush()
            j = batch_of(i)
            ev[i][0].record(stream)
            if j is not None:
                launch(win_dev[j])
            ev[i][1].record(stream)
            if j is not None:
                cnt["applied"] += applied_of[j]
                if not timed:
                    sts = sg.stats()
                    cnt["swept"] += sts[0].unique_centers
                    cnt["written"] += sts[0].voxels_written
                    cnt["skipped"] += sts[0].centers_skipped
                    cnt["rows"] += sts[0].rows_swept
        if replica:
            timed_merge()  # the last (possibly partial) pass
        torch.cuda.synchronize()
        launches = L.dbt_launch_count() - launches0
        merge_ms = sum(a.elapsed_time(b) for a, b in merges)
        dev_ms = sum(a.elapsed_time(b) for a, b in ev) + merge_ms
        cnt["merge_ms"] = merge_ms
        cnt["merges"] = len(merges)
        return dev_ms, launches, cnt

    with ClockSampler(local) as clk:
        dev_ms, launches, cnt = run_pass(timed=True)
    applied = cnt["applied"]
    local_applied = applied
    if dist is not None:
        t = torch.tensor([dev_ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dev_ms = float(t.item())
        if replica:  # every rank integrated its own scans
            a = torch.tensor([applied], dtype=torch.int64, device=dev)
            dist.all_reduce(a)
            applied = int(a.item())
        dist.barrier()
    value = applied / (dev_ms / 1e3)

    # per-kernel device time: a second, identical pass with CUDA events around
    # every kernel on its own stream (not inside the timed region above)
    prof_ms, _, pc = run_pass(timed=False)
    swept, written, skipped, rows = pc["swept"], pc["written"], pc["skipped"], pc["rows"]
    names = ctypes.create_string_buffer(32 * 16)
    ms = (ctypes.c_double * 16)()
    cnt_ = (ctypes.c_int64 * 16)()
    nk = ctypes.c_int32()
    L.dbt_profile_read(g_local.handle, names, ms, cnt_, 16, ctypes.byref(nk))
    kernels = {}
    for i in range(nk.value):
        nm = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
        kernels[nm] = {"ms_total": ms[i], "launches": int(cnt_[i]), "avg_us": ms[i] / max(cnt_[i], 1) * 1e3}
    L.dbt_profile_enable(g_local.handle, 0)

    # ---------------- roofline of the dominant kernel ------------------------
    # Dominant = the critical-path kernel with the most event time per step
    # (sweep on the main stream; the shadow kernel runs beside it).
    dom = "sweep_kernel"
    kd = kernels.get(dom, {"avg_us": float("nan"), "launches": 0})
    peak, peak_src = measured_peaks()
    steps_with_work = max(1, sum(1 for i in range(args.steps) if batch_of(i) is not None))
    applied_per_launch = local_applied / steps_with_work
    tr = kernel_traffic(args.config, B) if world == 1 else None
    dram = (tr or {}).get("kernels", {}).get(dom, {}).get("dram_bytes")
    # bytes the sweep touches (live device counters): two 32-byte sectors of
    # the 16-bit length cache per kernel row it read after culling (a row's
    # 1-4 16-byte chunks span 1-2 sectors); the MIN reductions of lowered
    # chunks hit the same sectors
    touched = (rows * 64 if rows else swept * K_EDGE ** 3 * 2) / steps_with_work
    alg = b_alg(shadow_cells) * applied_per_launch / (1 if replica else max(world, 1))
    if dram is not None:
        achieved, basis = dram / (kd["avg_us"] * 1e-6) / 1e9, (
            "ncu dram__bytes_read.sum + dram__bytes_write.sum per launch of this kernel on this workload "
            f"({tr.get('source', '?')}) / its live CUDA-event launch time")
    else:
        achieved, basis = touched / (kernels.get("sweep_kernel", kd)["avg_us"] * 1e-6) / 1e9, (
            "no ncu capture of this workload in profiles/kernel_traffic.json: bytes the sweep touches (live device "
            "counters) / its live CUDA-event launch time")
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if replica else ("strong" if world > 1 else "weak"), "vs_baseline": None,
        "dtype": "u32/f64", "data": "synthetic (seeded ray-cast scenes with the BASELINE configs' shapes)",
        "config": config_desc(w, B, ilv, multi, l2="not flushed (diagnostic)" if args.no_flush else flush.desc()),
        "gpu_launches": int(launches),
        "kernels": kernels,
        "profiled_step_ms": prof_ms / args.steps,
        "timing": "timed pass: launches queue ahead (no per-step host sync, no per-kernel events); applied "
                  "returns per window batch from an untimed counting pass; kernel times from a second identical "
                  "pass with per-kernel CUDA events",
        "clocks": clk.summary(),
        **({"merge_ms": cnt["merge_ms"], "merges": cnt["merges"]} if replica else {}),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": dram, "peak_source": peak_src, "basis": basis,
                     "kernel_avg_us": kd["avg_us"],
                     "touched_bytes_per_launch": touched,
                     "touched_gbs": touched / (kernels.get("sweep_kernel", kd)["avg_us"] * 1e-6) / 1e9,
                     "rows_swept_per_launch": rows / steps_with_work,
                     "centres_swept_per_launch": swept / steps_with_work,
                     "returns_skipped_per_launch": skipped / steps_with_work,
                     "ncu_per_launch": (tr or {}).get("kernels")},
        "alg_savings": {"b_alg_bytes_per_return": b_alg(shadow_cells),
                        "b_alg_bytes_per_launch": alg,
                        "b_alg_gbs_over_sweep": alg / (kernels.get("sweep_kernel", kd)["avg_us"] * 1e-6) / 1e9,
                        "def": "SURVEY.md 8(d) 4*21^3 + 4*|S| B per applied return (the reference's per-return "
                               "traffic) x applied returns / sweep time; above the HBM peak by design: the engine "
                               "sweeps each centre once, skips centres whose stamp is applied (certificates), culls "
                               "voxels a closer certified centre covers and lowers a 16-bit length cache instead of the 4-byte masks"},
    }

    # ---------------- e2e through the public API ----------------------------
    if not args.no_e2e:
        line.update(run_e2e(args, w, B, pre, win, scans, sg, bank, params, dist, rank, world, replica, dev, flush,
                            batch_of, P, seg, torch, _native, L, integrate_frame, integrate_frames, ScanFrame))
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w, B, scans)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


def run_e2e(args, w, B, pre, win, scans, sg, bank, params, dist, rank, world, replica, dev, flush, batch_of, P,
            seg, torch, _native, L, integrate_frame, integrate_frames, ScanFrame):
    """The same window through the public API with host scans (pinned, then
    pageable numpy), host wall clock per call, max over ranks."""
    out = {}
    g = sg.local
    pinned = {}
    if rank == 0 or replica:
        for k, s in scans.items():
            buf = ctypes.c_void_p()
            _native.check(L.dbt_host_alloc(s.nbytes, ctypes.byref(buf)))
            arr = np.ctypeslib.as_array((ctypes.c_float * s.size).from_address(buf.value)).reshape(s.shape)
            arr[...] = s
            pinned[k] = (buf, arr)

    def call(ids, src):
        """One public-API call for the scans ids; returns (applied, h2d bytes)."""
        if world > 1 and not replica:
            # slab mode: rank 0 copies the host scans, broadcasts, every rank
            # stamps its planes, stats read back (per-step collectives)
            if rank == 0:
                pts = torch.from_numpy(np.concatenate([src[k] for k in ids])).to(dev, non_blocking=True)
            else:
                pts = None
            counts = [len(scans[k]) for k in ids] if rank == 0 else None
            c = torch.tensor(counts if counts is not None else [0] * len(ids), dtype=torch.int64, device=dev)
            dist.broadcast(c, 0)
            counts = c.cpu().tolist()
            if rank != 0:
                pts = torch.empty((sum(counts), 3), dtype=torch.float32, device=dev)
            dist.broadcast(pts, 0)
            sg.integrate_device(bank, pts, counts, np.stack([w.poses[k] for k in ids]), params)
            sts = sg.stats()
            return sum(x.points_in - x.points_discarded for x in sts), (sum(counts) * 12 if rank == 0 else 0)
        if replica:
            sg._note_params(params)
        frames = [ScanFrame(points=src[k], pose=w.poses[k]) for k in ids]
        sts = [integrate_frame(g, bank, frames[0], params)] if len(ids) == 1 else integrate_frames(g, bank, frames,
                                                                                                  params)
        return sum(x.points_in - x.points_discarded for x in sts), sum(src[k].nbytes for k in ids)

    def refill(src):
        L.dbt_grid_reset(g.handle)
        for k in pre:
            call([k], src)
        if replica:
            sg.mark()

    def e2e_pass(src):
        el, pts_n, h2d = 0.0, 0, 0
        for s in range(args.warmup):
            if s % P == 0:
                if s and replica:
                    sg.merge()
                refill(src)
            if batch_of(s) is not None:
                call(win[batch_of(s)], src)
        if replica:
            sg.merge()
        if dist is not None:
            dist.barrier()
        for i in range(args.steps):
            if i % P == 0:
                if i and replica:
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    sg.merge()
                    torch.cuda.synchronize()
                    el += time.perf_counter() - t0
                refill(src)
            j = batch_of(i)
            if not args.no_flush:
                flush()
            torch.cuda.synchronize()
            if j is None:
                continue
            t0 = time.perf_counter()
            a, b = call(win[j], src)
            el += time.perf_counter() - t0
            pts_n += a
            h2d += b
        if replica:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            sg.merge()
            torch.cuda.synchronize()
            el += time.perf_counter() - t0
        if dist is not None:
            t = torch.tensor([el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            el = float(t.item())
            if replica:
                a = torch.tensor([pts_n, h2d], dtype=torch.int64, device=dev)
                dist.all_reduce(a)
                pts_n, h2d = int(a[0].item()), int(a[1].item())
        return pts_n / el, el, h2d

    def e2e_async_pass(src):
        """integrate_frame_async, calls pipelined (up to 2 outstanding: the
        next scan's host work and host->device copy overlap the previous
        scan's kernels); every call's FrameStats is collected inside the
        timed region. No L2 flush between the pipelined calls (it would sit
        on the critical path); refills between passes are untimed."""
        from paper_2509_20081_b200 import integrate_frame_async

        el, pts_n, h2d = 0.0, 0, 0
        for timed, n_steps in ((False, args.warmup), (True, args.steps)):
            pend = []
            t0 = None
            for i in range(n_steps):
                if i % P == 0:
                    for f in pend:
                        a = f.result()
                        pts_n += (a.points_in - a.points_discarded) if timed else 0
                    pend = []
                    if timed and t0 is not None:
                        el += time.perf_counter() - t0
                    torch.cuda.synchronize()
                    refill(src)
                    g.synchronize()
                    t0 = time.perf_counter()
                j = batch_of(i)
                if j is None:
                    continue
                k = win[j][0]
                pend.append(integrate_frame_async(g, bank, ScanFrame(points=src[k], pose=w.poses[k]), params))
                h2d += src[k].nbytes if timed else 0
                if len(pend) > 2:
                    a = pend.pop(0).result()
                    pts_n += (a.points_in - a.points_discarded) if timed else 0
            for f in pend:
                a = f.result()
                pts_n += (a.points_in - a.points_discarded) if timed else 0
            if timed and t0 is not None:
                el += time.perf_counter() - t0
        return pts_n / el, el, h2d

    api = ("paper_2509_20081_b200.integrate_frame (dbt_integrate_frame)" if B == 1 else
           "paper_2509_20081_b200.integrate_frames (dbt_integrate_scans)")
    if world > 1 and not replica:
        api = "rank 0: H2D copy of the host scans + NCCL broadcast; ShardedGrid.integrate_device + stats read, every rank"
    pin_src = {k: a for k, (_, a) in pinned.items()} if pinned else scans
    v, el, h2d = e2e_pass(pin_src)
    sync = {"value": v, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
            "d2h_bytes_per_step": 32 + 32 * B, "ms_per_step": el / args.steps * 1e3,
            "api": api + ", pinned float32 host scans, one synchronous call per step, L2 flushed before each"
            + (", every rank its own scans, then ReplicatedGrid.merge" if replica else "")}
    if B == 1 and world == 1:
        # headline: the pipelined public call (what a fuse loop issues)
        va, ela, h2da = e2e_async_pass(pin_src)
        out["e2e"] = {"value": va, "unit": UNIT, "h2d_bytes_per_step": h2da // args.steps,
                      "d2h_bytes_per_step": 64, "ms_per_step": ela / args.steps * 1e3,
                      "api": "paper_2509_20081_b200.integrate_frame_async (dbt_integrate_frame_async + "
                             "dbt_frame_wait), pinned float32 host scans, calls pipelined (<= 2 outstanding), every "
                             "call's FrameStats read inside the timed region, L2 not flushed between calls"}
        out["e2e_sync"] = sync
    else:
        out["e2e"] = sync
    v2, el2, _ = e2e_pass(scans if (rank == 0 or replica) else {})
    out["e2e_pageable"] = {"value": v2, "unit": UNIT, "ms_per_step": el2 / args.steps * 1e3,
                           "api": api + ", pageable numpy float32 scans (staged by one H2D copy per scan)"}
    if B == 1 and world == 1:
        # what a stock fuse loop holds: plain numpy scans, pipelined calls
        # (cudaMemcpyAsync from pageable memory stages through the driver and
        # blocks the host for the copy, while the previous scan's kernels run)
        v3, el3, _ = e2e_async_pass(scans)
        out["e2e_pageable_async"] = {"value": v3, "unit": UNIT, "ms_per_step": el3 / args.steps * 1e3,
                                     "api": "paper_2509_20081_b200.integrate_frame_async, pageable numpy float32 "
                                            "scans, calls pipelined (<= 2 outstanding)"}
    for buf, _ in pinned.values():
        L.dbt_host_free(buf)
    return out


if __name__ == "__main__":
    main()
