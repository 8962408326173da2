"""Benchmark: LiDAR points integrated per second (BASELINE.json metric).

Default workload (configs[1] of BASELINE.json, the single-GPU config the
metric is quoted on): config 2 — 100-scan trajectory in the synthetic box
room, 64 beams x 1024 azimuths (65 536 float32 returns per scan), 0.05 m
voxels on the 400x400x100 room padded by 11 voxels (422x422x122; the literal
grid discards every wall return), K=21 kernel, 40x40 bins, shadow radius 1.
`--config N` selects another BASELINE config (3: street 2000x2000x100 @ 0.1 m,
4: 4000x4000x400 @ 0.02 m, 5: config-3 scans, `--batch S` per launch).

A step integrates the next scan (or the next S scans, one launch) of the
trajectory into the grid that holds all previous scans (the grid is reset
when the trajectory wraps, outside the timed region). L2 is flushed (256 MB
write) between timed steps.

  value : applied returns / device seconds, scans resident in HBM, CUDA
          events on the launch stream around each step (launch sequence incl.
          the concurrent shadow stream and the counter copy), summed over K
          steps, max over ranks.
  e2e   : same metric through the public API (integrate_frame /
          integrate_frames over PINNED host float32 scans): validation, H2D,
          launches, D2H of the FrameStats counters, host wall clock per call.

python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                [--config 2] [--batch 1]
Under torchrun (N>1) every rank owns an x-slab of the grid; rank 0 holds the
scans and broadcasts each step's points over NCCL inside the timed region.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
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


def b_alg(shadow_cells: float) -> float:
    """algorithmic bytes per applied return = 4*K^3 + 4*|S|
    (mask read for every cube cell + hits/sign read-write on shadow cells),
    defined on the reference's 4-byte mask layout."""
    return 4.0 * K_EDGE ** 3 + 4.0 * shadow_cells


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback (B200_PROFILING.md)"


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


def gen_scans(w, n):
    """Scans 0..n-1 of the trajectory (ray casting in a process pool for the
    street scenes, ~2.6 s per config-3 scan)."""
    if w.config <= 2 or n <= 2:
        return [w.scan(k) for k in range(n)]
    with ProcessPoolExecutor(max_workers=min(n, os.cpu_count() or 1)) as ex:
        return list(ex.map(_scan_job, [(w.config, k) for k in range(n)]))


def cpu_grid_for(w):
    """Grid the CPU samples run on. Config 4's 6.4e9-voxel grid needs 38 GB
    of reference host arrays; per-scan CPU cost does not depend on grid size
    (BASELINE.md §2), so its sample uses the config-4 window
    of tests/cases.py (1000x1000x400 at the same origin offset)."""
    if w.config == 4:
        return (1000, 1000, 400), (0.0, 90.0, -0.22), "config-4 scene on its 1000x1000x400 window grid"
    return w.dims, w.origin, "same grid"


def cpu_baseline(w, scans, budget_s=12.0, threads=None):
    """Oracle port (C preprocessing + C serial-order stamping, x-slab threads
    over all host cores) on the first scans of the same trajectory until the
    time budget is spent. Returns applied returns / s."""
    import oracle

    threads = threads or oracle.os_threads()
    ob = oracle.OracleBank.build(size=K_EDGE, shadow_radius=w.shadow_radius)
    dims, origin, note = cpu_grid_for(w)
    g = oracle.OracleGrid(dims, w.voxel_size, origin)
    applied = 0
    t0 = time.perf_counter()
    k = 0
    while k < len(scans):
        st = oracle.integrate_frame(g, ob, scans[k], w.poses[k], threads=threads, c_prep=True)
        applied += st.points_in - st.points_discarded
        k += 1
        if time.perf_counter() - t0 > budget_s:
            break
    el = time.perf_counter() - t0
    return {"value": applied / el, "unit": UNIT, "cores": threads, "kind": "port",
            "sample": f"config-{w.config} scans 0..{k - 1} ({k} scans, {applied} applied returns) in {el:.1f} s, "
                      f"{note}, oracle C port (libm transcendentals), {threads} threads (x-slab stamping)"}


def run_reference(args, rank, world):
    """--impl reference: the reference algorithm's CPU implementation (the
    oracle port of the Python reference, which cannot travel to the GPU box)
    on the same workload, all host threads, one scan per step."""
    if rank != 0:
        return
    import oracle

    w = workloads.get(args.config)
    n = args.warmup + args.steps
    scans = gen_scans(w, min(n, w.n_scans))
    threads = oracle.os_threads()
    ob = oracle.OracleBank.build(size=K_EDGE, shadow_radius=w.shadow_radius)
    dims, origin, note = cpu_grid_for(w)
    g = oracle.OracleGrid(dims, w.voxel_size, origin)
    applied, el = 0, 0.0
    for s in range(n):
        k = s % len(scans)
        if k == 0 and s > 0:
            g = oracle.OracleGrid(dims, w.voxel_size, origin)
        t0 = time.perf_counter()
        st = oracle.integrate_frame(g, ob, scans[k], w.poses[k], threads=threads, c_prep=True)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            applied += st.points_in - st.points_discarded
            el += dt
    value = applied / el
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
        "config": config_desc(w, 1),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{args.steps} timed scans of config {args.config} (full scans, {note}), oracle "
                                   f"C port of the reference integrate_frame, {threads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def config_desc(w, batch, interleave=0, replica=False):
    scene = "synthetic room" if w.config <= 2 else "synthetic street (ground, 40 buildings, 200 poles)"
    return {"workload": f"config {w.config}: {scene}, {w.n_scans}-scan trajectory, {w.beams}x{w.n_az} float32 "
                        f"returns/scan, {w.voxel_size} m voxels, grid {w.dims[0]}x{w.dims[1]}x{w.dims[2]}"
                        + (" (literal room grid padded by 11)" if w.config <= 2 else ""),
            "kernel": f"{K_EDGE}^3", "bins": "40x40", "shadow_radius": w.shadow_radius, "t_occ": 2, "h_max": 255,
            "scans_per_step": batch,
            "step": f"{batch} scan(s) integrated into the trajectory grid in one launch",
            "l2": "flushed between steps (256 MB write)",
            "parallelism": ("data-parallel whole-grid replicas: each rank integrates its own scans (consecutive "
                            "trajectory scans dealt round-robin), one exact merge (MIN/MIN/SUM all-reduces) at the "
                            "end of the timed region" if replica else
                            f"x-interleaved slabs ({interleave}-plane blocks dealt round-robin over the ranks)"
                            if interleave else
                            "x-slab sharding" if int(os.environ.get("WORLD_SIZE", "1")) > 1 else "single GPU")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--batch", type=int, default=1, help="scans per launch (config 5: 1/8/32/128)")
    ap.add_argument("--max-scans", type=int, default=None, help="distinct scans to generate (default: all needed)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-flush", action="store_true", help="diagnostics only: keep L2 warm between steps")
    ap.add_argument("--interleave", type=int, default=None,
                    help="slab mode: x-block width of interleaved sharding (default 64, at most nx / 2N)")
    ap.add_argument("--multi", default="replica", choices=["replica", "slab"],
                    help="N > 1: data-parallel whole-grid replicas with one exact merge at the end of the "
                         "timed region (default), or x-sharded slabs with a per-step point broadcast")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    args.warmup = max(args.warmup, 3)

    import torch

    from paper_2509_20081_b200 import _native
    from paper_2509_20081_b200 import (IntegrationParams, ScanFrame, build_kernel_bank, integrate_frame,
                                       integrate_frames, new_grid)
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
    need = (args.warmup + args.steps) * B
    n_avail = min(w.n_scans, need if args.max_scans is None else min(need, args.max_scans))
    n_avail = max(B, n_avail - n_avail % B)  # whole batches; the trajectory wraps with a grid reset
    scans = gen_scans(w, n_avail)
    steps_per_pass = n_avail // B
    bank = build_kernel_bank(size=K_EDGE, shadow_radius=w.shadow_radius)
    shadow_cells = float(np.mean([len(o) for o in bank.shadow_offsets]))
    params = IntegrationParams()
    L = _native.lib()
    dev = f"cuda:{local}"

    # ---------------- device-resident value --------------------------------
    multi = args.multi if world > 1 else "single"
    replica = multi == "replica"
    W = world if replica else 1  # step-batches consumed per step (all ranks)
    if replica:
        ilv = 0
        sg = ReplicatedGrid(w.dims, w.voxel_size, w.origin, dist, device=local)
    else:
        # 64-plane blocks, narrower when the grid has too few for every rank
        ilv = args.interleave if args.interleave is not None else (
            min(64, max(1, w.dims[0] // (2 * world))) if world > 1 else 0)
        sg = ShardedGrid(w.dims, w.voxel_size, w.origin, rank, world, device=local, interleave=ilv or None)
    # one device buffer per step-batch (concatenated scans), built before timing
    batches = []
    for j in range(steps_per_pass):
        idx = list(range(j * B, (j + 1) * B))
        counts = [len(scans[k]) for k in idx]
        poses = np.stack([w.poses[k] for k in idx])
        pts = torch.from_numpy(np.concatenate([scans[k] for k in idx])).to(dev) if (rank == 0 or replica) else None
        batches.append((pts, counts, poses))

    # Replicas: every pass over the trajectory is split into W contiguous
    # segments, one per rank (each scan integrated once per pass, and a
    # rank's consecutive scans overlap like the single-GPU sequence); a pass
    # ends with the merge (the pass's global map), then a reset.
    seg = (rank * steps_per_pass // W, (rank + 1) * steps_per_pass // W)
    P = -(-steps_per_pass // W)  # steps per pass (longest segment)

    def batch_of(s):
        """Step-batch this rank integrates at step s, or None (short segment)."""
        i = s % P
        return seg[0] + i if seg[0] + i < seg[1] else None

    def new_pass(s):
        return s % P == 0

    def reset_grid():
        if replica:
            sg.reset()
        else:
            L.dbt_grid_reset(sg.local.handle)
    flush = torch.empty(64 << 20, dtype=torch.float32, device=dev)  # 256 MB > L2
    stream = torch.cuda.Stream(device=local)  # every timed op (flush, broadcast, engine) on this stream
    torch.cuda.set_stream(stream)

    def do_step(s, j=None):
        j = batch_of(s) if j is None else j
        if j is None:
            return
        pts, counts, poses = batches[j]
        if not replica:
            if rank != 0:
                pts = torch.empty((sum(counts), 3), dtype=torch.float32, device=dev)
            if dist is not None:
                dist.broadcast(pts, 0)
        sg.integrate_device(bank, pts, counts, poses, params, stream=stream)

    # applied returns of every distinct batch (discards do not depend on the
    # grid state), so the timed pass needs no per-step read-back
    applied_of = []
    for j in range(steps_per_pass):
        if j == 0:
            reset_grid()
        do_step(0, j)
        applied_of.append(sum(x.points_in - x.points_discarded for x in sg.stats()))

    def run_pass(timed):
        """warmup + steps from a reset grid; timed: no host sync or profiling
        inside the region (launches queue ahead), else per-step stats and
        per-kernel CUDA events."""
        L.dbt_profile_enable(sg.local.handle, 0 if timed else 1)
        reset_grid()
        for s in range(args.warmup):
            if s and new_pass(s):
                if replica:
                    sg.merge(stream=stream)
                reset_grid()
            do_step(s)
        torch.cuda.synchronize()
        L.dbt_profile_reset(sg.local.handle)
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
            s = args.warmup + i
            if new_pass(s):
                if replica and i > 0:
                    timed_merge()
                reset_grid()
            if not args.no_flush:
                flush.zero_()
            ev[i][0].record(stream)
            do_step(s)
            ev[i][1].record(stream)
            if batch_of(s) is not None:
                cnt["applied"] += applied_of[batch_of(s)]
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
    L.dbt_profile_read(sg.local.handle, names, ms, cnt_, 16, ctypes.byref(nk))
    kernels = {}
    for i in range(nk.value):
        nm = names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode()
        kernels[nm] = {"ms_total": ms[i], "launches": int(cnt_[i]), "avg_us": ms[i] / max(cnt_[i], 1) * 1e3}
    L.dbt_profile_enable(sg.local.handle, 0)

    sweep = kernels.get("sweep_kernel", {"avg_us": float("nan"), "launches": 0})
    peak, peak_src = measured_peaks()
    # per launch of THIS rank: its own scans (replicas) or its slab's share
    applied_per_launch = local_applied / max(args.steps, 1)
    alg_bytes = b_alg(shadow_cells) * applied_per_launch / (1 if replica else max(world, 1))
    achieved = alg_bytes / (sweep["avg_us"] * 1e-6) / 1e9
    # bytes the sweep actually touches (device counters): one 32-byte sector of
    # the 1-byte distance cache per kernel row it read after culling (a row's
    # 1-4 chunks span 1-2 sectors) + the 4-byte RED.AND and the cache byte of
    # every lowered voxel (the shadow kernel runs concurrently). Generic
    # (non-culling) sweep: the full K^3 cube of every swept centre.
    touched = ((rows * 32 if rows else swept * K_EDGE ** 3) + written * 5) / max(args.steps, 1)
    traffic, lts = None, None
    tpath = os.path.join(ROOT, "profiles", "kernel_traffic.json")
    if os.path.exists(tpath) and args.config == 2 and B == 1:
        tr = json.load(open(tpath)).get("kernels", {})
        sw = tr.get("sweep_kernel", {})
        if "dram_bytes" in sw:
            traffic = sw["dram_bytes"]
        lts = {k: v for k, v in tr.items()}
    # the roof of a launch whose mask footprint fits L2 is the
    # measured L2 atomic (4-byte RED.AND) throughput, HBM otherwise
    l2 = (ctypes.c_double * 3)()
    _native.check(L.dbt_probe_l2(local, 48 << 20, l2))
    mask_bytes = 4 * w.dims[0] * w.dims[1] * w.dims[2]
    l2_size = torch.cuda.get_device_properties(local).L2_cache_size
    survey_roof = ("l2_red", l2[1]) if mask_bytes <= l2_size else ("hbm", peak)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak" if replica else "strong", "vs_baseline": None, "dtype": "u32/f64", "data": "synthetic",
        "config": config_desc(w, B, ilv, replica=replica),
        "gpu_launches": int(launches),
        "kernels": kernels,
        "profiled_step_ms": prof_ms / args.steps,
        "timing": "timed pass: launches queue ahead (no per-step host sync, no per-kernel events); "
                  "applied returns per scan from an untimed counting pass; kernel times from a second "
                  "identical pass with per-kernel CUDA events",
        "clocks": clk.summary(),
        **({"merge_ms": cnt["merge_ms"], "merges": cnt["merges"]} if replica else {}),
        "roofline": {"bound": "hbm", "kernel": "sweep_kernel", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                     "alg_bytes_per_launch": alg_bytes,
                     "alg_bytes_def": f"4*21^3 + 4*|S| = {b_alg(shadow_cells):.0f} B per applied return "
                                      "(SURVEY.md 8(d)) x applied returns per launch",
                     "traffic_source": "ncu dram__bytes_read+write per sweep launch (config 2), "
                                       "profiles/kernel_traffic.json",
                     "touched_bytes_per_launch": touched,
                     "touched_gbs": touched / (sweep["avg_us"] * 1e-6) / 1e9,
                     "why_frac_above_1": "B_alg is the reference's per-return traffic; the engine sweeps each "
                                         "centre voxel once (dedup), skips centres whose stamp is already applied "
                                         "(certificates), skips the voxels a closer certified neighbour centre "
                                         "covers (culling) and reads a 1-byte cache: touched/traffic are the "
                                         "bytes actually moved",
                     "rows_swept_per_launch": rows / max(args.steps, 1),
                     "centres_swept_per_launch": swept / max(args.steps, 1),
                     "returns_skipped_per_launch": skipped / max(args.steps, 1),
                     "l2_probe": {"red_and_gops": l2[0], "red_and_gbs": l2[1], "ldcg_gbs": l2[2],
                                  "buffer_bytes": 48 << 20,
                                  "how": "dbt_probe_l2: coalesced 4-byte RED.AND / 8-byte ld.cg over an "
                                         "L2-resident 48 MB buffer, best of 4 (CUDA events)"},
                     "survey_roof": {"kind": survey_roof[0], "peak_gbs": survey_roof[1],
                                     "achieved_gbs": achieved, "frac": achieved / survey_roof[1],
                                     "why": f"SURVEY.md 8(d): reference mask array {mask_bytes / 1e6:.0f} MB "
                                            f"vs L2 {l2_size / 1e6:.0f} MB"},
                     "ncu_per_launch": lts},
    }

    # ---------------- e2e through the public API ----------------------------
    # N = 1: integrate_frame(s) on pinned host scans; replicas: every rank
    # the same on its own scans, then the merge (collective), max over ranks
    if world == 1 or replica:
        if replica:
            rg = ReplicatedGrid(w.dims, w.voxel_size, w.origin, dist, device=local)
            rg._note_params(params)
            g = rg.local
        else:
            g = new_grid(w.dims, w.voxel_size, w.origin, memory_cap=1 << 42, device=local)
        pinned = []
        for s in scans:
            buf = ctypes.c_void_p()
            _native.check(L.dbt_host_alloc(s.nbytes, ctypes.byref(buf)))
            arr = np.ctypeslib.as_array((ctypes.c_float * s.size).from_address(buf.value)).reshape(s.shape)
            arr[...] = s
            pinned.append((buf, arr))
        e_el, e_pts, h2d = 0.0, 0, 0
        if dist is not None:
            dist.barrier()
        for s in range(args.warmup + args.steps):
            if new_pass(s):
                if replica:
                    if s > args.warmup:  # the pass's global map, timed
                        torch.cuda.synchronize()
                        t0 = time.perf_counter()
                        rg.merge()
                        torch.cuda.synchronize()
                        e_el += time.perf_counter() - t0
                    rg.reset()
                else:
                    L.dbt_grid_reset(g.handle)
            j = batch_of(s)
            if j is None:
                continue
            ks = range(j * B, (j + 1) * B)
            if s >= args.warmup:
                flush.zero_()
                torch.cuda.synchronize()
            t0 = time.perf_counter()
            if B == 1:
                sts = [integrate_frame(g, bank, ScanFrame(points=pinned[j][1], pose=w.poses[j]), params)]
            else:
                sts = integrate_frames(g, bank, [ScanFrame(points=pinned[k][1], pose=w.poses[k]) for k in ks],
                                       params)
            dt = time.perf_counter() - t0
            if s >= args.warmup:
                e_el += dt
                e_pts += sum(x.points_in - x.points_discarded for x in sts)
                h2d += sum(pinned[k][1].nbytes for k in ks)
        if replica:
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            rg.merge()
            torch.cuda.synchronize()
            e_el += time.perf_counter() - t0
            t = torch.tensor([e_el], dtype=torch.float64, device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            a = torch.tensor([e_pts, h2d], dtype=torch.int64, device=dev)
            dist.all_reduce(a)
            e_el, e_pts, h2d = float(t.item()), int(a[0].item()), int(a[1].item())
        line["e2e"] = {"value": e_pts / e_el, "unit": UNIT, "h2d_bytes_per_step": h2d // args.steps,
                       "d2h_bytes_per_step": 32 + 32 * B, "ms_per_step": e_el / args.steps * 1e3,
                       "api": ("paper_2509_20081_b200.integrate_frame (dbt_integrate_frame)" if B == 1 else
                               "paper_2509_20081_b200.integrate_frames (dbt_integrate_batch)")
                              + ", pinned float32 scans"
                              + (", every rank its own scans, then ReplicatedGrid.merge" if replica else "")}
        for buf, _ in pinned:
            L.dbt_host_free(buf)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_baseline(w, scans)
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
