"""What each rank of the slab mode does at N GPUs, on one GPU: the bench's
scans (prefill 0-9 untimed, window 10-29 timed) integrated into each
interleaved part (bench.py's block width dealt over N ranks), device
resident, L2 flushed per step. Prints the slowest part's per-scan time, the
single-GPU time and the criterion slowest <= 1.3 * (single / N + prep)
(VERDICT r1 item 4). The per-step NCCL point broadcast is not included.

usage: python tools/slab_parts.py [config=4] [N ...]"""
import ctypes
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import workloads  # noqa: E402
from paper_2509_20081_b200 import _native, build_kernel_bank  # noqa: E402
from paper_2509_20081_b200.grid import VoxelGrid  # noqa: E402

import os
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 4
Ns = [int(v) for v in sys.argv[2:]] or [1, 2, 4, 8]
WIDTH = int(os.environ.get("SLAB_WIDTH", "64"))  # bench.py's default block width
w = workloads.get(cfg)
L = _native.lib()
scans = [torch.from_numpy(w.scan(k)).cuda() for k in range(30)]
bank = build_kernel_bank(shadow_radius=w.shadow_radius)
prm = _native.make_params()
flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
L.dbt_profile_enable  # noqa


def run_part(g, timed_from=10):
    tot, prep = 0.0, 0.0
    acc = np.zeros(4)
    L.dbt_profile_enable(g.handle, 1)
    for k in range(len(scans)):
        if k == timed_from:
            torch.cuda.synchronize()
            L.dbt_profile_reset(g.handle)
        flush.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        cnt = np.array([scans[k].shape[0]], np.int64)
        pose = np.ascontiguousarray(w.poses[k].reshape(-1))
        a.record()
        _native.check(L.dbt_integrate_device(g.handle, bank.device_handle(0), ctypes.c_void_p(scans[k].data_ptr()),
                                             0, cnt.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), 1,
                                             ctypes.c_void_p(pose.ctypes.data), ctypes.byref(prm), ctypes.c_void_p(0)))
        b.record()
        torch.cuda.synchronize()
        if k >= timed_from:
            tot += a.elapsed_time(b)
            st = (_native.Stats * 1)()
            L.dbt_stats_read(g.handle, st, 1)
            acc += [st[0].unique_centers, st[0].rows_swept, st[0].voxels_written, st[0].centers_skipped]
    names = ctypes.create_string_buffer(32 * 16)
    ms = (ctypes.c_double * 16)()
    cn = (ctypes.c_int64 * 16)()
    nk = ctypes.c_int32()
    L.dbt_profile_read(g.handle, names, ms, cn, 16, ctypes.byref(nk))
    ks = {names.raw[32 * i:32 * i + 32].split(b"\0")[0].decode(): ms[i] / max(cn[i], 1) * 1e3 for i in range(nk.value)}
    L.dbt_profile_enable(g.handle, 0)
    n = len(scans) - timed_from
    ks["counters"] = (acc / n).round().astype(int).tolist()  # centres swept, rows, REDs, skipped per scan
    return tot / n * 1e3, ks


single = None
for N in Ns:
    worst, worst_k, parts = 0.0, None, []
    only = os.environ.get("SLAB_ONLY")  # "N:r": run only part r of N (profiling)
    for r in range(N):
        if only and (int(only.split(":")[0]) != N or int(only.split(":")[1]) != r):
            continue
        width = min(WIDTH, w.dims[0] // (2 * N))
        g = VoxelGrid(w.dims, w.voxel_size, w.origin, interleave=(width, N, r)) if N > 1 else \
            VoxelGrid(w.dims, w.voxel_size, w.origin)
        us, ks = run_part(g)
        parts.append((round(us, 1), ks["counters"]))
        if us > worst:
            worst, worst_k = us, ks
        del g
        torch.cuda.empty_cache()
    if N == 1:
        single = worst
    prep = worst_k.get("prep_kernel", 0.0)
    crit = 1.3 * (single / N + prep) if single else float("nan")
    print(f"config {cfg} N={N}: slowest part {worst:.1f} us/scan (prep {prep:.1f}, sweep "
          f"{worst_k.get('sweep_kernel', 0):.1f}, shadow {worst_k.get('shadow_kernel', 0):.1f}); single {single or float('nan'):.1f}; "
          f"criterion 1.3*(single/N + prep) = {crit:.1f} -> {'met' if worst <= crit else 'NOT met'}; width {WIDTH}, "
          f"parts {parts}", flush=True)
