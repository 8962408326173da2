"""Per-config markdown table for DESIGN.md §5 from tools/bench_all.sh logs:
python tools/doc_table.py <tag>  (reads gpurun_out/<tag>_bench_cfg*_b*.log)."""
import glob
import json
import sys

T = sys.argv[1]
names = {("1", "1"): "1 (1 scan, fresh grid every step)", ("2", "1"): "2 (100-scan room, 0.05 m)",
         ("3", "1"): "3 (street, 0.1 m, 2000×2000×100)", ("4", "1"): "**4 (0.02 m, 6.4×10⁹ voxels)**",
         ("5", "8"): "5, 8 scans per launch", ("5", "32"): "5, 32 scans per launch", ("5", "128"): "5, 128 scans per launch"}
print("| config | device-resident | step | e2e pipelined | e2e sync | e2e pageable (sync / pipelined) | sweep roofline (DRAM) | CPU port (16 thr) |")
print("|---|---|---|---|---|---|---|---|")
for (c, b), name in names.items():
    f = f"gpurun_out/{T}_bench_cfg{c}_b{b}.log"
    d = json.loads(open(f).read().strip().splitlines()[-1])
    r = json.loads(open(f.replace("_bench_cfg", "_bench_ref_cfg")).read().strip().splitlines()[-1])
    M = lambda k: f"{d[k]['value'] / 1e6:,.0f}".replace(",", " ") if k in d else "—"
    pipe = M("e2e") if "e2e_sync" in d else "—"
    sync = M("e2e_sync") if "e2e_sync" in d else M("e2e")
    pg = M("e2e_pageable") + (" / " + M("e2e_pageable_async") if "e2e_pageable_async" in d else "")
    frac = f"{d['roofline']['frac']:.2f}" if (c, b) in (("4", "1"), ("2", "1")) else "—"
    n = lambda v: f"{v:,.0f}".replace(",", " ")
    print(f"| {name} | {n(d['value'] / 1e6)} | {n(d['ms_per_step'] * 1e3)} µs | {pipe} | {sync} | {pg} | {frac} | {r['value'] / 1e6:.2f} |")
