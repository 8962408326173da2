#!/bin/bash
# Per-config bench lines of the current build (GPU box, repo root):
#   bash tools/bench_all.sh <tag>   -> gpurun_out/<tag>_bench_cfg*.log
T=${1:-r2}
for spec in "1 1" "2 1" "3 1" "4 1" "5 8" "5 32" "5 128"; do
  set -- $spec
  python bench.py --config $1 --batch $2 > gpurun_out/${T}_bench_cfg$1_b$2.log 2>&1
  python bench.py --impl reference --config $1 --batch $2 > gpurun_out/${T}_bench_ref_cfg$1_b$2.log 2>&1
done
python - "$T" <<'PY'
import glob, json, sys
T = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{T}_bench_cfg*_b*.log")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        r = json.loads(open(f.replace("_bench_cfg", "_bench_ref_cfg")).read().strip().splitlines()[-1])
        es = d.get('e2e_sync', d['e2e'])
        print(f"{f:40s} value {d['value'] / 1e6:8.1f} M/s  step {d['ms_per_step'] * 1e3:7.1f} us  e2e {d['e2e']['value'] / 1e6:7.1f} "
              f"({d['e2e']['ms_per_step'] * 1e3:.1f} us)  sync {es['value'] / 1e6:7.1f}  pageable {d['e2e_pageable']['value'] / 1e6:7.1f}  frac {d['roofline']['frac']:.3f}  "
              f"sweep {d['kernels']['sweep_kernel']['avg_us']:.1f} us  ref {r['value'] / 1e6:.3f} M/s  clocks {d['clocks']['sm_mhz']}")
    except Exception as e:
        print(f, "failed", e)
PY
