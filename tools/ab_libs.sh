#!/bin/bash
# Same-box A/B of engine builds: tools/ab_libs.sh ROUNDS lib1.so lib2.so ... [-- bench args]
# Runs bench.py alternately with each library (DBT_LIB) and prints value / e2e.
rounds=$1; shift
libs=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do libs+=("$1"); shift; done
[ "$1" == "--" ] && shift
for r in $(seq "$rounds"); do
  for lib in "${libs[@]}"; do
    out=$(DBT_LIB="$lib" timeout 300 python bench.py --no-cpu-baseline "$@" 2>/dev/null | tail -1)
    python - "$lib" "$out" <<'PY'
import json, sys
try:
    d = json.loads(sys.argv[2])
    e = d.get('e2e', {'value': float('nan'), 'ms_per_step': float('nan')})
    print(f"{sys.argv[1]:32s} value {d['value'] / 1e6:8.1f}  e2e {e['value'] / 1e6:7.1f}  step {d['ms_per_step'] * 1e3:6.1f} us "
          f"e2e step {e['ms_per_step'] * 1e3:6.1f} us  " + " ".join(f"{k} {v['avg_us']:.1f}" for k, v in d['kernels'].items()), flush=True)
except Exception as e:
    print(sys.argv[1], "failed", e, sys.argv[2][:200])
PY
  done
done
