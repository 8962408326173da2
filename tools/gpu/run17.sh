python -m pytest tests -x -q -m gpu -k "async or Async or live_reference or shim" > gpurun_out/s5_async_tests.log 2>&1; echo tests rc=$?; tail -n 3 gpurun_out/s5_async_tests.log
python bench.py --no-cpu-baseline > gpurun_out/s5_bench_c4.log 2>&1; echo rc=$?
python bench.py --no-cpu-baseline --config 2 > gpurun_out/s5_bench_c2.log 2>&1; echo rc=$?
python bench.py --no-cpu-baseline --config 3 > gpurun_out/s5_bench_c3.log 2>&1; echo rc=$?
for c in 4 2 3; do tail -n 1 gpurun_out/s5_bench_c$c.log | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print(d['config']['workload'][:10], 'value %.1f step %.1f us'%(d['value']/1e6, d['ms_per_step']*1e3), ' '.join('%s %.1f'%(k, d[k]['value']/1e6) for k in ('e2e','e2e_sync','e2e_pageable','e2e_pageable_async') if k in d))
"; done
