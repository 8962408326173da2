python -m pytest tests/test_integration_shim.py -x -q -m gpu > gpurun_out/s5_shim_tests.log 2>&1; echo tests rc=$?; tail -n 3 gpurun_out/s5_shim_tests.log
for o in none az8 az16 az32 az64 az128 az256 none; do
  a=""; [ $o != none ] && a="--diag-order $o"
  python bench.py --no-cpu-baseline --no-e2e $a 2>/dev/null | tail -n 1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('$o', 'value %.1f step %.1f us sweep %.1f'%(d['value']/1e6, d['ms_per_step']*1e3, d['kernels']['sweep_kernel']['avg_us']))
"
done 2>&1 | tee gpurun_out/s5_azorder_c4.log
for o in none az16 az64; do
  a=""; [ $o != none ] && a="--diag-order $o"
  python bench.py --no-cpu-baseline --no-e2e --config 3 $a 2>/dev/null | tail -n 1 | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c3 $o', 'value %.1f step %.1f us sweep %.1f'%(d['value']/1e6, d['ms_per_step']*1e3, d['kernels']['sweep_kernel']['avg_us']))
"
done 2>&1 | tee gpurun_out/s5_azorder_c3.log
