for c in 4 2; do for rep in 1 2; do for m in write clean none; do
  if [ $m = none ]; then f="--no-flush"; else f="--flush $m"; fi
  python bench.py --config $c --steps 40 --warmup 5 --no-cpu-baseline --no-e2e $f > gpurun_out/abf_c${c}_${m}_${rep}.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/abf_c${c}_${m}_${rep}.log').read().strip().splitlines()[-1]); print('c$c $m $rep', round(d['value']/1e6,1), round(d['ms_per_step']*1e3,1), {k:round(v['avg_us'],1) for k,v in d['kernels'].items()})"
done; done; done
