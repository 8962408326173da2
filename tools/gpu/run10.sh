for o in none morton xyz random; do
  a=""; [ $o != none ] && a="--diag-order $o"
  echo "$o $(python bench.py --no-cpu-baseline --no-e2e $a | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e6,1), round(d["ms_per_step"]*1e3,1), {k: round(v["avg_us"],1) for k,v in d["kernels"].items()})')"
done > gpurun_out/order_ab.log 2>&1
