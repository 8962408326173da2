python -m pytest tests/test_trajectories.py tests/test_multirank_engine.py -x -q -m gpu -k "queued or sharded" > gpurun_out/graph_dev_tests.log 2>&1; echo rc=$?
for r in 1 2; do for c in 4 2; do
  echo "graph c$c $(python bench.py --config $c --no-cpu-baseline --no-e2e | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e6,1), round(d["ms_per_step"]*1e3,1), d["gpu_launches"])')"
  echo "nograph c$c $(DBT_NO_GRAPH=1 python bench.py --config $c --no-cpu-baseline --no-e2e | python -c 'import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(round(d["value"]/1e6,1), round(d["ms_per_step"]*1e3,1), d["gpu_launches"])')"
done; done > gpurun_out/graph_dev_ab.log 2>&1
