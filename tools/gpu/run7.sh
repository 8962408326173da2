python -m pytest tests -x -q -m gpu -k "not cfg3_traj128 and not config4_full" > gpurun_out/gpu_tests_graph.log 2>&1; echo rc=$?
for c in 2 4; do
  python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_graph_c$c.log 2>&1
  DBT_NO_GRAPH=1 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_nograph_c$c.log 2>&1
done
