python -m pytest tests/test_multirank_engine.py -x -q -m gpu > gpurun_out/mr_engine.log 2>&1; echo rc=$?
python bench.py --no-cpu-baseline > gpurun_out/bench_c4b.log 2>&1
