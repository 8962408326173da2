# Round 2, session 2: verify HEAD (GPU suite, smoke, bench on configs 4 and 2)
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s2_smoke.log 2>&1; echo smoke_rc=$?
timeout 1500 python -m pytest tests -x -q -m gpu > gpurun_out/s2_tests.log 2>&1; echo tests_rc=$?
python bench.py > gpurun_out/s2_bench_c4.log 2>&1; echo bench4_rc=$?
python bench.py --config 2 > gpurun_out/s2_bench_c2.log 2>&1; echo bench2_rc=$?
python bench.py --config 5 --batch 32 > gpurun_out/s2_bench_c5.log 2>&1; echo bench5_rc=$?
