# Last check of HEAD: smoke, full GPU suite, default bench line and reference arm
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo smoke rc=$?
( time python -m pytest tests -x -q -m gpu ) > gpurun_out/final_gputests.log 2>&1; echo tests rc=$?
python bench.py > gpurun_out/final_bench.log 2>&1; echo bench rc=$?
python bench.py --impl reference > gpurun_out/final_bench_ref.log 2>&1; echo ref rc=$?
tail -n 1 gpurun_out/final_smoke.log; grep -E "passed|failed" gpurun_out/final_gputests.log | tail -n 1
tail -n 1 gpurun_out/final_bench.log | cut -c1-260; tail -n 1 gpurun_out/final_bench_ref.log | cut -c1-200
