# Verification of HEAD: smoke, full GPU suite, default bench + reference arm, profiles (r2e), per-config bench lines.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1; echo smoke rc=$?
( time python -m pytest tests -x -q -m gpu ) > gpurun_out/r2e_gputests.log 2>&1; echo tests rc=$?
python bench.py > gpurun_out/r2e_bench_default.log 2>&1; echo bench rc=$?
python bench.py --impl reference > gpurun_out/r2e_bench_ref.log 2>&1; echo ref rc=$?
bash tools/capture_profiles.sh r2e 4
bash tools/capture_profiles.sh r2e 2
bash tools/bench_all.sh r2e > gpurun_out/r2e_bench_all.txt 2>&1
tail -n 3 gpurun_out/r2e_gputests.log; tail -n 1 gpurun_out/r2e_bench_default.log; cat gpurun_out/r2e_bench_all.txt
