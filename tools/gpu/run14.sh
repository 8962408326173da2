# Re-entry verification of HEAD: full GPU suite, profiles of the f16-cache build (r2d), per-config bench lines.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2d_smoke.log 2>&1; echo smoke rc=$?
( time python -m pytest tests -x -q -m gpu ) > gpurun_out/r2d_gputests.log 2>&1; echo tests rc=$?
python bench.py > gpurun_out/r2d_bench_default.log 2>&1; echo bench rc=$?
python bench.py --impl reference > gpurun_out/r2d_bench_ref.log 2>&1; echo ref rc=$?
bash tools/capture_profiles.sh r2d 4
bash tools/capture_profiles.sh r2d 2
bash tools/bench_all.sh r2d > gpurun_out/r2d_bench_all.txt 2>&1
tail -n 3 gpurun_out/r2d_gputests.log; tail -n 1 gpurun_out/r2d_bench_default.log; cat gpurun_out/r2d_bench_all.txt
