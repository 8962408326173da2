# Verification of HEAD: smoke, full GPU suite, default bench + reference arm, profiles (r2g), per-config bench lines.
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2g_smoke.log 2>&1; echo smoke rc=$?
( time python -m pytest tests -x -q -m gpu ) > gpurun_out/r2g_gputests.log 2>&1; echo tests rc=$?
python bench.py > gpurun_out/r2g_bench_default.log 2>&1; echo bench rc=$?
python bench.py --impl reference > gpurun_out/r2g_bench_ref.log 2>&1; echo ref rc=$?
bash tools/capture_profiles.sh r2g 4
bash tools/capture_profiles.sh r2g 2
bash tools/bench_all.sh r2g > gpurun_out/r2g_bench_all.txt 2>&1
tail -n 3 gpurun_out/r2g_gputests.log; tail -n 1 gpurun_out/r2g_bench_default.log; cat gpurun_out/r2g_bench_all.txt
python tools/slab_parts.py 4 1 2 4 8 > gpurun_out/r2g_slab_parts.log 2>&1; tail -n 12 gpurun_out/r2g_slab_parts.log
