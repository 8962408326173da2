bash tools/capture_profiles.sh r2 4
bash tools/capture_profiles.sh r2 2
python bench.py > gpurun_out/r2_bench_default.log 2>&1
