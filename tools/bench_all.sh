#!/bin/bash
# Per-config bench lines (BASELINE.json configs 1-5) into gpurun_out/bench_cfg*.log
python bench.py --config 1 --steps 50 --warmup 5 > gpurun_out/bench_cfg1.log 2>&1
python bench.py --config 2 > gpurun_out/bench_cfg2.log 2>&1
python bench.py --config 3 --steps 40 --warmup 4 --max-scans 44 > gpurun_out/bench_cfg3.log 2>&1
python bench.py --config 4 --steps 24 --warmup 3 --max-scans 27 > gpurun_out/bench_cfg4.log 2>&1
for b in 8 32; do
  python bench.py --config 5 --batch $b --steps 4 --warmup 1 --max-scans $((5*b)) --no-cpu-baseline > gpurun_out/bench_cfg5_b$b.log 2>&1
done
python bench.py --impl reference --config 2 --steps 20 --warmup 2 > gpurun_out/bench_ref_cfg2.log 2>&1
