#!/bin/bash
# Profiles of the current build (run on the GPU box from the repo root):
#   bash tools/capture_profiles.sh <tag>
# 1. the bench line without a profiler, 2. the ncu launch list of the same
# command (gpu__time_duration, --clock-control none), 3. DRAM / LTS traffic per
# kernel, 4. one --set full capture of each engine kernel on config-2 scan 19
# (prof_cfg.py, L2 flushed between scans). Outputs in gpurun_out/.
set -u
T=${1:-r03}
B="python bench.py --steps 30 --warmup 5 --no-cpu-baseline"
$B > gpurun_out/${T}_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep|sweep|shadow" --csv \
    --log-file gpurun_out/${T}_launches_bench.csv $B > gpurun_out/${T}_ncu_launches.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum \
    --clock-control none -k regex:"prep|sweep|shadow" --csv --print-units base \
    --log-file gpurun_out/${T}_traffic_bench.csv $B > gpurun_out/${T}_ncu_traffic.log 2>&1
python tools/prof_cfg.py 2 21 > gpurun_out/${T}_prof_cfg2.log 2>&1 || exit 1
ncu --set full --clock-control none --import-source on -k regex:"prep|sweep|shadow" -s 57 -c 3 \
    -o gpurun_out/${T}_cfg2_full python tools/prof_cfg.py 2 21 > gpurun_out/${T}_ncu_full.log 2>&1
tail -n 2 gpurun_out/${T}_ncu_full.log
