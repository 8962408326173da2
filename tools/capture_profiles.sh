#!/bin/bash
# Profiles of the current build (run on the GPU box from the repo root):
#   bash tools/capture_profiles.sh <tag> [config=4]
# 1. the bench line without a profiler, 2. the ncu launch list of the same
# command (gpu__time_duration, --clock-control none), 3. DRAM / LTS traffic
# per kernel over the timed window's launches, 4. one --set full capture of
# the sweep and shadow kernels of window scan 5. Outputs in gpurun_out/.
# Filtered launch indices (prep|sweep|shadow, 3 per scan): counting pass 30
# scans, then refill 10 + warmup 3 + refill 10 -> the timed window starts at
# launch 3*(30+23) = 159 and spans 60.
set -u
T=${1:-r2}
C=${2:-4}
B="python bench.py --config $C --steps 20 --warmup 3 --no-cpu-baseline --no-e2e"
$B > gpurun_out/${T}_c${C}_bench.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"prep|sweep|shadow" --csv \
    --log-file gpurun_out/${T}_c${C}_launches.csv $B > gpurun_out/${T}_c${C}_ncu_launches.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum \
    --clock-control none -k regex:"prep|sweep|shadow" -s 159 -c 60 --csv --print-units base \
    --log-file gpurun_out/${T}_c${C}_traffic.csv $B > gpurun_out/${T}_c${C}_ncu_traffic.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"sweep|shadow" -s 116 -c 2 \
    -o gpurun_out/${T}_c${C}_full $B > gpurun_out/${T}_c${C}_ncu_full.log 2>&1
tail -n 2 gpurun_out/${T}_c${C}_ncu_full.log
