#!/bin/bash
# ncu evidence for the mesher and the exact voxels_written kernels (GPU box):
#   bash tools/capture_mesh_profiles.sh <tag>
set -u
T=${1:-r05}
python tools/prof_mesh.py --exact > gpurun_out/${T}_prof_mesh.log 2>&1 || exit 1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"mesh_|exact_|replica_" --csv --print-units base \
    --log-file gpurun_out/${T}_mesh_launches.csv python tools/prof_mesh.py --exact > gpurun_out/${T}_ncu_mesh_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"mesh_flags|mesh_active|mesh_vert|mesh_tri|exact_count" -c 7 \
    -o gpurun_out/${T}_mesh_full python tools/prof_mesh.py --exact > gpurun_out/${T}_ncu_mesh_full.log 2>&1
tail -n 2 gpurun_out/${T}_ncu_mesh_full.log
