set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
python -m pytest tests/test_trajectories.py -x -q -m gpu > gpurun_out/traj.log 2>&1; echo traj_rc=$?
timeout 900 python bench.py > gpurun_out/bench_c4.log 2>&1; echo bench_rc=$?
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/bench_c2.log 2>&1; echo bench2_rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum --clock-control none -k regex:"prep|sweep|shadow" -s 159 -c 60 --csv --print-units base --log-file gpurun_out/c4_traffic.csv python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 3 > gpurun_out/c4_ncu_traffic.log 2>&1; echo ncu1_rc=$?
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"sweep|shadow" -s 116 -c 4 -o gpurun_out/c4_full python bench.py --no-cpu-baseline --no-e2e --steps 20 --warmup 3 > gpurun_out/c4_ncu_full.log 2>&1; echo ncu2_rc=$?
tail -3 gpurun_out/c4_ncu_full.log
