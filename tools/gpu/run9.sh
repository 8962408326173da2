python -m pytest tests/test_trajectories.py -x -q -m gpu -k "cfg3" > gpurun_out/traj_cfg3.log 2>&1; echo rc=$?
/usr/bin/time -v python -m pytest tests/test_full_size.py -x -q -m gpu > gpurun_out/full_size.log 2>&1; echo rc=$?
