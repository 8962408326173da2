python -m pytest tests/test_trajectories.py tests/test_gpu_parity.py -x -q -m gpu -k "cfg4 or small or batched" > gpurun_out/sb_tests.log 2>&1; echo rc=$?
bash tools/ab_libs.sh 3 .ab_libs/sb3/libdbtsdf.so .ab_libs/sb5/libdbtsdf.so -- --no-e2e > gpurun_out/sb_ab_c4.log 2>&1
bash tools/ab_libs.sh 1 .ab_libs/sb3/libdbtsdf.so .ab_libs/sb5/libdbtsdf.so -- --no-e2e --config 2 > gpurun_out/sb_ab_c2.log 2>&1
