# RED.AND.64 pairs vs one RED per voxel in the culling sweep
timeout 900 python -m pytest tests/test_trajectories.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/ab1_tests.log 2>&1; echo tests_rc=$?
bash tools/ab_libs.sh 3 .ab_libs/single/libdbtsdf.so .ab_libs/pairs/libdbtsdf.so -- --no-e2e > gpurun_out/ab1_c4.log 2>&1
bash tools/ab_libs.sh 2 .ab_libs/single/libdbtsdf.so .ab_libs/pairs/libdbtsdf.so -- --no-e2e --config 2 > gpurun_out/ab1_c2.log 2>&1
bash tools/ab_libs.sh 2 .ab_libs/single/libdbtsdf.so .ab_libs/pairs/libdbtsdf.so -- --no-e2e --config 3 > gpurun_out/ab1_c3.log 2>&1
bash tools/ab_libs.sh 2 .ab_libs/single/libdbtsdf.so .ab_libs/pairs/libdbtsdf.so -- --no-e2e --config 5 --batch 32 > gpurun_out/ab1_c5.log 2>&1
