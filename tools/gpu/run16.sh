# micro-optimised phase B / batch loop: parity subset, then A/B against the hoist build
( time python -m pytest tests/test_trajectories.py tests/test_gpu_parity.py -x -q -m gpu ) > gpurun_out/s5_micro_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/s5_micro_tests.log
L=".ab_libs/hoist/libdbtsdf.so .ab_libs/micro/libdbtsdf.so"
bash tools/ab_libs.sh 3 $L -- --no-e2e > gpurun_out/s5_ab2_c4.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 2 > gpurun_out/s5_ab2_c2.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 3 > gpurun_out/s5_ab2_c3.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 5 --batch 32 > gpurun_out/s5_ab2_c5.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 1 > gpurun_out/s5_ab2_c1.log 2>&1
cat gpurun_out/s5_ab2_c*.log
