# 32-bit row-task emission: parity subset (main build = e32), then A/B against HEAD
( time python -m pytest tests/test_trajectories.py tests/test_gpu_parity.py tests/test_multirank_engine.py -x -q -m gpu ) > gpurun_out/s5_e32_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/s5_e32_tests.log
L=".ab_libs/head/libdbtsdf.so .ab_libs/e32/libdbtsdf.so"
bash tools/ab_libs.sh 3 $L -- --no-e2e > gpurun_out/s5_ab7_c4.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 2 > gpurun_out/s5_ab7_c2.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 3 > gpurun_out/s5_ab7_c3.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 5 --batch 32 > gpurun_out/s5_ab7_c5.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 1 > gpurun_out/s5_ab7_c1.log 2>&1
for c in 4 2 3 5 1; do echo "== config $c"; cut -c1-50,100-170 gpurun_out/s5_ab7_c$c.log; done
