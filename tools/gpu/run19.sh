# uniform-stream certificate gather: equality check build, parity subset, A/B
DBT_LIB=.ab_libs/unicheck/libdbtsdf.so python bench.py --no-cpu-baseline --no-e2e > gpurun_out/s5_unicheck_c4.log 2>&1; echo unicheck c4 rc=$?
DBT_LIB=.ab_libs/unicheck/libdbtsdf.so python bench.py --no-cpu-baseline --no-e2e --config 2 > gpurun_out/s5_unicheck_c2.log 2>&1; echo unicheck c2 rc=$?
DBT_LIB=.ab_libs/unicheck/libdbtsdf.so python bench.py --no-cpu-baseline --no-e2e --config 5 --batch 8 > gpurun_out/s5_unicheck_c5.log 2>&1; echo unicheck c5 rc=$?
tail -n 2 gpurun_out/s5_unicheck_c4.log | cut -c1-300
( time python -m pytest tests/test_trajectories.py tests/test_gpu_parity.py -x -q -m gpu ) > gpurun_out/s5_uni_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/s5_uni_tests.log
L=".ab_libs/hoist/libdbtsdf.so .ab_libs/uni/libdbtsdf.so"
bash tools/ab_libs.sh 3 $L -- --no-e2e > gpurun_out/s5_ab3_c4.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 2 > gpurun_out/s5_ab3_c2.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 3 > gpurun_out/s5_ab3_c3.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 5 --batch 32 > gpurun_out/s5_ab3_c5.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 1 > gpurun_out/s5_ab3_c1.log 2>&1
cat gpurun_out/s5_ab3_c*.log
