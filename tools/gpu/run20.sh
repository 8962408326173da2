# plane-cut loop over set bits; batch-size / balance knobs re-checked on the new phase A
L=".ab_libs/uni/libdbtsdf.so .ab_libs/plm/libdbtsdf.so .ab_libs/plmcw4/libdbtsdf.so .ab_libs/plmcw16/libdbtsdf.so .ab_libs/plmbal/libdbtsdf.so"
bash tools/ab_libs.sh 3 $L -- --no-e2e > gpurun_out/s5_ab4_c4.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 2 > gpurun_out/s5_ab4_c2.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 3 > gpurun_out/s5_ab4_c3.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 5 --batch 32 > gpurun_out/s5_ab4_c5.log 2>&1
cat gpurun_out/s5_ab4_c*.log
DBT_LIB=.ab_libs/plm/libdbtsdf.so python -m pytest tests/test_trajectories.py tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/s5_plm_tests.log 2>&1; echo tests rc=$?
tail -n 3 gpurun_out/s5_plm_tests.log
