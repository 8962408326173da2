# bounded batches per sweep block + high-priority shadow stream (graphs off for both arms)
export DBT_NO_GRAPH=1
L=".ab_libs/plmcw4/libdbtsdf.so .ab_libs/bpb4/libdbtsdf.so .ab_libs/bpb2/libdbtsdf.so .ab_libs/bpb8/libdbtsdf.so .ab_libs/bpb4np/libdbtsdf.so"
bash tools/ab_libs.sh 2 $L -- --no-e2e > gpurun_out/s5_ab6_c4.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 2 > gpurun_out/s5_ab6_c2.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 5 --batch 32 > gpurun_out/s5_ab6_c5.log 2>&1
for c in 4 2 5; do echo "== config $c"; cut -c1-50,100-170 gpurun_out/s5_ab6_c$c.log; done
DBT_LIB=.ab_libs/bpb4/libdbtsdf.so python -m pytest tests/test_trajectories.py -x -q -m gpu -k "cfg4 or config4 or c4" > gpurun_out/s5_bpb_tests.log 2>&1; echo tests rc=$?; tail -n 2 gpurun_out/s5_bpb_tests.log
