bash tools/ab_libs.sh 2 .ab_libs/base/libdbtsdf.so .ab_libs/warp/libdbtsdf.so -- --no-e2e --steps 20 --warmup 3 > gpurun_out/ab3_c4.log 2>&1
bash tools/ab_libs.sh 2 .ab_libs/base/libdbtsdf.so .ab_libs/warp/libdbtsdf.so -- --no-e2e --steps 20 --warmup 3 --config 2 > gpurun_out/ab3_c2.log 2>&1
DBT_LIB=.ab_libs/warp/libdbtsdf.so python -m pytest tests/test_trajectories.py -q -m gpu -k "queued" > gpurun_out/ab3_parity.log 2>&1
