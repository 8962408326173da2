python -m pytest tests -x -q -m gpu > gpurun_out/split_tests.log 2>&1; echo tests_rc=$?
bash tools/ab_libs.sh 2 .ab_libs/rec8/libdbtsdf.so .ab_libs/split/libdbtsdf.so -- --no-e2e > gpurun_out/split_ab_c4.log 2>&1
bash tools/ab_libs.sh 2 .ab_libs/rec8/libdbtsdf.so .ab_libs/split/libdbtsdf.so -- --no-e2e --config 2 > gpurun_out/split_ab_c2.log 2>&1
bash tools/ab_libs.sh 1 .ab_libs/rec8/libdbtsdf.so .ab_libs/split/libdbtsdf.so -- --no-e2e --config 3 > gpurun_out/split_ab_c3.log 2>&1
bash tools/ab_libs.sh 1 .ab_libs/rec8/libdbtsdf.so .ab_libs/split/libdbtsdf.so -- --no-e2e --config 5 --batch 32 > gpurun_out/split_ab_c5.log 2>&1
