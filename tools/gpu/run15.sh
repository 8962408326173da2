# A/B: policy hoist, predicated chunk loads, no-shadow lower bound
L=".ab_libs/base/libdbtsdf.so .ab_libs/hoist/libdbtsdf.so .ab_libs/predc/libdbtsdf.so .ab_libs/pred/libdbtsdf.so .ab_libs/noshadow/libdbtsdf.so"
bash tools/ab_libs.sh 3 $L -- --no-e2e > gpurun_out/s5_ab1_c4.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 2 > gpurun_out/s5_ab1_c2.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 3 > gpurun_out/s5_ab1_c3.log 2>&1
cat gpurun_out/s5_ab1_c4.log gpurun_out/s5_ab1_c2.log gpurun_out/s5_ab1_c3.log
