L=".ab_libs/pg8/libdbtsdf.so .ab_libs/pg5/libdbtsdf.so .ab_libs/pg12/libdbtsdf.so .ab_libs/pg27/libdbtsdf.so"
bash tools/ab_libs.sh 2 $L -- --no-e2e > gpurun_out/s5_ab8_c4.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 2 > gpurun_out/s5_ab8_c2.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 3 > gpurun_out/s5_ab8_c3.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 5 --batch 32 > gpurun_out/s5_ab8_c5.log 2>&1
for c in 4 2 3 5; do echo "== config $c"; cut -c1-50,100-170 gpurun_out/s5_ab8_c$c.log; done
