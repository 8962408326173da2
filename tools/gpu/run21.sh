# centres per block batch re-tuned on the cheaper phase A
L=".ab_libs/plm/libdbtsdf.so .ab_libs/plmcw4/libdbtsdf.so .ab_libs/plmcw2/libdbtsdf.so .ab_libs/plmcw3/libdbtsdf.so .ab_libs/plmcw5/libdbtsdf.so .ab_libs/plmcw6/libdbtsdf.so"
bash tools/ab_libs.sh 2 $L -- --no-e2e > gpurun_out/s5_ab5_c4.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 2 > gpurun_out/s5_ab5_c2.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 3 > gpurun_out/s5_ab5_c3.log 2>&1
bash tools/ab_libs.sh 1 $L -- --no-e2e --config 5 --batch 32 > gpurun_out/s5_ab5_c5.log 2>&1
bash tools/ab_libs.sh 2 $L -- --no-e2e --config 1 > gpurun_out/s5_ab5_c1.log 2>&1
for c in 4 2 3 5 1; do echo "== config $c"; cut -c1-50,100-170 gpurun_out/s5_ab5_c$c.log; done
