set -x
bash tools/ab_libs.sh 2 .ab_libs/base/libdbtsdf.so .ab_libs/split/libdbtsdf.so .ab_libs/nored/libdbtsdf.so -- --no-e2e --steps 20 --warmup 3 > gpurun_out/ab2_c4.log 2>&1
python tools/redundancy.py 14 > gpurun_out/redundancy.log 2>&1
