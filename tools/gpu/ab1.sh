set -x
bash tools/ab_libs.sh 2 .ab_libs/base/libdbtsdf.so .ab_libs/nored/libdbtsdf.so .ab_libs/nocst/libdbtsdf.so .ab_libs/noshadow/libdbtsdf.so -- --no-e2e --steps 20 --warmup 3 > gpurun_out/ab1_c4.log 2>&1
bash tools/ab_libs.sh 1 .ab_libs/base/libdbtsdf.so .ab_libs/nored/libdbtsdf.so .ab_libs/nocst/libdbtsdf.so .ab_libs/noshadow/libdbtsdf.so -- --no-e2e --steps 20 --warmup 3 --config 2 > gpurun_out/ab1_c2.log 2>&1
python -m pytest tests/test_integration_shim.py -q -m gpu > gpurun_out/shim.log 2>&1
