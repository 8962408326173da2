set -x
python -m pytest tests -x -q -m gpu > gpurun_out/gpu_tests.log 2>&1; echo tests_rc=$?
python tools/slab_parts.py 2 > gpurun_out/slab_parts_c2.log 2>&1
python tools/slab_parts.py 4 > gpurun_out/slab_parts_c4.log 2>&1
