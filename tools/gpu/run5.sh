python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "slab or interleav or shard or part" > gpurun_out/slab_tests.log 2>&1; echo rc=$?
python tools/slab_parts.py 4 1 8 > gpurun_out/slab_c4.log 2>&1
