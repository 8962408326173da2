python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "Async" > gpurun_out/s5_async2_tests.log 2>&1; echo tests rc=$?; tail -n 3 gpurun_out/s5_async2_tests.log
