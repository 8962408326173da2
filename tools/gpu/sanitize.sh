# compute-sanitizer over the GPU parity suite's small cases (memcheck: global
# out-of-bounds / misaligned accesses and leaks; racecheck: shared-memory
# hazards; initcheck: reads of uninitialised global memory; synccheck)
set -x
K='small or batched or Reference or Certificate or Pending or Interleaved or SweepPaths or Exact or Replica or slab'
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1500 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 \
    python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "$K and not cfg" -p no:randomly > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
done
python tools/e2e_cfg.py 4 > gpurun_out/e2e_c4.log 2>&1
python tools/e2e_cfg.py 2 > gpurun_out/e2e_c2.log 2>&1
