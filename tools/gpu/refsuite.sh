# The reference's own hot-path suites against the drop-in (integration/pytest_b200.py).
# baseline/_ref = pip-installed reference package, baseline/_ref_tests = a scratch copy of
# its tests (both git-ignored, made in the build container for this call only).
export PYTHONPATH=$PWD/baseline/_ref:$PWD/integration
export BITSDF_B200_LIB=$PWD/paper_2509_20081_b200/libdbtsdf.so
T="baseline/_ref_tests/test_integrator.py baseline/_ref_tests/test_oracle.py baseline/_ref_tests/test_acceptance.py baseline/_ref_tests/test_mesher.py"
O="--rootdir baseline/_ref_tests -c /dev/null -p no:cacheprovider -rfEs -v"
( time python -m pytest $O $T ) > gpurun_out/refsuite_cpu_unpatched.log 2>&1; echo unpatched rc=$?
( time BITSDF_B200_CROSSCHECK=1 DBT_EXACT_VOXELS_WRITTEN=1 python -m pytest -p pytest_b200 $O $T ) > gpurun_out/refsuite_b200_crosscheck.log 2>&1; echo crosscheck rc=$?
( time python -m pytest -p pytest_b200 $O $T ) > gpurun_out/refsuite_b200.log 2>&1; echo plain rc=$?
tail -n 15 gpurun_out/refsuite_cpu_unpatched.log; tail -n 30 gpurun_out/refsuite_b200_crosscheck.log; tail -n 15 gpurun_out/refsuite_b200.log
