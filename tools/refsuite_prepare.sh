#!/bin/bash
# Build container only: make the reference runnable on the GPU box for
# tools/gpu/refsuite.sh and tests/test_integration_shim.py::test_live_reference_crosscheck.
#   baseline/_ref        pip --target install of the unmodified reference package (git-ignored, travels)
#   baseline/_ref_tests  scratch copy of the reference's own tests, for ONE gpurun call
#                        (git-ignored; delete it afterwards: tools/refsuite_prepare.sh clean)
set -e
cd "$(dirname "$0")/.."
if [ "$1" == "clean" ]; then rm -rf baseline/_ref_tests; exit 0; fi
rm -rf /tmp/refpkg baseline/_ref baseline/_ref_tests
cp -r /root/reference/pkg /tmp/refpkg   # the source tree is read-only; pip builds in a copy
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse --target baseline/_ref /tmp/refpkg
cp -r /root/reference/pkg/tests baseline/_ref_tests
echo "baseline/_ref and baseline/_ref_tests ready; run: gpurun -- 'bash tools/gpu/refsuite.sh'"
