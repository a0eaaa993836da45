#!/bin/bash
# Stage the UNMODIFIED reference for the --impl reference arm and the
# reference-suite test (tests/test_gpu_reference_suite.py): pip-install the
# package into baseline/_ref (git-ignored, travels to the GPU box) and copy
# its own pkg/tests next to it.  Needs /root/reference (this container only).
set -e
cd "$(dirname "$0")/.."
rm -rf /tmp/corutv_ref_src baseline/_ref
cp -r /root/reference/pkg /tmp/corutv_ref_src
# --no-deps: numpy is in the image; the wheelhouse has no numpy wheel to resolve
python -m pip install -q --no-index --no-build-isolation --no-deps --find-links /opt/wheelhouse \
    --target baseline/_ref /tmp/corutv_ref_src
cp -r /root/reference/pkg/tests baseline/_ref/ref_tests
echo "staged: $(ls baseline/_ref)"
