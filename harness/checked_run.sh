#!/bin/bash
# The checked build (device-side bounds / protocol assertions, -DIVFPQ_CHECKED)
# through the golden searches and the GPU parity tests.  Build here:
#   bash harness/variants_build.sh checked "-DIVFPQ_CHECKED"
# run on the box:
#   bash harness/checked_run.sh
L=$PWD/harness/variants/libivfpq_b200_checked.so
IVFPQ_LIB=$L timeout 600 python -m harness.sanitize_run
IVFPQ_LIB=$L timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin.py -x -q -m gpu 2>&1 | tail -2
