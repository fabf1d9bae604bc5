#!/bin/bash
# The GPU test-suite and the sanitizer workloads against the bounds-checked build
# (device FS_CHECK asserts; compute-sanitizer is closed on the GPU pool).
mkdir -p gpurun_out
FS_LIB=checked timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1
tail -4 gpurun_out/pytest_checked.log
FS_LIB=checked timeout 600 python tools/sanitize_case.py all > gpurun_out/checked_cases.log 2>&1; echo "cases rc=$?"; tail -5 gpurun_out/checked_cases.log
grep -c "FS_CHECK failed" gpurun_out/pytest_checked.log gpurun_out/checked_cases.log
