#!/bin/bash
# GPU-box: the whole -m gpu suite (log under gpurun_out/).
mkdir -p gpurun_out
timeout ${T:-900} python -m pytest tests -m gpu -q -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
