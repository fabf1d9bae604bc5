#!/bin/bash
# GPU-box check used during kernel work: parity tests, a short bench, launch list.
# usage (from the repo root, via gpurun): bash tools/gpucheck.sh [pytest-args...]
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider "$@" > gpurun_out/pytest_gpu.log 2>&1
tail -1 gpurun_out/pytest_gpu.log
B="python bench.py --config C2 --views 4 --steps 1 --warmup 1 --no-cpu --no-e2e --streams 1"
$B > gpurun_out/plain.log 2>&1 && \
  ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv \
      --log-file gpurun_out/launches.csv $B > gpurun_out/ncu.log 2>&1
python tools/launches.py gpurun_out/launches.csv 16 | head -4
