#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_acceptance.py tests/test_gpu_scene_ingest.py -q -s -p no:cacheprovider --durations=5 > gpurun_out/pytest_accept.log 2>&1; tail -25 gpurun_out/pytest_accept.log
