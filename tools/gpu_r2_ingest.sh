#!/bin/bash
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scene_ingest.py tests/test_gpu_multi.py -q -p no:cacheprovider > gpurun_out/pytest_ingest.log 2>&1; tail -15 gpurun_out/pytest_ingest.log
timeout 600 python tools/bench_scene_ingest.py --out gpurun_out/scene_ingest_c2.json 2>&1 | tail -3
