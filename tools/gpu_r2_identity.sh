#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python tools/shard_identity.py --out gpurun_out/shard_identity.json > gpurun_out/shard_identity.log 2>&1; echo rc=$?
tail -5 gpurun_out/shard_identity.log
