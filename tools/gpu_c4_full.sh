#!/bin/bash
# C4 at full size (3M Gaussians, 300 views 1920x1080, E=64) against the oracle on all host threads.
mkdir -p gpurun_out
timeout 2400 python tools/parity_full.py --config C4 --out gpurun_out/parity_full_c4_r2.json > gpurun_out/parity_full_c4.log 2>&1; echo rc=$?
tail -c 600 gpurun_out/parity_full_c4.log
