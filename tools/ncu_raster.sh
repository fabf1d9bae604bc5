#!/bin/bash
# One ncu --set full capture of the raster kernel (third launch) on C2.
mkdir -p gpurun_out
B="python bench.py --config C2 --views 4 --steps 1 --warmup 1 --no-cpu --no-e2e --streams 1"
$B > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:raster_kernel -s 2 -c 1 -f \
      -o gpurun_out/prof_raster $B > gpurun_out/ncu_full.log 2>&1
