#!/bin/bash
# One ncu --set full capture of the third launch of kernel regex $1 on C2 -> gpurun_out/prof_$2.ncu-rep
mkdir -p gpurun_out
B="python bench.py --config C2 --views 4 --steps 1 --warmup 1 --no-cpu --no-e2e --streams 1"
$B > gpurun_out/plain.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:$1 -s 2 -c 1 -f \
      -o gpurun_out/prof_$2 $B > gpurun_out/ncu_$2.log 2>&1
