#!/bin/bash
# A/B of full 4-stream C2 solves (ms/step) for each _variants/*.so
LIB=paper_2409_08270_b200/_lib/libflashsplat_b200.so
cp $LIB /tmp/lib_orig.so
for v in _variants/*.so; do
  n=$(basename $v .so); cp $v $LIB
  for r in 1 2; do
    python bench.py --no-e2e --no-cpu --steps 6 ${AB_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['ms_per_step'],2), round(d['roofline']['avg_launch_ms']*1e3,1))"
  done
done
cp /tmp/lib_orig.so $LIB
