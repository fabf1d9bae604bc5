#!/bin/bash
# Same-box A/B of _variants/*.so on the default bench (device value and e2e), two rounds.
LIB=paper_2409_08270_b200/_lib/libflashsplat_b200.so
cp $LIB /tmp/lib_orig.so
for r in 1 2; do
for v in _variants/*.so; do
  n=$(basename $v .so); cp $v $LIB
  python bench.py --no-cpu --no-check --steps ${STEPS:-6} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); e=d['e2e']; print('$n', round(d['ms_per_step'],2), 'e2e', round(e['s_per_scene']*1e3,2), 'pageable', round(e['s_per_scene_pageable_inputs']*1e3,2))"
done
done
cp /tmp/lib_orig.so $LIB
