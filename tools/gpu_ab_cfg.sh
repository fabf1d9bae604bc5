#!/bin/bash
# Same-box A/B of _variants/*.so on the bench configs in $CFGS (default C2 C4), two rounds.
LIB=paper_2409_08270_b200/_lib/libflashsplat_b200.so
cp $LIB /tmp/lib_orig.so
for r in 1 2; do
for cfg in ${CFGS:-C2 C4}; do
for v in _variants/*.so; do
  n=$(basename $v .so); cp $v $LIB
  python bench.py --config $cfg --no-e2e --no-cpu --no-check --steps ${STEPS:-6} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg $n', round(d['ms_per_step'],2), 'raster_us', round(d['roofline']['avg_launch_ms']*1e3,1))"
done
done
done
cp /tmp/lib_orig.so $LIB
