#!/bin/bash
# A/B of the spatial scene order (fs_order.cu): FS_SCENE_ORDER=0 keeps input order.
for cfg in ${CFGS:-C2 C4}; do
for r in 1 2; do
  for o in 0 1; do
    FS_SCENE_ORDER=$o python bench.py --config $cfg --no-e2e --no-cpu --no-check --steps ${STEPS:-6} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg order=$o', round(d['ms_per_step'],2), 'raster_us', round(d['roofline']['avg_launch_ms']*1e3,1))"
  done
done
done
