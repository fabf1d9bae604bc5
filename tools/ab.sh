#!/bin/bash
# A/B kernel variants on the GPU box: every _variants/<name>.so is copied over the
# in-tree library in turn and the C2 launch list is taken (per-kernel averages).
mkdir -p gpurun_out
LIB=paper_2409_08270_b200/_lib/libflashsplat_b200.so
cp $LIB /tmp/lib_orig.so
B="python bench.py --config ${AB_CFG:-C2} --views 4 --steps 1 --warmup 1 --no-cpu --no-e2e --streams 1"
for v in _variants/*.so; do
  n=$(basename $v .so)
  cp $v $LIB
  if [ -n "$AB_K" ]; then
    timeout 600 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "$AB_K" > gpurun_out/ab_$n.pytest.log 2>&1
    echo "$n: $(tail -1 gpurun_out/ab_$n.pytest.log)"
  fi
  $B > gpurun_out/ab_$n.log 2>&1 && \
    ncu --metrics gpu__time_duration.sum --clock-control none -c 500 --csv \
        --log-file gpurun_out/ab_$n.csv $B > /dev/null 2>&1
  python tools/launches.py gpurun_out/ab_$n.csv 16 | grep -E "raster_kernel|project_kernel|bin_emit|bin_count|TOTAL" | sed "s/^/$n: /"
done
cp /tmp/lib_orig.so $LIB
