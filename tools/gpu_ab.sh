#!/bin/bash
# A/B: parity subset + full C2 solve timing for every _variants/*.so
mkdir -p gpurun_out
LIB=paper_2409_08270_b200/_lib/libflashsplat_b200.so
cp $LIB /tmp/lib_orig.so
for v in _variants/*.so; do
  n=$(basename $v .so); cp $v $LIB
  timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_render.py tests/test_gpu_configs.py -x -q -p no:cacheprovider -k "${AB_K:-not nothing}" > gpurun_out/ab_$n.pytest.log 2>&1
  echo "$n: $(tail -1 gpurun_out/ab_$n.pytest.log)"
done
for r in 1 2; do
for v in _variants/*.so; do
  n=$(basename $v .so); cp $v $LIB
  python bench.py --no-e2e --no-cpu --no-check --steps 8 ${AB_ARGS} 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$n', round(d['ms_per_step'],2), 'raster_us', round(d['roofline']['avg_launch_ms']*1e3,1), 'exact', d['counters_per_step']['exact_evals'], 'steps', d['counters_per_step']['tile_steps'])"
done
done
cp /tmp/lib_orig.so $LIB
