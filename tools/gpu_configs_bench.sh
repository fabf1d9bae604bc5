#!/bin/bash
# bench.py over every BASELINE config (+ the iid worst cases) -> gpurun_out/bench_r2_<cfg>.json
mkdir -p gpurun_out
for cfg in C1 C2 C3 C4 C5; do
  timeout 900 python bench.py --config $cfg --steps ${STEPS:-8} > gpurun_out/bench_r2_$cfg.json 2> gpurun_out/bench_r2_$cfg.err
  tail -1 gpurun_out/bench_r2_$cfg.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', round(d['ms_per_step'],2), round(d['e2e']['s_per_scene']*1e3,2), round(d['e2e']['s_per_scene_pageable_inputs']*1e3,2), d['shard_check']['matrix_bit_identical'], d['clocks']['sm_mhz'])"
done
for cfg in C2 C3; do
  timeout 900 python bench.py --config $cfg --iid --steps 6 --no-cpu > gpurun_out/bench_r2_${cfg}_iid.json 2>/dev/null
  tail -1 gpurun_out/bench_r2_${cfg}_iid.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg-iid', round(d['ms_per_step'],2), round(d['e2e']['s_per_scene']*1e3,2))"
done
