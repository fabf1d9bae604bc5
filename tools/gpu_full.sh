#!/bin/bash
# Full GPU suite + the C2 bench line (the driver's round-end commands) + checked build suite
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; tail -1 gpurun_out/bench_c2.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2', d['ms_per_step'], d['e2e']['s_per_scene'], d['roofline']['avg_launch_ms'], d['shard_check']['matrix_bit_identical'], d['clocks'])"
if [ -n "$CHECKED" ]; then make -s -j8 -C paper_2409_08270_b200/csrc checked > gpurun_out/make_checked.log 2>&1; FS_LIB=checked timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_checked.log 2>&1; echo "checked: $(tail -1 gpurun_out/pytest_checked.log)"; fi
