mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -p no:cacheprovider > gpurun_out/pytest_multi.log 2>&1; tail -15 gpurun_out/pytest_multi.log
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; tail -5 gpurun_out/pytest_gpu.log
for acc in fixed f64; do timeout 300 python bench.py --acc $acc --no-cpu > gpurun_out/bench_c2_$acc.log 2>&1; tail -1 gpurun_out/bench_c2_$acc.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$acc', d['ms_per_step'], d['e2e']['s_per_scene'], d['roofline']['avg_launch_ms'], d['shard_check'])"; done
