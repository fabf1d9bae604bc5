#!/bin/bash
mkdir -p gpurun_out/parity
FS_PARITY_DIR=gpurun_out/parity timeout 1500 python -m pytest tests/test_gpu_configs.py -q -p no:cacheprovider --durations=0 > gpurun_out/pytest_configs.log 2>&1
tail -15 gpurun_out/pytest_configs.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node=1 --master-addr=127.0.0.1 --master-port=29533 bench.py --steps 4 --no-cpu > gpurun_out/bench_torchrun1.log 2>&1
tail -1 gpurun_out/bench_torchrun1.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['n_gpus'], d['ms_per_step'], d['e2e']['s_per_scene'], d['config']['parallelism'], d['shard_check'])"
