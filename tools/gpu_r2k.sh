#!/bin/bash
# round 2: run_host / with_batch tests; bench under torchrun (1 rank) and via the self-launcher
mkdir -p gpurun_out
( timeout 900 python -m pytest tests/test_gpu_run_host.py -q -m gpu 2>&1 | tail -5
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --no-configs --no-variants --cpu-seconds 2 2>&1 | grep '^{' > gpurun_out/r2k_bench_torchrun1.jsonl; echo "torchrun rc $?"
  python -c "import json; d=json.loads(open('gpurun_out/r2k_bench_torchrun1.jsonl').readline()); print({k: d[k] for k in ('value','n_gpus','ms_per_step','scaling')}, d['config']['parallelism'])"
) > gpurun_out/r2k.log 2>&1
cat gpurun_out/r2k.log
