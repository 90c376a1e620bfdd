#!/bin/bash
# Final-state check: GPU parity suite, smoke, the default bench line (ours) and
# the reference arm, plus a torchrun (1 process) launch of the bench.
mkdir -p gpurun_out
timeout 600 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python __graft_entry__.py --smoke-only > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.log 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 1 --steps 20 --warmup 3 --no-e2e --no-cpu --no-variants > gpurun_out/bench_torchrun.log 2>&1
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; tail -c 400 gpurun_out/bench.log; echo; tail -c 300 gpurun_out/bench_ref.log; echo; tail -c 300 gpurun_out/bench_torchrun.log
