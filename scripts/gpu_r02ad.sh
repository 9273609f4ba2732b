#!/bin/bash
# round 2: 2 GPUs -- multi-GPU parity tests, SP bench, data-parallel training bench (NCCL all-reduce)
mkdir -p gpurun_out/r02ad
timeout 900 python -m pytest tests/test_peer_sp.py tests/test_sequence_parallel.py -q -m gpu > gpurun_out/r02ad/pytest_mgpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02ad/pytest_mgpu.log
timeout 600 python bench.py --gpus 2 > gpurun_out/r02ad/bench_sp2.log 2>&1
timeout 900 python bench.py --gpus 2 --mode train --steps 5 --warmup 3 > gpurun_out/r02ad/bench_train_dp2.log 2>&1
