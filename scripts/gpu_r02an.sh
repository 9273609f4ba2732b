#!/bin/bash
# round 2: 4 GPUs -- multi-GPU tests, SP bench (C2, C4), data-parallel training
mkdir -p gpurun_out/r02an
timeout 900 python -m pytest tests/test_peer_sp.py tests/test_sequence_parallel.py -q -m gpu > gpurun_out/r02an/pytest_mgpu.log 2>&1
echo "rc=$?" >> gpurun_out/r02an/pytest_mgpu.log
timeout 600 python bench.py --gpus 4 > gpurun_out/r02an/bench_sp4_c2.log 2>&1
timeout 600 python bench.py --gpus 2 > gpurun_out/r02an/bench_sp2_c2.log 2>&1
timeout 600 python bench.py > gpurun_out/r02an/bench_sp1_c2.log 2>&1
timeout 900 python bench.py --gpus 4 --config C4 --steps 3 > gpurun_out/r02an/bench_sp4_c4.log 2>&1
timeout 900 python bench.py --gpus 4 --mode train --steps 5 --warmup 3 > gpurun_out/r02an/bench_train_dp4.log 2>&1
