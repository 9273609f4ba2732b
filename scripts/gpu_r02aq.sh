#!/bin/bash
mkdir -p gpurun_out/r02aq
timeout 900 python -m pytest tests/test_gpu_train_sp.py -x -q > gpurun_out/r02aq/train_sp_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02aq/train_sp_tests.log
timeout 900 python bench.py --gpus 2 --mode train --train-tiles --steps 5 --warmup 3 > gpurun_out/r02aq/bench_train_tiles2.log 2>&1
timeout 900 python bench.py --gpus 2 --mode train --steps 5 --warmup 3 > gpurun_out/r02aq/bench_train_dp2.log 2>&1
