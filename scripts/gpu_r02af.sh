#!/bin/bash
mkdir -p gpurun_out/r02af
ORBIT2_SYNC_CHECK=1 timeout 900 python -m pytest tests/test_gpu_train.py -x -q -k wide > gpurun_out/r02af/train_wide.log 2>&1
echo "rc=$?" >> gpurun_out/r02af/train_wide.log
timeout 900 python bench.py --mode train --config C3 --steps 3 --warmup 3 > gpurun_out/r02af/bench_train_c3.log 2>&1
