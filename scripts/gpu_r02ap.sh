#!/bin/bash
mkdir -p gpurun_out/r02ap
timeout 600 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/r02ap/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ap/train_tests.log
timeout 900 python bench.py --mode train --steps 5 --warmup 3 > gpurun_out/r02ap/bench_train_C2.log 2>&1
