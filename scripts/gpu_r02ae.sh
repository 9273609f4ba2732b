#!/bin/bash
mkdir -p gpurun_out/r02ae
ORBIT2_SYNC_CHECK=1 timeout 600 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/r02ae/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ae/train_tests.log
timeout 900 python scripts/train_ab.py C2 16 liborbit2.so > gpurun_out/r02ae/ab_train.log 2>&1
