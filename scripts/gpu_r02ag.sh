#!/bin/bash
mkdir -p gpurun_out/r02ag
ORBIT2_SYNC_CHECK=1 timeout 600 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/r02ag/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02ag/train_tests.log
timeout 900 python scripts/train_ab.py C2 16 liborbit2.so > gpurun_out/r02ag/ab_train_c2.log 2>&1
timeout 900 python scripts/train_ab.py C3 16 liborbit2.so > gpurun_out/r02ag/ab_train_c3.log 2>&1
