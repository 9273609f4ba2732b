#!/bin/bash
# round 2: attention backward with query halves in ping-pong (softmax overlaps the other half's MMAs)
mkdir -p gpurun_out/r02v
ORBIT2_SYNC_CHECK=1 timeout 600 python -m pytest tests/test_gpu_train.py -x -q -s > gpurun_out/r02v/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02v/train_tests.log
timeout 900 python scripts/train_ab.py C2 16 liborbit2.so liborbit2_nopf.so > gpurun_out/r02v/ab_train.log 2>&1
