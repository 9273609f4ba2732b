#!/bin/bash
# round 2: compression kernels parity (f4), training parity after the wgrad wave fix, timing
mkdir -p gpurun_out/r02z
ORBIT2_SYNC_CHECK=1 timeout 900 python -m pytest tests/test_gpu_compress.py -x -q -s > gpurun_out/r02z/compress_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02z/compress_tests.log
timeout 600 python -m pytest tests/test_gpu_train.py -x -q > gpurun_out/r02z/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02z/train_tests.log
timeout 900 python scripts/train_ab.py C2 16 liborbit2.so > gpurun_out/r02z/ab_train.log 2>&1
