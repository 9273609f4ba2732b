#!/bin/bash
# round 2: first GPU run of the training step (f3): parity vs the oracle, then the full GPU suite
mkdir -p gpurun_out/r02r
export ORBIT2_SYNC_CHECK=1
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -s > gpurun_out/r02r/train_tests.log 2>&1
echo "train tests rc=$?" >> gpurun_out/r02r/train_tests.log
unset ORBIT2_SYNC_CHECK
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r02r/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r02r/pytest.log
