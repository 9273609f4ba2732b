#!/bin/bash
# round 2: packed-math attention-backward softmax, packed GELU' epilogue; parity + smoke + timing
mkdir -p gpurun_out/r02x
ORBIT2_SYNC_CHECK=1 timeout 600 python -m pytest tests/test_gpu_train.py -x -q -s > gpurun_out/r02x/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02x/train_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02x/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r02x/smoke.log
timeout 900 python scripts/train_ab.py C2 16 liborbit2.so > gpurun_out/r02x/ab_train.log 2>&1
