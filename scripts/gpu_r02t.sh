#!/bin/bash
# round 2: training parity after the GELU' / LN-backward changes; attention-backward A/B (atomics, exps)
mkdir -p gpurun_out/r02t
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -s > gpurun_out/r02t/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02t/train_tests.log
timeout 900 python scripts/train_ab.py C2 16 liborbit2.so liborbit2_nodq.so liborbit2_nosm.so liborbit2_nodqsm.so > gpurun_out/r02t/ab_train.log 2>&1
