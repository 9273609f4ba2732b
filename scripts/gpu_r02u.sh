#!/bin/bash
# round 2: training parity after GELU' / LN-backward / loss / TMA dQ-reduce changes; A/B vs no dQ
mkdir -p gpurun_out/r02u
timeout 600 python -m pytest tests/test_gpu_train.py -x -q -s > gpurun_out/r02u/train_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02u/train_tests.log
timeout 900 python scripts/train_ab.py C2 16 liborbit2.so liborbit2_nodq.so > gpurun_out/r02u/ab_train.log 2>&1
