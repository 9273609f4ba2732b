#!/bin/bash
# loss kernel with the Huber divisions hoisted (multiply by 1 / delta) vs the previous commit: training parity, C2 A/B
OUT=gpurun_out/r02by
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_train_sp.py -m gpu -q -x > $OUT/pytest_train.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_train.log
timeout 900 python scripts/train_ab.py C2 64 $P/liborbit2_old.so $P/liborbit2.so > $OUT/train_ab_C2.log 2>&1
