#!/bin/bash
# weight-gradient split count A/B (default, base 16 / 8 waves, base 32 / 16 waves) on the C3 and C2 training steps
OUT=gpurun_out/r02bf
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
timeout 900 python scripts/train_ab.py C3 16 $P/liborbit2.so $P/liborbit2_w16.so $P/liborbit2_w32.so > $OUT/train_ab_C3.log 2>&1
timeout 900 python scripts/train_ab.py C2 64 $P/liborbit2.so $P/liborbit2_w16.so $P/liborbit2_w32.so > $OUT/train_ab_C2.log 2>&1
