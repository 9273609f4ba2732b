#!/bin/bash
# weight-gradient splits by a chunk target (<= 64 / 128 chunks of 64 tokens per CTA) vs the fill heuristic and base-32 splits
OUT=gpurun_out/r02bg
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
timeout 900 python scripts/train_ab.py C3 16 $P/liborbit2.so $P/liborbit2_w32.so $P/liborbit2_c64.so $P/liborbit2_c128.so > $OUT/train_ab_C3.log 2>&1
timeout 900 python scripts/train_ab.py C2 64 $P/liborbit2.so $P/liborbit2_w32.so $P/liborbit2_c64.so $P/liborbit2_c128.so > $OUT/train_ab_C2.log 2>&1
