#!/bin/bash
# two-Q-tile attention: exponentials per 16 on the FMA pipe (polynomial) 0 / 2 (default) / 4, re-tuned
# after the row-sum split, C2 A/B
OUT=gpurun_out/r02bt
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2_po0.so $P/liborbit2.so $P/liborbit2_po4.so $P/liborbit2_po0.so $P/liborbit2.so $P/liborbit2_po4.so" timeout 900 python scripts/ab_kernels.py C2 64 10 > $OUT/ab_C2.log 2>&1
