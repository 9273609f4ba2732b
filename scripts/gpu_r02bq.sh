#!/bin/bash
# attention (two-Q-tile kernel) row sums: 1 / 2 / 4 partial sums, C2 A/B (the three-Q-tile kernel keeps 1)
OUT=gpurun_out/r02bq
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2_rs1.so $P/liborbit2_rs2.so $P/liborbit2.so $P/liborbit2_rs1.so $P/liborbit2_rs2.so $P/liborbit2.so" timeout 900 python scripts/ab_kernels.py C2 64 10 > $OUT/ab_C2.log 2>&1
AB_LIBS="$P/liborbit2_rs1.so $P/liborbit2.so" timeout 600 python scripts/ab_kernels.py C3 16 10 > $OUT/ab_C3.log 2>&1
