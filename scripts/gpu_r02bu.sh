#!/bin/bash
# three-Q-tile attention row sums: 1 (default) vs 2 partial sums, C3 A/B
OUT=gpurun_out/r02bu
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so $P/liborbit2_a3s2.so $P/liborbit2.so $P/liborbit2_a3s2.so" timeout 900 python scripts/ab_kernels.py C3 16 10 > $OUT/ab_C3.log 2>&1
