#!/bin/bash
# two-Q-tile attention block max with 4 / 8 / 16 independent running maxima (exact: output bit-identical), C2 A/B
OUT=gpurun_out/r02bs
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so $P/liborbit2_mx8.so $P/liborbit2_mx16.so $P/liborbit2.so $P/liborbit2_mx8.so $P/liborbit2_mx16.so" timeout 900 python scripts/ab_kernels.py C2 64 10 > $OUT/ab_C2.log 2>&1
