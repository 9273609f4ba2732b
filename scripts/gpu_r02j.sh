#!/bin/bash
OUT=gpurun_out/r02j
mkdir -p $OUT
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2_attn3.so $P/liborbit2_a3d400.so $P/liborbit2_a3d700.so" timeout 600 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2.log 2>&1
ORBIT2_LIB=$P/liborbit2_a3d700tl.so timeout 120 python scripts/attn3_timeline.py C2 16 > $OUT/timeline_d700.log 2>&1
