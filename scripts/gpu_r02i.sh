#!/bin/bash
# r02i: attn3 variants (poly share, ring depth, register realloc) + clock64 timeline.
OUT=gpurun_out/r02i
mkdir -p $OUT
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2_attn3.so $P/liborbit2_a3p4.so $P/liborbit2_a3p0.so $P/liborbit2_a3kv4.so $P/liborbit2_a3nr.so" timeout 600 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2.log 2>&1
ORBIT2_LIB=$P/liborbit2_a3tl.so timeout 120 python scripts/attn3_timeline.py C2 16 > $OUT/timeline.log 2>&1
