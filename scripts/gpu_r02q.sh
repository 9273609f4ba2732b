#!/bin/bash
OUT=gpurun_out/r02q
mkdir -p $OUT
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so $P/liborbit2_a2s600.so $P/liborbit2_a2s1000.so" timeout 600 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2.log 2>&1
ORBIT2_LIB=$P/liborbit2_a2tl.so timeout 120 python scripts/attn_timeline.py C2 16 > $OUT/timeline_base.log 2>&1
ORBIT2_LIB=$P/liborbit2_a2s1000tl.so timeout 120 python scripts/attn_timeline.py C2 16 > $OUT/timeline_s1000.log 2>&1
ORBIT2_E2E_GROUPS=16 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-profile > $OUT/bench_e2e16.log 2>&1
ORBIT2_E2E_GROUPS=8 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-profile > $OUT/bench_e2e8.log 2>&1
ORBIT2_E2E_GROUPS=32 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-profile > $OUT/bench_e2e32.log 2>&1
