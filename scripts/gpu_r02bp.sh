#!/bin/bash
# attention row sums: 1 chain (round-2 code) vs 4 / 8 independent partial sums; C2 and C3 A/B + parity
OUT=gpurun_out/r02bp
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2_rs1.so $P/liborbit2.so $P/liborbit2_rs8.so $P/liborbit2_rs1.so $P/liborbit2.so $P/liborbit2_rs8.so" timeout 900 python scripts/ab_kernels.py C2 64 10 > $OUT/ab_C2.log 2>&1
AB_LIBS="$P/liborbit2_rs1.so $P/liborbit2.so $P/liborbit2_rs8.so" timeout 600 python scripts/ab_kernels.py C3 16 10 > $OUT/ab_C3.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
