#!/bin/bash
# LayerNorm statistics with short dependency chains (block tail: paired squares; GEMM LN
# epilogues: 4 partial sums) vs the previous commit: C2 A/B, training C2 A/B, parity
OUT=gpurun_out/r02br
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2_old.so $P/liborbit2.so $P/liborbit2_old.so $P/liborbit2.so" timeout 900 python scripts/ab_kernels.py C2 64 10 > $OUT/ab_C2.log 2>&1
timeout 900 python scripts/train_ab.py C2 64 $P/liborbit2_old.so $P/liborbit2.so > $OUT/train_ab_C2.log 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m gpu -q -x > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
