#!/bin/bash
# epilogue TMEM double-buffered loads (chunk c + 1 in flight while c is processed) vs none:
# C2 / C3 inference, C2 / C3 training; parity subset
OUT=gpurun_out/r02bm
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2_ntp.so $P/liborbit2.so $P/liborbit2_ntp.so $P/liborbit2.so" timeout 600 python scripts/ab_kernels.py C3 16 10 > $OUT/ab_C3.log 2>&1
AB_LIBS="$P/liborbit2_ntp.so $P/liborbit2.so $P/liborbit2_ntp.so $P/liborbit2.so" timeout 600 python scripts/ab_kernels.py C2 64 10 > $OUT/ab_C2.log 2>&1
timeout 900 python scripts/train_ab.py C2 64 $P/liborbit2_ntp.so $P/liborbit2.so > $OUT/train_ab_C2.log 2>&1
timeout 900 python scripts/train_ab.py C3 16 $P/liborbit2_ntp.so $P/liborbit2.so > $OUT/train_ab_C3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_parity.py -m gpu -q -x -k "train or cta_pair or sampled" > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
