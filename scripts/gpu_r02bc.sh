#!/bin/bash
# pair GEMMs (5-stage residual, tanh GELU epilogue) vs single-CTA: inference C3, training C2 / C3; parity subset
OUT=gpurun_out/r02bc
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2_np.so $P/liborbit2.so $P/liborbit2_np.so $P/liborbit2.so" timeout 600 python scripts/ab_kernels.py C3 16 10 > $OUT/ab_C3.log 2>&1
timeout 900 python scripts/train_ab.py C2 64 $P/liborbit2_np.so $P/liborbit2.so $P/liborbit2_np.so $P/liborbit2.so > $OUT/train_ab_C2.log 2>&1
timeout 900 python scripts/train_ab.py C3 16 $P/liborbit2_np.so $P/liborbit2.so > $OUT/train_ab_C3.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m gpu -q -x -k "sampled or train or full or unfused" > $OUT/pytest_sub.log 2>&1
echo "pytest exit $?" >> $OUT/pytest_sub.log
