#!/bin/bash
# CTA-pair (cta_group::2) GEMMs: A/B against single-CTA tiles at C3 / C4, then the parity tests that use them
OUT=gpurun_out/r02ba
mkdir -p $OUT
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2_np.so $P/liborbit2.so $P/liborbit2_np.so $P/liborbit2.so" timeout 300 python scripts/ab_kernels.py C3 16 10 > $OUT/ab_C3.log 2>&1
echo "ab exit $?" >> $OUT/ab_C3.log
if grep -q "TOTAL" $OUT/ab_C3.log; then
  timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_train.py -m gpu -q -x -k "sampled or train or full" > $OUT/pytest_sub.log 2>&1
  echo "pytest exit $?" >> $OUT/pytest_sub.log
  AB_LIBS="$P/liborbit2_np.so $P/liborbit2.so" timeout 600 python scripts/ab_kernels.py C4 1 3 > $OUT/ab_C4.log 2>&1
fi
