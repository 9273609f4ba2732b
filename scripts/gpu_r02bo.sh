#!/bin/bash
# embedding epilogue: position-embedding chunk loaded one chunk ahead vs not: C2 A/B + parity
OUT=gpurun_out/r02bo
mkdir -p $OUT
P=$PWD/paper_2505_04802_b200
AB_LIBS="$P/liborbit2_epp0.so $P/liborbit2.so $P/liborbit2_epp0.so $P/liborbit2.so" timeout 600 python scripts/ab_kernels.py C2 64 10 > $OUT/ab_C2.log 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py -m gpu -q -x > $OUT/pytest.log 2>&1
echo "pytest exit $?" >> $OUT/pytest.log
