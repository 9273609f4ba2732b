#!/bin/bash
# r02c: attention A/B (tail skip, desync) + peer-SP single-GPU test + parity subset.
OUT=gpurun_out/r02c
mkdir -p $OUT
P=paper_2505_04802_b200
export AB_LIBS="$P/liborbit2_base.so $P/liborbit2_skip.so $P/liborbit2_ds1.so $P/liborbit2_ds2.so"
timeout 400 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2.log 2>&1
timeout 300 python scripts/ab_kernels.py C3 16 5 > $OUT/ab_c3.log 2>&1
timeout 600 python -m pytest tests/test_peer_sp.py tests/test_gpu_parity.py -m gpu -q -x -k "peer or small or chunk or rank or C2_full or packing or repeated" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
