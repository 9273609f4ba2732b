#!/bin/bash
# r02e: separable SIMT stitch, TMA gather (attribute fix), parity subset, A/B of stitch forms.
OUT=gpurun_out/r02e
mkdir -p $OUT
P=paper_2505_04802_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_peer_sp.py -m gpu -q -x -s -k "small or C2_full or chunk or rank or packing or repeated or coordinate or zero_head or peer or bench_configuration or unfused" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
AB_LIBS="$P/liborbit2.so" timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_default.log 2>&1
AB_LIBS="$P/liborbit2.so" ORBIT2_STITCH_PER_ELEMENT=1 timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_stitch_perelem.log 2>&1
AB_LIBS="$P/liborbit2.so" ORBIT2_TMA_STITCH=1 timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_stitch_tma.log 2>&1
