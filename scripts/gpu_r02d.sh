#!/bin/bash
# r02d: TMA gather + TMA stitch + 64-key tail skip: parity subset, A/B, peer SP over 2 GPUs.
OUT=gpurun_out/r02d
mkdir -p $OUT
P=paper_2505_04802_b200
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_peer_sp.py -m gpu -q -x -s -k "small or C2_full or chunk or rank or packing or repeated or coordinate or zero_head or peer or bench_configuration" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
export AB_LIBS="$P/liborbit2_noskip.so $P/liborbit2_skip64.so"
timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2.log 2>&1
timeout 300 python scripts/ab_kernels.py C3 16 5 > $OUT/ab_c3.log 2>&1
AB_LIBS="$P/liborbit2.so" ORBIT2_SIMT_GATHER=1 ORBIT2_SIMT_STITCH=1 timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_simt_gather_stitch.log 2>&1
