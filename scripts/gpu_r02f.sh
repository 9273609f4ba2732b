#!/bin/bash
# r02f: lazy row max A/B, parity subset incl. lazy-vs-eager test, peer SP 2-GPU tests.
OUT=gpurun_out/r02f
mkdir -p $OUT
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so" timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_lazy.log 2>&1
AB_LIBS="$P/liborbit2.so" ORBIT2_ATTN_EAGER_MAX=1 timeout 300 python scripts/ab_kernels.py C2 64 5 > $OUT/ab_c2_eager.log 2>&1
AB_LIBS="$P/liborbit2.so" timeout 300 python scripts/ab_kernels.py C3 16 5 > $OUT/ab_c3_lazy.log 2>&1
AB_LIBS="$P/liborbit2.so" ORBIT2_ATTN_EAGER_MAX=1 timeout 300 python scripts/ab_kernels.py C3 16 5 > $OUT/ab_c3_eager.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_peer_sp.py -m gpu -q -s -k "small or C2_full or chunk or rank or packing or repeated or coordinate or zero_head or peer or bench_configuration or lazy" > $OUT/pytest.log 2>&1; echo "pytest exit $?" >> $OUT/pytest.log
