#!/bin/bash
mkdir -p gpurun_out/r02am
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so $P/liborbit2_bex2.so" timeout 600 python scripts/ab_kernels.py C2 64 5 > gpurun_out/r02am/ab_bex2_c2.log 2>&1
ORBIT2_LIB=$P/liborbit2_bex2.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -k "C2 or c2" -s > gpurun_out/r02am/parity_bex2.log 2>&1
echo "rc=$?" >> gpurun_out/r02am/parity_bex2.log
