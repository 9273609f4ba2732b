#!/bin/bash
# packed erf-GELU epilogue in the generic GEMM (D >= 1024 MLP-up): A/B at C3 and C4
mkdir -p gpurun_out/r02ax
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so $P/liborbit2_g2.so $P/liborbit2.so $P/liborbit2_g2.so" timeout 900 python scripts/ab_kernels.py C3 16 10 > gpurun_out/r02ax/ab_C3.log 2>&1
AB_LIBS="$P/liborbit2.so $P/liborbit2_g2.so" timeout 900 python scripts/ab_kernels.py C4 1 3 > gpurun_out/r02ax/ab_C4.log 2>&1
