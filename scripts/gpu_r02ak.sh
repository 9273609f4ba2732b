#!/bin/bash
mkdir -p gpurun_out/r02ak
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so $P/liborbit2_p3.so $P/liborbit2_p4.so $P/liborbit2_p6.so" timeout 900 python scripts/ab_kernels.py C2 64 5 > gpurun_out/r02ak/ab_poly_c2.log 2>&1
