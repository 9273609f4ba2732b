#!/bin/bash
# pair GEMM tuning: 4 vs 5 stages, erf vs tanh GELU epilogue (C3), and pair vs single in training (C2)
OUT=gpurun_out/r02bb
mkdir -p $OUT
P=paper_2505_04802_b200
AB_LIBS="$PWD/$P/liborbit2.so $PWD/$P/liborbit2_p5.so $PWD/$P/liborbit2_gt.so $PWD/$P/liborbit2.so $PWD/$P/liborbit2_p5.so $PWD/$P/liborbit2_gt.so" timeout 600 python scripts/ab_kernels.py C3 16 10 > $OUT/ab_C3.log 2>&1
timeout 900 python scripts/train_ab.py C2 64 $PWD/$P/liborbit2_np.so $PWD/$P/liborbit2.so $PWD/$P/liborbit2_np.so $PWD/$P/liborbit2.so > $OUT/train_ab_C2.log 2>&1
timeout 900 python scripts/train_ab.py C3 16 $PWD/$P/liborbit2_np.so $PWD/$P/liborbit2.so > $OUT/train_ab_C3.log 2>&1
