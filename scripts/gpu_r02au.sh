#!/bin/bash
# block_tc grid-size A/B: is the block tail bound by a shared resource (L2) or per SM?
mkdir -p gpurun_out/r02au
P=paper_2505_04802_b200
AB_LIBS="$P/liborbit2.so $P/liborbit2_bg2.so $P/liborbit2_bg4.so" timeout 600 python scripts/ab_kernels.py C2 64 5 > gpurun_out/r02au/ab_grid.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv >> gpurun_out/r02au/ab_grid.log
