#!/bin/bash
# order vs power: is the first process's slower attention a warm-up effect or power capping?
mkdir -p gpurun_out/r02av
P=paper_2505_04802_b200
nvidia-smi --query-gpu=clocks.sm,power.draw,power.limit,clocks_throttle_reasons.active --format=csv -lms 200 > gpurun_out/r02av/smi.csv &
SMI=$!
AB_LIBS="$P/liborbit2.so $P/liborbit2.so $P/liborbit2_bg2.so $P/liborbit2.so" timeout 600 python scripts/ab_kernels.py C2 64 20 > gpurun_out/r02av/ab_order.log 2>&1
kill $SMI
